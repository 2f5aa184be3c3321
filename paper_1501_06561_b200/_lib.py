"""ctypes loader for libfd.so (the C ABI declared in include/fd.h).

Argument marshalling only.  There is no fallback: if the in-tree CUDA library
is missing, importing the package still works but every call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfd.so")

FD_OK = 0
STATUS = {
    0: "FD_OK", -1: "FD_ERR_INVALID_ARG", -2: "FD_ERR_SHAPE", -3: "FD_ERR_ALIGNMENT",
    -4: "FD_ERR_WORKSPACE", -5: "FD_ERR_NONFINITE", -6: "FD_ERR_ZERO_NORM", -7: "FD_ERR_CUDA",
    -8: "FD_ERR_UNSUPPORTED", -9: "FD_ERR_STATE",
}
VARIANT = {"fd": 0, "fast_fd": 1, "alpha_fd": 2, "fast_alpha_fd": 3, "isvd": 4, "fast_isvd": 5,
           "fast_alpha_fd_paper": 6, "ssd": 7, "cfd": 8}
FD_MAX_N = 416

# every symbol include/fd.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "fd_workspace_bytes", "fd_create", "fd_append_rows", "fd_host_stage_bytes", "fd_append_rows_host", "fd_sketch", "fd_merge", "fd_shard_sketch",
    "fd_destroy", "fd_reset", "fd_profile", "fd_profile_read", "fd_cov_workspace_bytes", "fd_cov_gram_workspace_bytes", "fd_cov_gram_partial", "fd_cov_err_from_gram", "fd_cov_frob_from_gram", "fd_cov_err",
    "fd_proj_workspace_bytes", "fd_proj_err_from_gram", "fd_proj_err", "fd_hash_workspace_bytes", "fd_hash_sketch",
    "fd_last_error", "fd_version",
]


class FdConfig(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int64), ("ell", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("n_shards", ctypes.c_int32), ("device", ctypes.c_int32)]


class FdStats(ctypes.Structure):
    _fields_ = [("rows_seen", ctypes.c_int64), ("n_shrinks", ctypes.c_int64), ("frob_sq", ctypes.c_double),
                ("delta_total", ctypes.c_double), ("removed_mass", ctypes.c_double), ("nonfinite", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class FdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python build.py` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, dbl, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_size_t
        dp = ctypes.POINTER(ctypes.c_double)
        L.fd_workspace_bytes.argtypes = [ctypes.POINTER(FdConfig)]
        L.fd_workspace_bytes.restype = sz
        L.fd_create.argtypes = [ctypes.POINTER(FdConfig), vp, sz, vp, ctypes.POINTER(vp)]
        L.fd_append_rows.argtypes = [vp, vp, i64, i64]
        L.fd_host_stage_bytes.argtypes = [ctypes.POINTER(FdConfig), i64]
        L.fd_host_stage_bytes.restype = sz
        L.fd_append_rows_host.argtypes = [vp, vp, i64, i64, vp, sz]
        L.fd_sketch.argtypes = [vp, vp, ctypes.POINTER(FdStats)]
        L.fd_merge.argtypes = [vp, vp, i32, vp, ctypes.POINTER(FdStats)]
        L.fd_shard_sketch.argtypes = [vp, i32, vp]
        L.fd_destroy.argtypes = [vp]
        L.fd_reset.argtypes = [vp]
        L.fd_profile.argtypes = [vp, i32]
        L.fd_profile_read.argtypes = [vp, dp, ctypes.POINTER(ctypes.c_int64), i32]
        L.fd_profile_read.restype = ctypes.c_int32
        L.fd_cov_workspace_bytes.argtypes = [i64]
        L.fd_cov_workspace_bytes.restype = sz
        L.fd_cov_gram_workspace_bytes.argtypes = [i64, i64]
        L.fd_cov_gram_workspace_bytes.restype = sz
        L.fd_cov_gram_partial.argtypes = [vp, i64, i64, i64, vp, vp, sz, vp]
        L.fd_cov_err_from_gram.argtypes = [vp, vp, i32, i64, dbl, dp, dp, dp, vp, sz, vp]
        L.fd_cov_frob_from_gram.argtypes = [vp, i64, dp, vp]
        L.fd_cov_err.argtypes = [vp, i64, i64, vp, i32, i64, dp, dp, dp, vp, sz, vp]
        L.fd_proj_workspace_bytes.argtypes = [i64, i32, i32]
        L.fd_proj_workspace_bytes.restype = sz
        L.fd_proj_err_from_gram.argtypes = [vp, vp, i32, i64, dbl, i32, dp, dp, dp, vp, sz, vp]
        L.fd_proj_err.argtypes = [vp, i64, i64, vp, i32, i64, i32, dp, vp, sz, vp]
        L.fd_hash_workspace_bytes.argtypes = [i64, i32]
        L.fd_hash_workspace_bytes.restype = sz
        L.fd_hash_sketch.argtypes = [vp, i64, i64, i64, i32, i32, ctypes.c_uint64, i64, vp, vp, sz, vp]
        for f in ("fd_create", "fd_append_rows", "fd_append_rows_host", "fd_sketch", "fd_merge", "fd_shard_sketch", "fd_destroy",
                  "fd_reset", "fd_profile",
                  "fd_cov_gram_partial", "fd_cov_err_from_gram", "fd_cov_frob_from_gram", "fd_cov_err", "fd_proj_err_from_gram", "fd_proj_err", "fd_hash_sketch"):
            getattr(L, f).restype = ctypes.c_int
        L.fd_last_error.restype = ctypes.c_char_p
        L.fd_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def check(status):
    if status != FD_OK:
        raise FdError(status, lib().fd_last_error().decode())
    return status
