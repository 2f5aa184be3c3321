"""paper_1501_06561_b200 — B200-native Frequent Directions sketching (arXiv:1501.06561).

Python binding of libfd.so (C ABI in include/fd.h).  This layer marshals
arguments only: every step of the sketch and of the evaluator runs in the
sm_100a kernels of libfd.so.  PyTorch supplies device memory (the workspace),
the CUDA stream and torch.distributed process groups.

    sk = Sketcher(d=1024, ell=128, variant="fast_fd", n_shards=1184)
    sk.append(A)                       # A: cuda fp32 (n x d) tensor
    B, stats = sk.sketch()             # ell x d sketch (last row zero)
    res = cov_err(A, B)                # ||A^T A - B^T B||_2 / ||A||_F^2
"""
from __future__ import annotations

import ctypes

from ._lib import FD_MAX_N, VARIANT, FdConfig, FdError, FdStats, check, lib

__all__ = ["Sketcher", "cov_err", "cov_gram_partial", "cov_err_from_gram", "cov_frob_from_gram", "proj_err", "proj_err_from_gram", "hash_sketch", "FdError", "VARIANT", "FD_MAX_N",
           "is_batched"]


def _torch():
    import torch
    return torch


def is_batched(variant: str) -> bool:
    return variant.startswith("fast_")


def _as_rows(t, d):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or t.dim() != 2 or t.dtype != torch.float32:
        raise TypeError("rows must be a 2-D float32 torch tensor")
    if t.shape[1] != d:
        raise ValueError(f"rows have {t.shape[1]} columns, sketch has d={d}")
    if t.shape[0] > 0 and t.stride(1) != 1:
        t = t.contiguous()
    return t


class Sketcher:
    """One FD sketch stream (handle + workspace) on a CUDA device."""

    def __init__(self, d: int, ell: int, variant: str = "fast_fd", alpha: float = 0.2, n_shards: int = 1,
                 device=None, stream=None):
        torch = _torch()
        if variant not in VARIANT:
            raise ValueError(f"unknown variant {variant!r}; one of {sorted(VARIANT)}")
        device = torch.device("cuda") if device is None else torch.device(device)
        if device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.d, self.ell, self.variant, self.alpha, self.n_shards = int(d), int(ell), variant, float(alpha), int(n_shards)
        self.cfg = FdConfig(self.d, self.ell, VARIANT[variant], self.alpha, self.n_shards,
                            self.device.index if self.device.index is not None else 0)
        nbytes = lib().fd_workspace_bytes(ctypes.byref(self.cfg))
        if nbytes == 0:
            raise FdError(-1, "invalid configuration")
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        check(lib().fd_create(ctypes.byref(self.cfg), self.ws.data_ptr(), nbytes, self.stream.cuda_stream,
                              ctypes.byref(h)))
        self.h = h
        self._keep = []  # host inputs kept alive until the next sync point
        self._stage = None  # device staging buffer of fd_append_rows_host

    # -- streaming ---------------------------------------------------------
    def append(self, rows):
        """Append rows (n x d fp32).  Device tensors are read in place (async).
        Host tensors go through fd_append_rows_host: each lockstep round's rows
        are copied host -> device into a staging buffer while the previous round
        computes (pin the host tensor for the copies to overlap)."""
        torch = _torch()
        rows = _as_rows(rows, self.d)
        if rows.shape[0] == 0:
            return self
        if not rows.is_cuda:
            ld = rows.stride(0)
            nbytes = lib().fd_host_stage_bytes(ctypes.byref(self.cfg), ld)
            if self._stage is None or self._stage.numel() < nbytes:
                self._stage = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._keep.append(rows)   # must outlive the asynchronous copies
            check(lib().fd_append_rows_host(self.h, rows.data_ptr(), rows.shape[0], ld, self._stage.data_ptr(),
                                            self._stage.numel()))
            return self
        check(lib().fd_append_rows(self.h, rows.data_ptr(), rows.shape[0], rows.stride(0)))
        return self

    def sketch(self, out=None, stats: bool = True):
        """ell x d sketch (non-destructive snapshot).  Returns (B, stats-dict or None)."""
        torch = _torch()
        B = out if out is not None else torch.empty((self.ell, self.d), dtype=torch.float32, device=self.device)
        st = FdStats() if stats else None
        check(lib().fd_sketch(self.h, B.data_ptr(), ctypes.byref(st) if st is not None else None))
        if stats:
            self._keep.clear()
        return B, (st.as_dict() if st is not None else None)

    def merge(self, sketches, out=None, stats: bool = False):
        """Merge a (count x ell x d) device tensor of sketches by the recursive-halving tree."""
        torch = _torch()
        S = sketches.contiguous()
        assert S.dim() == 3 and S.shape[1] == self.ell and S.shape[2] == self.d and S.is_cuda
        B = out if out is not None else torch.empty((self.ell, self.d), dtype=torch.float32, device=self.device)
        st = FdStats() if stats else None
        check(lib().fd_merge(self.h, S.data_ptr(), S.shape[0], B.data_ptr(),
                             ctypes.byref(st) if st is not None else None))
        return B, (st.as_dict() if st is not None else None)

    def shard_sketch(self, shard: int, out=None):
        torch = _torch()
        B = out if out is not None else torch.empty((self.ell, self.d), dtype=torch.float32, device=self.device)
        check(lib().fd_shard_sketch(self.h, int(shard), B.data_ptr()))
        return B

    def reset(self):
        """Start a fresh stream with the same handle and workspace."""
        check(lib().fd_reset(self.h))
        if self._keep:
            # the last staged host->device copies may still read the pinned inputs
            self.stream.synchronize()
            self._keep.clear()
        return self

    def profile(self, enable=True):
        check(lib().fd_profile(self.h, 1 if enable else 0))

    KERNELS = ("ingest", "gram", "eig", "recon", "trd", "bt", "perrow")

    def profile_read(self):
        """{kernel: (total_ms, launches)} since the last read (synchronises)."""
        k = len(self.KERNELS)
        ms = (ctypes.c_double * k)()
        n = (ctypes.c_int64 * k)()
        lib().fd_profile_read(self.h, ms, n, k)
        return {k: (ms[i], n[i]) for i, k in enumerate(self.KERNELS)}

    def close(self):
        if getattr(self, "h", None):
            lib().fd_destroy(self.h)
            self.h = None
            self.ws = None
            self._stage = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# -- evaluator -------------------------------------------------------------
def _cov_ws(d, device):
    torch = _torch()
    n = lib().fd_cov_workspace_bytes(int(d))
    return torch.empty(n, dtype=torch.uint8, device=device), n


def cov_gram_partial(A, AtA, stream=None):
    """AtA (d x d fp64 cuda) += A^T A (tcgen05 int8 slices, exact int32 sums, fp64 drains)."""
    torch = _torch()
    A = _as_rows(A, AtA.shape[0])
    s = stream if stream is not None else torch.cuda.current_stream(A.device)
    nb = lib().fd_cov_gram_workspace_bytes(A.shape[0], A.shape[1])
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=A.device)
    check(lib().fd_cov_gram_partial(A.data_ptr(), A.shape[0], A.stride(0), A.shape[1], AtA.data_ptr(),
                                    ws.data_ptr(), nb, s.cuda_stream))
    return AtA


def cov_frob_from_gram(AtA, stream=None):
    """||A||_F^2 = trace(AtA) of a d x d fp64 cuda Gram (fd_cov_frob_from_gram; synchronises)."""
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(AtA.device)
    out = ctypes.c_double()
    check(lib().fd_cov_frob_from_gram(AtA.data_ptr(), AtA.shape[0], ctypes.byref(out), s.cuda_stream))
    return out.value


def cov_err_from_gram(AtA, B, frob_sq, stream=None):
    torch = _torch()
    d = AtA.shape[0]
    B = B.contiguous()
    ws, n = _cov_ws(d, AtA.device)
    s = stream if stream is not None else torch.cuda.current_stream(AtA.device)
    err, hi, lo = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    check(lib().fd_cov_err_from_gram(AtA.data_ptr(), B.data_ptr(), B.shape[0], d, float(frob_sq), ctypes.byref(err),
                                     ctypes.byref(hi), ctypes.byref(lo), ws.data_ptr(), n, s.cuda_stream))
    return dict(err=err.value, lmax=hi.value, lmin=lo.value, frob=float(frob_sq))


def cov_err(A, B, stream=None):
    """cov-err of sketch B (ell x d) for rows A (n x d), both cuda fp32."""
    torch = _torch()
    d = B.shape[1]
    A = _as_rows(A, d)
    B = B.contiguous()
    ws, n = _cov_ws(d, A.device)
    s = stream if stream is not None else torch.cuda.current_stream(A.device)
    err, hi, lo = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    check(lib().fd_cov_err(A.data_ptr(), A.shape[0], A.stride(0), B.data_ptr(), B.shape[0], d, ctypes.byref(err),
                           ctypes.byref(hi), ctypes.byref(lo), ws.data_ptr(), n, s.cuda_stream))
    frob = None
    return dict(err=err.value, lmax=hi.value, lmin=lo.value, frob=frob)


def proj_err_from_gram(AtA, B, frob_sq, k=10, stream=None):
    """proj-err (k = 10 per PAPER.md:572) of sketch B (ell x d cuda fp32)
    from AtA (d x d cuda fp64, fd_cov_gram_partial) and frob_sq = ||A||_F^2."""
    torch = _torch()
    d = AtA.shape[0]
    B = B.contiguous()
    n = lib().fd_proj_workspace_bytes(int(d), int(B.shape[0]), int(k))
    ws = torch.empty(max(n, 1), dtype=torch.uint8, device=AtA.device)
    s = stream if stream is not None else torch.cuda.current_stream(AtA.device)
    pe, nu, de = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    check(lib().fd_proj_err_from_gram(AtA.data_ptr(), B.data_ptr(), B.shape[0], d, float(frob_sq), int(k),
                                      ctypes.byref(pe), ctypes.byref(nu), ctypes.byref(de), ws.data_ptr(), n,
                                      s.cuda_stream))
    return dict(err=pe.value, num=nu.value, den=de.value, frob=float(frob_sq))


def proj_err(A, B, k=10, stream=None):
    """proj-err of sketch B (ell x d) for rows A (n x d), both cuda fp32."""
    torch = _torch()
    d = B.shape[1]
    A = _as_rows(A, d)
    B = B.contiguous()
    n = lib().fd_proj_workspace_bytes(int(d), int(B.shape[0]), int(k))
    nb = n + (d * d * 8 + 255) // 256 * 256 + lib().fd_cov_gram_workspace_bytes(A.shape[0], d)
    ws = torch.empty(nb, dtype=torch.uint8, device=A.device)
    s = stream if stream is not None else torch.cuda.current_stream(A.device)
    pe = ctypes.c_double()
    check(lib().fd_proj_err(A.data_ptr(), A.shape[0], A.stride(0), B.data_ptr(), B.shape[0], d, int(k),
                            ctypes.byref(pe), ws.data_ptr(), nb, s.cuda_stream))
    return dict(err=pe.value)


def hash_sketch(A, ell, s=4, seed=0, row0=0, B=None, stream=None):
    """Hashing (s = 1) / OSNAP sketch: B (ell x d cuda fp64) += S A for the
    rows A (n x d cuda fp32) = rows row0.. of the stream.  Returns B (fp64 accumulator)."""
    torch = _torch()
    d = A.shape[1]
    A = _as_rows(A, d)
    if B is None:
        B = torch.zeros((ell, d), dtype=torch.float64, device=A.device)
    assert B.dtype == torch.float64 and B.is_contiguous() and tuple(B.shape) == (ell, d)
    n = lib().fd_hash_workspace_bytes(int(d), int(ell))
    ws = torch.empty(max(n, 1), dtype=torch.uint8, device=A.device)
    st = stream if stream is not None else torch.cuda.current_stream(A.device)
    check(lib().fd_hash_sketch(A.data_ptr(), A.shape[0], A.stride(0), d, int(ell), int(s), int(seed), int(row0),
                               B.data_ptr(), ws.data_ptr(), n, st.cuda_stream))
    return B
