"""CPU-side checks of the C ABI (no GPU needed): the in-tree libfd.so loads,
exports every symbol include/fd.h declares, and rejects bad configurations
before touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    from paper_1501_06561_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "fd.h")).read()
    declared = set(re.findall(r"^\s*(?:fd_status|size_t|int32_t|const char\*)\s+(fd_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.fd_version().decode().startswith("fd-b200")


def test_library_is_sm100a():
    import subprocess
    so = os.path.join(ROOT, "paper_1501_06561_b200", "libfd.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _cfg(**kw):
    from paper_1501_06561_b200._lib import FdConfig
    c = dict(d=64, ell=16, variant=1, alpha=0.2, n_shards=1, device=0)
    c.update(kw)
    return FdConfig(c["d"], c["ell"], c["variant"], c["alpha"], c["n_shards"], c["device"])


def test_workspace_bytes_and_validation():
    from paper_1501_06561_b200 import _lib
    L = _lib.lib()
    assert L.fd_workspace_bytes(ctypes.byref(_cfg())) > 0
    assert L.fd_workspace_bytes(ctypes.byref(_cfg(d=0))) == 0
    assert L.fd_workspace_bytes(ctypes.byref(_cfg(ell=1))) == 0
    assert L.fd_workspace_bytes(ctypes.byref(_cfg(n_shards=0))) == 0
    assert L.fd_workspace_bytes(ctypes.byref(_cfg(variant=3, alpha=0.0))) == 0
    assert L.fd_workspace_bytes(ctypes.byref(_cfg(variant=9))) == 0
    # bigger P -> bigger workspace
    assert L.fd_workspace_bytes(ctypes.byref(_cfg(n_shards=8))) > L.fd_workspace_bytes(ctypes.byref(_cfg()))
    h = ctypes.c_void_p()
    assert L.fd_create(ctypes.byref(_cfg(ell=1)), None, 0, None, ctypes.byref(h)) == -1
    assert L.fd_create(ctypes.byref(_cfg(ell=209, variant=1)), ctypes.c_void_p(1), 1 << 40, None,
                       ctypes.byref(h)) == -8
    assert L.fd_create(ctypes.byref(_cfg()), None, 0, None, ctypes.byref(h)) == -4
    assert L.fd_cov_workspace_bytes(0) == 0 and L.fd_cov_workspace_bytes(64) > 64 * 64 * 8


def test_append_argument_errors_without_device():
    from paper_1501_06561_b200 import _lib
    L = _lib.lib()
    assert L.fd_append_rows(None, None, 0, 0) == -1
    assert L.fd_sketch(None, None, None) == -1
    assert L.fd_cov_err_from_gram(ctypes.c_void_p(8), ctypes.c_void_p(8), 4, 16, 0.0, ctypes.byref(ctypes.c_double()),
                                  None, None, None, 0, None) == -6
