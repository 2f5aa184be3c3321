"""fdgen — seeded synthetic input generators for the five BASELINE.json workloads.

This module is the ONE piece shared by the CPU oracle (tests) and the GPU path
(bench / tests): it produces the input rows A and nothing else.  It contains
none of the sketching method's arithmetic.

Rows are produced by ``libfdgen.so`` (fdgen/csrc): a host generator and a
device generator built from the same ``__host__ __device__`` source, which use
only correctly-rounded IEEE operations, so both produce identical fp32 bytes
(checked by ``tests/test_gpu_parity.py::test_generator_host_device_bitexact``).
The small fp64 factor matrices (D·U of the low-rank signal, the drifting
subspaces V_j, the fixed direction e) come from numpy ``default_rng(seed)`` and
LAPACK QR here, once per workload, and are passed to both generators.

Recipes (DESIGN.md §3 states them with the paper citations):
  noisy   A = S·D·U + N/ζ                 PAPER.md:539-541 (Random Noisy), D_ii = 1-(i-1)/k
  image   clip(rint(255·minmax(S·D·U) + σN), 0, 255)/255   (BASELINE config 3)
  drift   block-wise 8-dim subspaces, scale 1.5^(j mod 5), e every 100th row (config 5)
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfdgen.so")

KIND_NOISY, KIND_IMAGE, KIND_DRIFT = 0, 1, 2


class FdgParams(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("d", ctypes.c_int64),
        ("k", ctypes.c_int),
        ("key0", ctypes.c_uint32),
        ("key1", ctypes.c_uint32),
        ("noise_scale", ctypes.c_double),
        ("DU", ctypes.c_void_p),
        ("e", ctypes.c_void_p),
        ("xmin", ctypes.c_double),
        ("xmax", ctypes.c_double),
        ("block_rows", ctypes.c_int64),
        ("period", ctypes.c_int64),
        ("nblocks", ctypes.c_int),
        ("growth", ctypes.c_double),
        ("cycle", ctypes.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `python build.py` first")
        L = ctypes.CDLL(_LIB_PATH)
        L.fdg_host_rows.argtypes = [ctypes.POINTER(FdgParams), ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.c_int64]
        L.fdg_host_rows.restype = ctypes.c_int
        L.fdg_host_minmax.argtypes = [ctypes.POINTER(FdgParams), ctypes.c_int64, ctypes.c_int64,
                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.fdg_host_minmax.restype = ctypes.c_int
        L.fdg_dev_rows.argtypes = [ctypes.POINTER(FdgParams), ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.fdg_dev_rows.restype = ctypes.c_int
        L.fdg_dev_minmax.argtypes = [ctypes.POINTER(FdgParams), ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_void_p]
        L.fdg_dev_minmax.restype = ctypes.c_int
        L.fdg_key_to_double.argtypes = [ctypes.c_ulonglong]
        L.fdg_key_to_double.restype = ctypes.c_double
        _lib = L
    return _lib


@dataclass
class Workload:
    name: str
    n: int
    d: int
    kind: int
    k: int
    seed: int
    ells: tuple
    factors: np.ndarray            # fp64, C-contiguous (k x d, or nblk x k x d)
    e: np.ndarray | None = None    # drift only
    noise_scale: float = 10.0
    xminmax: tuple | None = None   # image only (filled lazily)
    extra: dict = field(default_factory=dict)

    def params(self, factors_ptr=None, e_ptr=None) -> FdgParams:
        p = FdgParams()
        p.kind = self.kind
        p.d = self.d
        p.k = self.k
        p.key0 = self.seed & 0xFFFFFFFF
        p.key1 = (0x46440000 + self.kind * 0x101) ^ ((self.seed >> 32) & 0xFFFFFFFF)
        p.noise_scale = self.noise_scale
        p.DU = factors_ptr if factors_ptr is not None else self.factors.ctypes.data
        if self.e is not None:
            p.e = e_ptr if e_ptr is not None else self.e.ctypes.data
        if self.xminmax is not None:
            p.xmin, p.xmax = self.xminmax
        p.block_rows = self.extra.get("block_rows", 1)
        p.period = self.extra.get("period", 0)
        p.nblocks = self.extra.get("nblocks", 1)
        p.growth = self.extra.get("growth", 1.0)
        p.cycle = self.extra.get("cycle", 1)
        return p


def _orthonormal_rows(rng, k, d):
    """k x d matrix with orthonormal rows: Q^T of the QR of a d x k Gaussian (sign-fixed)."""
    g = rng.standard_normal((d, k))
    q, r = np.linalg.qr(g)
    q = q * np.sign(np.diag(r))[None, :]
    return np.ascontiguousarray(q.T)


def noisy_lowrank(name, n, d, k, seed=0, zeta=10.0, ells=()):
    """Random Noisy: A = S D U + N/zeta, D_ii = 1-(i-1)/k (reading C13)."""
    rng = np.random.default_rng(seed)
    U = _orthonormal_rows(rng, k, d)
    D = 1.0 - np.arange(k, dtype=np.float64) / k
    DU = np.ascontiguousarray(D[:, None] * U)
    return Workload(name, n, d, KIND_NOISY, k, seed, tuple(ells), DU, noise_scale=zeta)


def image_like(name, n, d, rank=100, sigma=8.0, seed=0, ells=()):
    """Config 3 (CIFAR-10-shaped stand-in, reading C14)."""
    rng = np.random.default_rng(seed)
    U = _orthonormal_rows(rng, rank, d)
    D = 1.0 - np.arange(rank, dtype=np.float64) / rank
    DU = np.ascontiguousarray(D[:, None] * U)
    return Workload(name, n, d, KIND_IMAGE, rank, seed, tuple(ells), DU, noise_scale=sigma)


def drift(name, n, d, nblocks=20, sub=8, growth=1.5, cycle=5, period=100, e_norm=3.0, seed=0, ells=()):
    """Config 5 (drifting subspaces, reading C15)."""
    rng = np.random.default_rng(seed)
    e = rng.standard_normal(d)
    e = np.ascontiguousarray(e_norm * e / np.linalg.norm(e))
    V = np.stack([_orthonormal_rows(rng, sub, d) for _ in range(nblocks)])
    V = np.ascontiguousarray(V)
    extra = dict(block_rows=n // nblocks, period=period, nblocks=nblocks, growth=growth, cycle=cycle)
    return Workload(name, n, d, KIND_DRIFT, sub, seed, tuple(ells), V, e=e, noise_scale=1.0, extra=extra)


def config(cfg: str, seed: int = 0, n: int | None = None) -> Workload:
    """The five BASELINE.json configs (c1..c5). `n` overrides the row count (prefix)."""
    if cfg == "c1":
        w = noisy_lowrank("c1", 2000, 64, 8, seed, ells=(16,))
    elif cfg == "c2":
        w = noisy_lowrank("c2", 10000, 500, 50, seed, ells=(20, 40, 60, 80, 100))
    elif cfg == "c3":
        w = image_like("c3", 60000, 3072, seed=seed, ells=(50, 100, 200))
    elif cfg == "c4":
        w = noisy_lowrank("c4", 8388608, 1024, 64, seed, ells=(128,))
    elif cfg == "c5":
        w = drift("c5", 200000, 256, seed=seed, ells=(32,))
    else:
        raise ValueError(cfg)
    if n is not None:
        w.n = n
    return w


def host_minmax(w: Workload, row0=0, nrows=None):
    nrows = w.n if nrows is None else nrows
    mn, mx = ctypes.c_double(), ctypes.c_double()
    p = w.params()
    rc = lib().fdg_host_minmax(ctypes.byref(p), row0, nrows, ctypes.byref(mn), ctypes.byref(mx))
    if rc != 0:
        raise RuntimeError("fdg_host_minmax failed")
    return mn.value, mx.value


def host_rows(w: Workload, row0: int = 0, nrows: int | None = None, nthreads: int = 0) -> np.ndarray:
    """Rows [row0, row0+nrows) of the workload as a C-contiguous fp32 array (host generator)."""
    nrows = w.n - row0 if nrows is None else nrows
    if w.kind == KIND_IMAGE and w.xminmax is None:
        raise RuntimeError("image workload needs xminmax (host_minmax over all rows, or the device one)")
    out = np.empty((nrows, w.d), dtype=np.float32)
    nthreads = nthreads or min(16, os.cpu_count() or 1)
    p = w.params()
    if nrows * w.d < 1 << 20 or nthreads == 1:
        rc = lib().fdg_host_rows(ctypes.byref(p), row0, nrows, out.ctypes.data, w.d)
        if rc != 0:
            raise RuntimeError("fdg_host_rows failed")
        return out
    import concurrent.futures as cf
    chunk = (nrows + nthreads - 1) // nthreads

    def work(t):
        a = t * chunk
        b = min(nrows, a + chunk)
        if a >= b:
            return 0
        return lib().fdg_host_rows(ctypes.byref(p), row0 + a, b - a, out.ctypes.data + a * w.d * 4, w.d)

    with cf.ThreadPoolExecutor(nthreads) as ex:
        rcs = list(ex.map(work, range(nthreads)))
    if any(rcs):
        raise RuntimeError("fdg_host_rows failed")
    return out


class DeviceGenerator:
    """Device-side generator (torch supplies memory and the stream)."""

    def __init__(self, w: Workload, device="cuda"):
        import torch
        self.w = w
        self.torch = torch
        self.device = torch.device(device)
        self.factors = torch.from_numpy(w.factors).to(self.device)
        self.e = torch.from_numpy(w.e).to(self.device) if w.e is not None else None
        if w.kind == KIND_IMAGE and w.xminmax is None:
            w.xminmax = self.minmax()

    def _params(self):
        return self.w.params(self.factors.data_ptr(), self.e.data_ptr() if self.e is not None else None)

    def minmax(self):
        torch = self.torch
        keys = torch.tensor([-1, 0], dtype=torch.int64, device=self.device)  # {~0, 0}
        p = self.w.params(self.factors.data_ptr(), None)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        rc = lib().fdg_dev_minmax(ctypes.byref(p), 0, self.w.n, keys.data_ptr(), stream)
        if rc != 0:
            raise RuntimeError("fdg_dev_minmax failed")
        k = keys.cpu().numpy().view(np.uint64)
        return lib().fdg_key_to_double(int(k[0])), lib().fdg_key_to_double(int(k[1]))

    def fill(self, out, row0: int = 0):
        """Write rows [row0, row0 + out.shape[0]) into the fp32 device tensor `out` (n x >=d)."""
        torch = self.torch
        assert out.dtype == torch.float32 and out.is_cuda and out.dim() == 2
        p = self._params()
        stream = torch.cuda.current_stream(out.device).cuda_stream
        rc = lib().fdg_dev_rows(ctypes.byref(p), row0, out.shape[0], out.data_ptr(), out.stride(0), stream)
        if rc != 0:
            raise RuntimeError("fdg_dev_rows failed")
        return out
