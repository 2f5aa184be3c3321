"""CPU fp64 oracle (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl
reference` leg may import this package.  It wraps oracle/liboracle.so (plain C,
see oracle/oracle.c for the paper citations of every step) and shares no code
with the CUDA path in paper_1501_06561_b200/.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

RULE_FD, RULE_ISVD, RULE_FD_T, RULE_SS, RULE_CFD = 0, 1, 2, 3, 4
# variant name -> (rule, alpha, batched)
VARIANTS = {
    "fd": (RULE_FD, 1.0, False),           # Alg. 1 + FD rule, per-row
    "fast_fd": (RULE_FD, 1.0, True),       # 2ell buffer, delta = sigma_ell^2 (C1)
    "alpha_fd": (RULE_FD, None, False),    # Alg. 2, per-row
    "fast_alpha_fd": (RULE_FD, None, True),  # Alg. 2 rule on the 2ell buffer (C3)
    "isvd": (RULE_ISVD, 1.0, False),
    "fast_isvd": (RULE_ISVD, 1.0, True),
    # paper-literal Fast alpha-FD: ell-row buffer, delta = sigma_t^2,
    # t = ell - ceil(alpha ell / 2) (C25)
    "fast_alpha_fd_paper": (RULE_FD_T, None, "literal"),
    # SpaceSaving Directions: Alg. 1 with ReduceRank-SS (Alg. 3), per-row
    "ssd": (RULE_SS, 1.0, False),
    # Compensative FD: FD, final sigma_hat = sqrt(sigma'^2 + Delta), per-row
    "cfd": (RULE_CFD, 1.0, False),
}

_dp = ctypes.POINTER(ctypes.c_double)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `python build.py oracle`")
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_jacobi_eig.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_jacobi_eig.restype = ctypes.c_int
        L.oracle_reduce_rank.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.oracle_reduce_rank.restype = ctypes.c_int
        L.oracle_reduce_rank_t.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                           ctypes.c_double, ctypes.c_void_p]
        L.oracle_reduce_rank_t.restype = ctypes.c_int
        L.oracle_sketch.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_sketch.restype = ctypes.c_int
        L.oracle_merge.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_merge.restype = ctypes.c_int
        L.oracle_gram.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_void_p, _dp]
        L.oracle_gram.restype = ctypes.c_int
        L.oracle_sym_extremes.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.oracle_sym_extremes.restype = ctypes.c_int
        L.oracle_lanczos_extremes.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, _dp, _dp]
        L.oracle_lanczos_extremes.restype = ctypes.c_int
        L.oracle_cov_err.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p]
        L.oracle_cov_err.restype = ctypes.c_int
        L.oracle_proj_err.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_void_p]
        L.oracle_proj_err.restype = ctypes.c_int
        _lib = L
    return _lib


def _nthreads(nthreads):
    return nthreads or (os.cpu_count() or 1)


def alpha_m(ell: int, alpha: float) -> int:
    """m = max(1, round(alpha*ell)) (reading C5; C llround = half away from zero)."""
    x = alpha * ell
    m = int(np.floor(x + 0.5))
    return max(1, m)


def jacobi_eig(M):
    """(w, V) of symmetric M by the oracle's cyclic Jacobi (unsorted)."""
    A = np.array(M, dtype=np.float64, order="C", copy=True)
    n = A.shape[0]
    w = np.empty(n)
    V = np.empty((n, n))
    sweeps = lib().oracle_jacobi_eig(A.ctypes.data, n, w.ctypes.data, V.ctypes.data)
    if sweeps < 0:
        raise RuntimeError("oracle Jacobi did not converge")
    return w, V


def reduce_rank(Bf, ell, rule=RULE_FD, alpha=1.0):
    """Apply one ReduceRank to the L x d buffer Bf; returns (B', delta, removed)."""
    B = np.array(Bf, dtype=np.float64, order="C", copy=True)
    L, d = B.shape
    m = ell if rule == RULE_ISVD else alpha_m(ell, alpha)
    st = np.zeros(3)
    rc = lib().oracle_reduce_rank(B.ctypes.data, L, d, ell, rule, m, st.ctypes.data)
    if rc:
        raise RuntimeError(f"oracle_reduce_rank rc={rc}")
    return B, st[0], st[1]


def reduce_rank_t(Bf, ell, alpha):
    """One paper-literal Fast alpha-FD ReduceRank of the L x d buffer Bf."""
    B = np.array(Bf, dtype=np.float64, order="C", copy=True)
    L, d = B.shape
    st = np.zeros(3)
    rc = lib().oracle_reduce_rank_t(B.ctypes.data, L, d, ell, float(alpha), st.ctypes.data)
    if rc:
        raise RuntimeError(f"oracle_reduce_rank_t rc={rc}")
    return B, st[0], st[1]


class SketchResult:
    def __init__(self, B, stats, shards=None):
        self.B = B
        self.frob_sq, self.delta_total, self.removed, self.n_shrinks, self.rows_seen = stats
        self.n_shrinks = int(self.n_shrinks)
        self.rows_seen = int(self.rows_seen)
        self.shards = shards


def sketch(A, ell, variant="fd", alpha=None, n_shards=1, appends=None, nthreads=0, want_shards=False):
    """Oracle sketch of A (n x d fp32) — Alg. 1 with the variant's rule (see VARIANTS)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    n, d = A.shape
    rule, a0, batched = VARIANTS[variant]
    if a0 is not None:          # FD / Fast FD / iSVD: alpha is fixed (1), any argument ignored
        alpha = a0
    elif alpha is None:
        alpha = 0.2
    L = 2 * ell if batched is True else ell
    B = np.zeros((ell, d))
    shards = np.zeros((n_shards, ell, d)) if want_shards else None
    st = np.zeros(5)
    app = None
    napp = 0
    if appends is not None:
        app = np.ascontiguousarray(appends, dtype=np.int64)
        assert app.sum() == n
        napp = len(app)
    rc = lib().oracle_sketch(A.ctypes.data, n, d, d, ell, rule, float(alpha), L, n_shards,
                             app.ctypes.data if app is not None else None, napp, _nthreads(nthreads),
                             B.ctypes.data, shards.ctypes.data if shards is not None else None, st.ctypes.data)
    if rc:
        raise RuntimeError(f"oracle_sketch rc={rc}")
    return SketchResult(B, st, shards)


def merge(sketches, ell, variant="fd", alpha=None):
    S = np.ascontiguousarray(sketches, dtype=np.float64)
    count, l2, d = S.shape
    assert l2 == ell
    rule, a0, _ = VARIANTS[variant]
    if a0 is not None:
        alpha = a0
    elif alpha is None:
        alpha = 0.2
    m = ell if rule == RULE_ISVD else alpha_m(ell, alpha)
    B = np.zeros((ell, d))
    st = np.zeros(5)
    rc = lib().oracle_merge(S.ctypes.data, count, d, ell, rule, m, float(alpha), B.ctypes.data, st.ctypes.data)
    if rc:
        raise RuntimeError(f"oracle_merge rc={rc}")
    return B, st


def gram(A, nthreads=0):
    A = np.ascontiguousarray(A, dtype=np.float32)
    n, d = A.shape
    out = np.empty((d, d))
    f = ctypes.c_double()
    lib().oracle_gram(A.ctypes.data, n, d, d, _nthreads(nthreads), out.ctypes.data, ctypes.byref(f))
    return out, f.value


def sym_extremes(M, jacobi_max=1024, kmax=512):
    M = np.ascontiguousarray(M, dtype=np.float64)
    hi, lo = ctypes.c_double(), ctypes.c_double()
    rc = lib().oracle_sym_extremes(M.ctypes.data, M.shape[0], jacobi_max, kmax, ctypes.byref(hi), ctypes.byref(lo))
    if rc:
        raise RuntimeError("oracle_sym_extremes failed")
    return hi.value, lo.value


def lanczos_extremes(M, kmax=512):
    M = np.ascontiguousarray(M, dtype=np.float64)
    hi, lo = ctypes.c_double(), ctypes.c_double()
    rc = lib().oracle_lanczos_extremes(M.ctypes.data, M.shape[0], kmax, ctypes.byref(hi), ctypes.byref(lo))
    if rc:
        raise RuntimeError("oracle_lanczos_extremes failed")
    return hi.value, lo.value


def cov_err(A, B, nthreads=0, jacobi_max=512, kmax=512):
    """cov-err = ||A^T A - B^T B||_2 / ||A||_F^2.

    Returns dict(err, lmax, lmin, frob) where lmax/lmin are the extreme
    eigenvalues of A^T A - B^T B divided by ||A||_F^2."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float64)
    n, d = A.shape
    out = np.zeros(4)
    rc = lib().oracle_cov_err(A.ctypes.data, n, d, d, B.ctypes.data, B.shape[0], _nthreads(nthreads),
                              jacobi_max, kmax, out.ctypes.data)
    if rc == -4:
        raise ValueError("||A||_F^2 = 0: cov-err undefined (SPEC.md:119)")
    if rc:
        raise RuntimeError(f"oracle_cov_err rc={rc}")
    return dict(err=out[0], lmax=out[1], lmin=out[2], frob=out[3])


def proj_err(A, B, k=10, nthreads=0, jacobi_max=512, kmax=512):
    """proj-err (k = 10 per PAPER.md:572) =
    ||A - pi_{B_k}(A)||_F^2 / ||A - A_k||_F^2, B_k = top-k right singular subspace of B.

    Returns dict(err, num, den, frob): num = ||A - pi_{B_k}(A)||_F^2, den = ||A - A_k||_F^2."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float64)
    n, d = A.shape
    if B.ndim != 2 or B.shape[1] != d:
        raise ValueError("B must be ell x d")
    out = np.zeros(4)
    rc = lib().oracle_proj_err(A.ctypes.data, n, d, d, B.ctypes.data, B.shape[0], int(k), _nthreads(nthreads),
                               jacobi_max, kmax, out.ctypes.data)
    if rc == -4:
        raise ValueError("||A||_F^2 = 0: proj-err undefined")
    if rc == -5:
        raise ValueError("||A - A_k||_F^2 = 0 (rank A <= k): proj-err undefined")
    if rc:
        raise RuntimeError(f"oracle_proj_err rc={rc}")
    return dict(err=out[0], num=out[1], den=out[2], frob=out[3])


def fd_t_indices(ell, alpha):
    """(t, R) of the paper-literal Fast alpha-FD (C25):
    delta = lambda_t (1-based), rows 0..R-1 kept.  Mirrors oracle.c fd_t_indices."""
    import math
    h = max(1, math.ceil(alpha * ell / 2.0 - 1e-9))
    m = alpha_m(ell, alpha)
    t = ell - h
    return t, max(ell - m, t - 1)


def hash_sketch(A, ell, s=4, seed=0, row0=0, B=None):
    """Hashing (s = 1) / OSNAP (s stacked blocks) sketch: B += S A with
    S = s count-sketch blocks of ell/s rows, entries +-1/sqrt(s) (C28)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    n, d = A.shape
    out = np.zeros((ell, d)) if B is None else B
    assert out.shape == (ell, d) and out.dtype == np.float64 and out.flags.c_contiguous
    L = lib()
    if not getattr(L, "_hash_typed", False):
        L.oracle_hash_sketch.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
        L.oracle_hash_sketch.restype = ctypes.c_int
        L._hash_typed = True
    rc = L.oracle_hash_sketch(A.ctypes.data, n, d, d, int(ell), int(s), int(seed), int(row0), out.ctypes.data)
    if rc:
        raise ValueError("hash_sketch: need 1 <= s <= ell and s | ell")
    return out
