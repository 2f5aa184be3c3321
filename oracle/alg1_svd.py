"""Alg. 1 with a library SVD, literally as the paper runs it (TEST INFRASTRUCTURE).

Only tests/ (and the scripts under tests/golden/) may import this module.  It is
the second oracle formulation: `oracle/oracle.c` forms the buffer Gram and
diagonalises it with cyclic Jacobi (slow: ~1.3 s per 256 x 1024 ReduceRank, so
the c4 bench configuration's 64 000 ReduceRanks + 2 367 merges would take ~7 CPU
hours per variant).  Here the step "[U, S, V] <- svd(B_[i])" of Alg. 1
(PAPER.md:235 [Sec. 2.3, Alg. 1]) is numpy's LAPACK SVD, the library routine the
paper's own experiments call (PAPER.md:490 [Sec. 3]: the sketches are Matlab
programs), and "B_[i] <- S'V^T" is written out as diag(sigma') V^T.
No blocking, fusion or reordering beyond the algorithm; every rule below is the
same reading as oracle.c (C1-C10):

  iSVD         sigma'_j = sigma_j for j < ell, 0 after        (C4)
  FD           sigma'_j = sqrt(max(sigma_j^2 - delta, 0)),
               delta = sigma_ell^2
  alpha-FD     the first ell - m values unchanged, the rest
               shrunk by delta = sigma_ell^2, m = max(1, round(alpha ell))
                                                               (Alg. 2; C5)
  slot rule    R = ell - 1 rows kept after every ReduceRank    (C6)
  Fast         buffer L = 2 ell, delta = sigma_ell^2           (C1, C3)
  final        one more ReduceRank of the buffer               (C9)
  merge(X, Y)  = ReduceRank([X; Y]), L = 2 ell                 (C10)

Shares no code with the CUDA path; pinned to oracle.c (an independent
formulation: Gram + Jacobi vs a direct SVD) by tests/test_oracle_pins.py
(`test_alg1_svd_*`).
"""
from __future__ import annotations

import numpy as np

# variant -> (rule, fixed alpha or None, batched)
_VARIANTS = {
    "fd": ("fd", 1.0, False),
    "fast_fd": ("fd", 1.0, True),
    "alpha_fd": ("fd", None, False),
    "fast_alpha_fd": ("fd", None, True),
    "isvd": ("isvd", 1.0, False),
    "fast_isvd": ("isvd", 1.0, True),
}


def _m(ell, alpha):
    """m = max(1, round(alpha ell)), half away from zero (reading C5)."""
    return max(1, int(np.floor(alpha * ell + 0.5)))


def _params(ell, variant, alpha):
    rule, a0, batched = _VARIANTS[variant]
    if a0 is not None:
        alpha = a0
    elif alpha is None:
        alpha = 0.2
    L = 2 * ell if batched else ell
    m = ell if rule == "isvd" else _m(ell, alpha)
    return rule, L, m


def reduce_rank(Bf, ell, rule, m):
    """One ReduceRank of the L x d fp64 buffer Bf (Alg. 1 lines svd .. B = S'V^T).
    Returns (B' as L x d with rows R.. zero, delta, removed)."""
    L, d = Bf.shape
    R = ell - 1
    _, s, Vt = np.linalg.svd(Bf, full_matrices=False)   # s descending
    lam = np.zeros(L)
    k = min(L, s.shape[0])
    lam[:k] = s[:k] * s[:k]                               # sigma_j^2
    delta = lam[ell - 1] if ell <= L else 0.0             # delta = sigma_ell^2
    sp2 = np.zeros(L)
    for j in range(L):
        if j >= R:
            sp2[j] = 0.0                                  # sigma'_ell = 0 in every rule
        elif rule == "isvd":
            sp2[j] = lam[j]
        elif j < ell - m:
            sp2[j] = lam[j]                               # alpha-FD: unchanged head
        else:
            sp2[j] = max(lam[j] - delta, 0.0)
    removed = float(np.sum(lam - sp2))
    out = np.zeros_like(Bf)
    for j in range(min(R, k)):
        out[j] = np.sqrt(sp2[j]) * Vt[j]                  # row j of S'V^T
    return out, float(delta), removed


def sketch_stream(A, ell, variant="fd", alpha=None):
    """One stream (one shard) through Alg. 1 + the final ReduceRank (C9).
    Returns (B ell x d fp64, stats5 = [frob_sq, Delta, removed, n_shrinks, rows_seen])."""
    rule, L, m = _params(ell, variant, alpha)
    A = np.asarray(A)
    n, d = A.shape
    Bf = np.zeros((L, d))
    st = np.zeros(5)
    occ = 0
    for i in range(n):
        a = A[i].astype(np.float64)
        Bf[occ] = a                                       # insert a_i into a zero row
        st[0] += float(a @ a)
        st[4] += 1
        occ += 1
        if occ == L:                                      # no zero valued rows left
            Bf, dl, rm = reduce_rank(Bf, ell, rule, m)
            st[1] += dl; st[2] += rm; st[3] += 1
            occ = ell - 1
    Bf, dl, rm = reduce_rank(Bf, ell, rule, m)            # final ReduceRank (C9)
    st[1] += dl; st[2] += rm; st[3] += 1
    return Bf[:ell].copy(), st


def merge(X, Y, ell, variant="fd", alpha=None):
    """merge(X, Y) = ReduceRank([X; Y]) (reading C10); stats5 = [0, delta, removed, 1, 0]."""
    rule, _, m = _params(ell, variant, alpha)
    Bf = np.concatenate([np.asarray(X, np.float64), np.asarray(Y, np.float64)], axis=0)
    out, dl, rm = reduce_rank(Bf, ell, rule, m)
    return out[:ell].copy(), np.array([0.0, dl, rm, 1.0, 0.0])
