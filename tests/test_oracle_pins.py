"""Pins for the CPU oracle against what the paper and the mathematics fix.

Every test here runs without a GPU.  None of them re-types the oracle's own
formula: each compares it with a hand-derived value (SPEC/paper), a closed
form, an invariant the paper proves, or an independent implementation
(numpy LAPACK eigh; a covariance-form FD written in numpy below).
"""
import os

import numpy as np
import pytest

import fdgen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _read_golden_rules():
    rows = []
    with open(os.path.join(HERE, "golden", "spec_reduce_rank_examples.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            head, sin, sout, delta = [x.strip() for x in line.split("|")]
            rule, alpha, ell = head.split()
            rows.append((rule, float(alpha), int(ell), [float(x) for x in sin.split()],
                         [float(x) for x in sout.split()], float(delta)))
    return rows


@pytest.mark.parametrize("case", _read_golden_rules())
def test_reduce_rank_hand_examples(case):
    """SPEC.md hand examples of the FD / alpha-FD / iSVD rules (PAPER.md:248, 254,
    319-325), the paper-literal Fast alpha-FD and ReduceRank-SS
    (PAPER.md:405-411), values re-derived by hand in tests/golden."""
    rule, alpha, ell, s_in, s_out, delta = case
    L = len(s_in)
    d = L + 1
    # rows of a random rotation scaled by the singular values -> svd(Bf) = those values
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    Bf = np.diag(s_in) @ Q[:L]
    if rule == "fastpfd":
        B, dl, removed = oracle.reduce_rank_t(Bf, ell, alpha)
    else:
        r = {"isvd": oracle.RULE_ISVD, "ss": oracle.RULE_SS}.get(rule, oracle.RULE_FD)
        B, dl, removed = oracle.reduce_rank(Bf, ell, r, alpha)
    sv = np.linalg.svd(B, compute_uv=False)
    expect = np.zeros(len(sv))
    expect[: len(s_out)] = s_out
    # compare sigma'^2 (sigma' = sqrt(sigma^2 - delta) turns eps-level ties into sqrt(eps))
    np.testing.assert_allclose(sv[: len(expect)] ** 2, expect ** 2, atol=1e-12 * max(1.0, max(s_in) ** 2))
    assert abs(dl - delta) < 1e-12 * max(1.0, max(s_in) ** 2)
    # ledger of this single step: removed mass = ||Bf||^2 - ||B'||^2
    assert abs(removed - (np.sum(np.square(s_in)) - np.sum(np.square(s_out)))) < 1e-10
    # retained rows are in the span of the input rows and mutually orthogonal
    G = B @ B.T
    assert np.allclose(G - np.diag(np.diag(G)), 0, atol=1e-12)


def test_stream_spec_example():
    """ell=2 FD, rows 2e1 then e2 -> spectrum (sqrt3, 0), Delta = 1 (plus final RR, lossless)."""
    A = np.array([[2, 0], [0, 1]], np.float32)
    r = oracle.sketch(A, 2, "fd")
    np.testing.assert_allclose(np.linalg.svd(r.B, compute_uv=False), [np.sqrt(3), 0], atol=1e-12)
    assert abs(r.delta_total - 1.0) < 1e-12
    assert r.n_shrinks == 2


def test_zero_stream():
    """all-zero rows -> B = 0, Delta = 0."""
    A = np.zeros((50, 7), np.float32)
    for v in oracle.VARIANTS:
        r = oracle.sketch(A, 4, v)
        assert np.all(r.B == 0) and r.delta_total == 0 and r.removed == 0


def test_jacobi_2x2_closed_form():
    a, b, c = 3.0, 1.25, -2.0
    w, V = oracle.jacobi_eig([[a, b], [b, c]])
    tr, det = a + c, a * c - b * b
    disc = np.sqrt(tr * tr / 4 - det)
    np.testing.assert_allclose(sorted(w), [tr / 2 - disc, tr / 2 + disc], rtol=1e-15)
    M = np.array([[a, b], [b, c]])
    np.testing.assert_allclose(M @ V, V * w[None, :], atol=1e-14)


@pytest.mark.parametrize("n", [5, 37, 128])
def test_jacobi_vs_lapack(n):
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, n))
    M = X + X.T
    w, V = oracle.jacobi_eig(M)
    np.testing.assert_allclose(np.sort(w), np.linalg.eigvalsh(M), atol=1e-11 * np.abs(M).max() * n)
    np.testing.assert_allclose(V.T @ V, np.eye(n), atol=1e-13 * n)
    np.testing.assert_allclose(M @ V, V * w[None, :], atol=1e-11 * n)


def test_lanczos_vs_jacobi():
    rng = np.random.default_rng(3)
    for d in (50, 200):
        X = rng.standard_normal((d + 20, d))
        M = X.T @ X - 0.5 * np.diag(rng.random(d))
        ev = np.linalg.eigvalsh(M)
        hi, lo = oracle.lanczos_extremes(M, kmax=d)
        assert abs(hi - ev[-1]) < 1e-9 * abs(ev[-1]) and abs(lo - ev[0]) < 1e-8 * abs(ev[-1])
        hj, lj = oracle.sym_extremes(M, jacobi_max=1024)
        assert abs(hj - ev[-1]) < 1e-10 * abs(ev[-1]) and abs(lj - ev[0]) < 1e-9 * abs(ev[-1])


# ---------------------------------------------------------------------------
# Independent covariance-form implementation (numpy, test-only).
# A ReduceRank maps the buffer covariance C = Bf^T Bf to V f(Lambda) V^T over the
# eigenpairs of C (d x d), which share their nonzero spectrum with the Gram form
# the oracle uses; slot counting is the same (occ -> ell-1 after each shrink).
# ---------------------------------------------------------------------------
def _cov_reduce(C, L, ell, rule, m, t=None, R=None):
    # t: delta = lambda_t (1-based); R: rows kept.  Every rule but the paper-literal
    # Fast alpha-FD has t = ell, R = ell - 1.
    t = ell if t is None else t
    R = ell - 1 if R is None else R
    d = C.shape[0]
    mu, V = np.linalg.eigh(C)
    mu, V = mu[::-1], V[:, ::-1]
    lam = np.zeros(max(L, d))
    lam[: min(d, L)] = np.maximum(mu[: min(d, L)], 0)
    delta = lam[t - 1] if t <= L else 0.0
    sp2 = np.zeros_like(lam)
    for j in range(R):
        if rule == "isvd" or j < ell - m:
            sp2[j] = lam[j]
        else:
            sp2[j] = max(lam[j] - delta, 0.0)
    k = min(d, R)
    Cn = (V[:, :k] * sp2[:k][None, :]) @ V[:, :k].T
    return Cn, delta, float(np.sum(lam[:L] - sp2[:L]))


def _cov_sketch(A, ell, rule, m, L, t=None, R=None):
    d = A.shape[1]
    C = np.zeros((d, d))
    occ = 0
    Delta = 0.0
    for a in A.astype(np.float64):
        C += np.outer(a, a)
        occ += 1
        if occ == L:
            C, dl, _ = _cov_reduce(C, L, ell, rule, m, t, R)
            Delta += dl
            occ = ell - 1 if R is None else R
    C, dl, _ = _cov_reduce(C, L, ell, rule, m, t, R)
    return C, Delta + dl


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("variant", ["fd", "fast_fd", "alpha_fd", "fast_alpha_fd", "isvd", "fast_isvd",
                                     "fast_alpha_fd_paper"])
def test_bruteforce_covariance_form(seed, variant):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 13))
    d = int(rng.integers(1, 7))
    ell = int(rng.integers(2, 5))
    A = rng.standard_normal((n, d)).astype(np.float32) * rng.uniform(0.5, 2.0, size=(n, 1)).astype(np.float32)
    rule, a0, batched = oracle.VARIANTS[variant]
    alpha = 0.5 if a0 is None else a0
    m = ell if rule == oracle.RULE_ISVD else oracle.alpha_m(ell, alpha)
    L = 2 * ell if batched is True else ell
    t, R = oracle.fd_t_indices(ell, alpha) if rule == oracle.RULE_FD_T else (None, None)
    r = oracle.sketch(A, ell, variant, alpha=alpha)
    C, Delta = _cov_sketch(A, ell, "isvd" if rule == oracle.RULE_ISVD else "fd", m, L, t, R)
    np.testing.assert_allclose(r.B.T @ r.B, C, atol=1e-10 * max(1.0, np.abs(C).max()))
    assert abs(r.delta_total - Delta) < 1e-10 * max(1.0, Delta)


def _c1():
    w = fdgen.config("c1")
    return fdgen.host_rows(w)


# the FD family (SSD and CFD have their own bounds, Theorem SS / PAPER.md:436, below)
FD_FAMILY = [v for v in oracle.VARIANTS if v not in ("ssd", "cfd")]


@pytest.mark.parametrize("variant", FD_FAMILY)
def test_properties_lemma1_lemma3(variant):
    """Props 1-2 via Lemma 1: 0 <= ||Ax||^2-||Bx||^2 <= Delta;
    Lemma 3: ||A||_F^2 - ||B||_F^2 = removed, = ell*Delta (FD per-row),
    m*Delta (alpha-FD per-row), Delta (iSVD per-row, one sigma^2 per step), >= m*Delta batched."""
    A = _c1()
    ell = 16
    rule, a0, batched = oracle.VARIANTS[variant]
    alpha = 0.2 if a0 is None else a0
    r = oracle.sketch(A, ell, variant, alpha=alpha)
    AtA, frob = oracle.gram(A)
    M = AtA - r.B.T @ r.B
    ev = np.linalg.eigvalsh(M)
    assert ev[0] >= -1e-10 * frob
    assert ev[-1] <= r.delta_total * (1 + 1e-10)
    bF = float(np.sum(r.B ** 2))
    assert abs((frob - bF) - r.removed) <= 1e-10 * frob
    m = ell if rule == oracle.RULE_ISVD else oracle.alpha_m(ell, alpha)
    if rule == oracle.RULE_ISVD:
        if not batched:
            assert abs(r.removed - r.delta_total) <= 1e-9 * frob
    elif rule == oracle.RULE_FD_T:
        # paper-literal Fast alpha-FD: rows ell-m+1..t lose exactly delta each
        t, _ = oracle.fd_t_indices(ell, alpha)
        assert r.removed >= (t - ell + m) * r.delta_total * (1 - 1e-12)
    elif not batched:
        assert abs(r.removed - m * r.delta_total) <= 1e-9 * frob
    else:
        assert r.removed >= m * r.delta_total * (1 - 1e-12)


@pytest.mark.parametrize("variant", ["fd", "fast_fd", "alpha_fd", "fast_alpha_fd"])
def test_error_bounds(variant):
    """Lemma / Theorem (k < alpha*ell reading C19):
    cov-err <= ||A - A_k||_F^2 / ((m - k) ||A||_F^2) for all integers 0 <= k < m."""
    A = _c1()
    ell = 16
    rule, a0, _ = oracle.VARIANTS[variant]
    alpha = 0.2 if a0 is None else a0
    m = oracle.alpha_m(ell, alpha)
    r = oracle.sketch(A, ell, variant, alpha=alpha)
    e = oracle.cov_err(A, r.B)
    s2 = np.linalg.svd(A.astype(np.float64), compute_uv=False) ** 2
    for k in range(m):
        tail = s2[k:].sum()
        assert e["err"] <= tail / ((m - k) * e["frob"]) * (1 + 1e-9)
    assert e["err"] <= 1.0 / m + 1e-12


@pytest.mark.parametrize("variant", list(oracle.VARIANTS))
def test_exact_when_rank_below_ell(variant):
    """rank(A) <= ell-1 (or n <= ell-1) => B^T B = A^T A (reading C2: ell-1, not ell)."""
    rng = np.random.default_rng(7)
    ell, d = 6, 20
    A = (rng.standard_normal((300, ell - 1)) @ rng.standard_normal((ell - 1, d))).astype(np.float32)
    r = oracle.sketch(A, ell, variant)
    AtA, frob = oracle.gram(A)
    assert np.abs(AtA - r.B.T @ r.B).max() <= 1e-10 * frob
    A2 = rng.standard_normal((ell - 1, d)).astype(np.float32)
    r2 = oracle.sketch(A2, ell, variant)
    AtA2, f2 = oracle.gram(A2)
    assert np.abs(AtA2 - r2.B.T @ r2.B).max() <= 1e-12 * f2


def test_rank_ell_only_bounded():
    """With rank(A) = ell the FD sketch is NOT exact in general (off-by-one of reading C2)."""
    rng = np.random.default_rng(8)
    ell, d = 6, 20
    A = (rng.standard_normal((300, ell)) @ rng.standard_normal((ell, d))).astype(np.float32)
    r = oracle.sketch(A, ell, "fd")
    e = oracle.cov_err(A, r.B)
    assert e["err"] > 1e-6


def test_cov_err_closed_forms():
    """cov-err: B=A -> 0; A=I2, B=0 -> 0.5;
    B=0 -> sigma_1^2/||A||_F^2 = 1/numeric-rank."""
    A = np.eye(2, dtype=np.float32)
    assert abs(oracle.cov_err(A, np.zeros((1, 2)))["err"] - 0.5) < 1e-15
    rng = np.random.default_rng(1)
    A = rng.standard_normal((40, 9)).astype(np.float32)
    assert oracle.cov_err(A, A.astype(np.float64))["err"] < 1e-13
    s = np.linalg.svd(A.astype(np.float64), compute_uv=False)
    e = oracle.cov_err(A, np.zeros((3, 9)))
    assert abs(e["err"] - s[0] ** 2 / np.sum(s ** 2)) < 1e-13
    with pytest.raises(ValueError):
        oracle.cov_err(np.zeros((3, 4), np.float32), np.zeros((2, 4)))


def test_cov_err_lanczos_path_matches_jacobi_path():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((400, 80)).astype(np.float32)
    B = rng.standard_normal((10, 80)) * 3
    e1 = oracle.cov_err(A, B, jacobi_max=1024)
    e2 = oracle.cov_err(A, B, jacobi_max=10, kmax=80)
    assert abs(e1["err"] - e2["err"]) < 1e-10 * e1["err"]


@pytest.mark.parametrize("variant", ["fd", "fast_alpha_fd", "isvd"])
def test_merge_symmetry_and_tree(variant):
    """B^T B of merge(X, Y) depends only on X^T X + Y^T Y (reading C10)."""
    A = _c1()
    r = oracle.sketch(A, 16, variant, n_shards=4, want_shards=True)
    X, Y = r.shards[0], r.shards[1]
    B1, _ = oracle.merge(np.stack([X, Y]), 16, variant)
    B2, _ = oracle.merge(np.stack([Y, X]), 16, variant)
    assert np.abs(B1.T @ B1 - B2.T @ B2).max() < 1e-10 * r.frob_sq
    # the P-shard sketch = recursive-halving tree over its shard sketches
    B, _ = oracle.merge(r.shards, 16, variant)
    assert np.abs(B.T @ B - r.B.T @ r.B).max() < 1e-12 * r.frob_sq
    # each shard sketch = the sketch of that shard's contiguous rows
    sizes = [500, 500, 500, 500]
    r0 = oracle.sketch(A[:500], 16, variant)
    assert np.abs(r0.B.T @ r0.B - r.shards[0].T @ r.shards[0]).max() < 1e-12 * r.frob_sq
    # merged sketch still satisfies Props 1-2 with the summed Delta
    AtA, frob = oracle.gram(A)
    ev = np.linalg.eigvalsh(AtA - r.B.T @ r.B)
    assert ev[0] > -1e-10 * frob and ev[-1] <= r.delta_total * (1 + 1e-10)
    assert abs(frob - np.sum(r.B ** 2) - r.removed) < 1e-10 * frob
    del sizes


def test_appends_split_per_call():
    """Each append call's rows are split into P contiguous ranges (C10)."""
    A = _c1()
    r = oracle.sketch(A, 16, "fast_fd", n_shards=2, appends=[1200, 800], want_shards=True)
    part0 = np.concatenate([A[:600], A[1200:1600]])
    r0 = oracle.sketch(part0, 16, "fast_fd")
    assert np.abs(r0.B - r.shards[0]).max() == 0.0


def test_table1_numeric_rank():
    """Table 1: Random Noisy numeric rank 14.93 with m=30 and D_ii=1-(i-1)/m."""
    g = {}
    with open(os.path.join(HERE, "golden", "table1_random_noisy.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                k, v = line.split()
                g[k] = float(v)
    w = fdgen.noisy_lowrank("t1", int(g["n"]), int(g["d"]), int(g["m"]), seed=0, zeta=g["zeta"])
    A = fdgen.host_rows(w).astype(np.float64)
    s = np.linalg.svd(A, compute_uv=False)
    nr = np.sum(s ** 2) / s[0] ** 2
    assert g["lo"] <= nr <= g["hi"], nr


def test_generator_expected_frobenius():
    """E||A||_F^2 = n (sum_i D_ii^2 + d / zeta^2) (SPEC.md:441 for the PAPER.md:539-541 construction)."""
    w = fdgen.config("c2")
    A = fdgen.host_rows(w).astype(np.float64)
    D = 1 - np.arange(50) / 50
    expect = w.n * (np.sum(D ** 2) + w.d / 100.0)
    assert abs(np.sum(A ** 2) / expect - 1) < 0.02


def test_generator_deterministic_and_rowwise():
    w = fdgen.config("c1")
    A = fdgen.host_rows(w)
    B = fdgen.host_rows(w, 700, 300)
    assert np.array_equal(A[700:1000], B)
    w5 = fdgen.config("c5", n=20000)
    w5.extra["block_rows"] = 10000
    C = fdgen.host_rows(w5, 0, 200)
    e = C[99].astype(np.float64)
    assert abs(np.linalg.norm(e) - 3.0) < 1e-6 and np.array_equal(C[99], C[199])


def test_paper_qualitative_order_c2():
    """PAPER.md:649-652 (qualitative, smoke only — parity unpinned for printed errors):
    on Random Noisy, FD is the worst and iSVD / 0.2-FD the best at small ell."""
    w = fdgen.config("c2")
    A = fdgen.host_rows(w)
    errs = {}
    for v in ("fd", "alpha_fd", "isvd"):
        r = oracle.sketch(A, 20, v)
        errs[v] = oracle.cov_err(A, r.B)["err"]
    assert errs["fd"] > errs["alpha_fd"] and errs["fd"] > errs["isvd"]
    assert errs["fd"] <= 1 / 20


# ---------------------------------------------------------------------------
# proj-err (k = 10)
# ---------------------------------------------------------------------------
def _orth(rng, n):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def test_proj_err_closed_form_rotated():
    """A = U diag(s) V^T, B = rows t_i v_i^T for i in S1 (large t) and S2 (small t):
    B_k = span{v_i : i in S1}, so ||A - pi_{B_k}(A)||_F^2 = sum_{i not in S1} s_i^2 and
    ||A - A_k||_F^2 = sum_{i >= k} s_i^2 (s sorted descending).  A transposed operand,
    left instead of right singular vectors, or a wrong top-k order all fail this."""
    rng = np.random.default_rng(7)
    d, k = 24, 4
    s = np.sort(rng.uniform(1.0, 10.0, d))[::-1]
    U, V = _orth(rng, d), _orth(rng, d)
    A = (U * s) @ V.T
    S1 = [1, 5, 9, 20]                    # not the top-k of A
    S2 = [0, 3, 7]                        # in B but with smaller weights
    rows = [30.0 * (j + 1) * V[:, i] for j, i in enumerate(S1)] + [0.5 * V[:, i] for i in S2]
    B = np.array(rows[::-1])              # row order must not matter
    Af = A.astype(np.float32)
    s32 = np.linalg.svd(Af.astype(np.float64), compute_uv=False)
    r = oracle.proj_err(Af, B, k=k)
    Vf = V[:, S1]
    num = float(np.sum(Af.astype(np.float64) ** 2)) - float(np.sum((Af.astype(np.float64) @ Vf) ** 2))
    den = float(np.sum(s32[k:] ** 2))
    assert abs(r["num"] - num) < 1e-9 * r["frob"]
    assert abs(r["den"] - den) < 1e-9 * r["frob"]
    expect = float(np.sum(np.delete(s, S1) ** 2) / np.sum(s[k:] ** 2))
    assert abs(r["err"] - expect) < 1e-5 * expect


def test_proj_err_of_A_itself_is_one_and_random_B_at_least_one():
    """B = A: B_k = A_k's subspace -> proj-err = 1; any B -> proj-err >= 1 (A_k optimal)."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((60, 20)).astype(np.float32)
    r = oracle.proj_err(A, A.astype(np.float64), k=5)
    assert abs(r["err"] - 1.0) < 1e-10
    for seed in range(3):
        B = np.random.default_rng(seed).standard_normal((8, 20))
        assert oracle.proj_err(A, B, k=5)["err"] >= 1.0 - 1e-12


def test_proj_err_fd_bound_and_lanczos_path():
    """FD sketch of c1: 1 <= proj-err <= ell/(ell - k) (Theorem of
    PAPER.md:374-377 at alpha = 1); the Lanczos top-k path agrees with full Jacobi."""
    A = _c1()
    ell, k = 16, 10
    r = oracle.sketch(A, ell, "fd")
    p = oracle.proj_err(A, r.B, k=k)
    assert 1.0 - 1e-12 <= p["err"] <= ell / (ell - k)
    p2 = oracle.proj_err(A, r.B, k=k, jacobi_max=0, kmax=64)
    assert abs(p2["err"] - p["err"]) < 1e-9 * p["err"]


def test_proj_err_undefined_cases():
    with pytest.raises(ValueError):
        oracle.proj_err(np.zeros((3, 4), np.float32), np.zeros((2, 4)), k=1)
    A = np.zeros((5, 6), np.float32); A[0, 0] = 1.0; A[1, 2] = 2.0      # rank 2 <= k
    with pytest.raises(ValueError):
        oracle.proj_err(A, np.ones((2, 6)), k=2)


# ---------------------------------------------------------------------------
# paper-literal Fast alpha-FD
# ---------------------------------------------------------------------------
def test_fd_t_indices_reading():
    """t = ell - ceil(alpha ell / 2), R = max(ell - m, t - 1) (C25)."""
    assert oracle.fd_t_indices(128, 0.2) == (115, 114)     # alpha ell / 2 = 12.8 -> 13
    assert oracle.fd_t_indices(20, 0.2) == (18, 17)        # 2.0 exactly -> 2
    assert oracle.fd_t_indices(20, 1.0) == (10, 9)         # Fast FD with an ell-row buffer
    assert oracle.fd_t_indices(50, 0.02) == (49, 49)       # m = 1: only sigma_ell shrinks


def test_cfd_spec_hand_example():
    """Compensative FD's final step (sigma_hat_j = sqrt(sigma'_j^2 + Delta)),
    by hand: ell = 2, rows 2e1, e2, e2 (d = 2).  The lazy ReduceRank of [2e1; e2] (spectrum (2, 1))
    shrinks by delta = 1 -> (sqrt3, 0); e2 takes the free slot; the final step on [sqrt3 e1; e2]
    (spectrum (sqrt3, 1)) shrinks by delta = 1 -> sigma' = (sqrt2, 0) and compensates with
    Delta = 1 + 1 = 2 -> sigma_hat = (sqrt(2 + 2), sqrt(0 + 2)) = (2, sqrt2); the mass
    ||A||_F^2 = 6 = 4 + 2 is preserved."""
    A = np.array([[2, 0], [0, 1], [0, 1]], np.float32)
    r = oracle.sketch(A, 2, "cfd")
    sv = np.linalg.svd(r.B, compute_uv=False)
    np.testing.assert_allclose(sv, [2.0, np.sqrt(2.0)], atol=1e-12)
    assert abs(r.delta_total - 2.0) < 1e-12
    assert r.n_shrinks == 2


def test_fast_alpha_fd_paper_alpha1_is_fast_fd():
    """alpha = 1 with 2 ell' rows is Fast FD with ell' (delta = lambda_ell' of a 2 ell'
    buffer, ell' - 1 rows kept): the same sketch, bit for bit, at P = 1 and P = 3."""
    A = _c1()
    for P in (1, 3):
        r1 = oracle.sketch(A, 8, "fast_fd", n_shards=P)
        r2 = oracle.sketch(A, 16, "fast_alpha_fd_paper", alpha=1.0, n_shards=P)
        assert np.array_equal(r2.B[:8], r1.B) and not np.any(r2.B[8:])
        assert r2.delta_total == r1.delta_total


def test_fast_alpha_fd_paper_bounds():
    """Fast alpha-FD with ell rows meets alpha-FD's bounds at half the
    rows: 0 <= ||Ax||^2 - ||Bx||^2 <= ||A - A_k||_F^2 / (alpha ell / 2 - k) for
    k < alpha ell / 2; the Frobenius ledger ||A||^2 - ||B||^2 = removed >= (t - ell + m) Delta."""
    A = _c1().astype(np.float64)
    n, d = A.shape
    sv = np.linalg.svd(A, compute_uv=False)
    for ell, alpha in ((16, 1.0), (40, 0.5), (60, 0.4)):
        r = oracle.sketch(A.astype(np.float32), ell, "fast_alpha_fd_paper", alpha=alpha)
        M = A.T @ A - r.B.T @ r.B
        w = np.linalg.eigvalsh((M + M.T) / 2)
        assert w[0] >= -1e-9 * sv[0] ** 2
        half = alpha * ell / 2
        for k in range(0, int(np.ceil(half))):
            if k < half:
                assert w[-1] <= np.sum(sv[k:] ** 2) / (half - k) * (1 + 1e-9)
        t, R = oracle.fd_t_indices(ell, alpha)
        m = oracle.alpha_m(ell, alpha)
        frob_a, frob_b = np.sum(A ** 2), np.sum(r.B ** 2)
        assert abs((frob_a - frob_b) - r.removed) < 1e-8 * frob_a
        assert (frob_a - frob_b) >= (t - ell + m) * r.delta_total * (1 - 1e-9)


# ---------------------------------------------------------------------------
# SpaceSaving Directions and Compensative FD
# ---------------------------------------------------------------------------
def test_ss_rule_closed_form():
    """ReduceRank-SS (Alg. 3) on a buffer with known singular values
    s_j e_{pi(j)}: delta = s_{ell-1}^2; the result has s_1..s_{ell-2}, 0 and
    sqrt(s_ell^2 + delta) along e_{pi(ell)}; the squared mass is unchanged."""
    ell, d = 9, 23
    rng = np.random.default_rng(21)
    s = np.sort(rng.uniform(1.0, 5.0, ell))[::-1]
    perm = rng.permutation(d)[:ell]
    Bf = np.zeros((ell, d))
    for j in range(ell):
        Bf[j, perm[j]] = s[j]
    Bf = Bf[rng.permutation(ell)]
    B, delta, removed = oracle.reduce_rank(Bf, ell, rule=oracle.RULE_SS)
    assert abs(delta - s[ell - 2] ** 2) < 1e-12 * s[0] ** 2
    assert abs(removed) < 1e-10 * s[0] ** 2
    col = np.sum(B ** 2, axis=0)                      # mass per original axis
    expect = np.zeros(d)
    expect[perm[: ell - 2]] = s[: ell - 2] ** 2
    expect[perm[ell - 1]] = s[ell - 1] ** 2 + s[ell - 2] ** 2
    np.testing.assert_allclose(col, expect, atol=1e-10 * s[0] ** 2)
    assert np.all(B[ell - 1] == 0.0)                   # the free slot


def test_ssd_theorem_ss_bounds():
    """Theorem SS: ||A||_F^2 = ||B||_F^2;
    | ||Ax||^2 - ||Bx||^2 | <= ||A - A_k||_F^2 / (ell/2 - 1/2 - k) for k < ell/2 - 1/2;
    ||A - pi_B^k(A)||_F^2 <= ||A - A_k||_F^2 (ell - 1) / (ell - 1 - 2k) for k < ell/2 - 1."""
    A = _c1()
    A64 = A.astype(np.float64)
    sv2 = np.linalg.svd(A64, compute_uv=False) ** 2
    for ell in (12, 16, 24):
        r = oracle.sketch(A, ell, "ssd")
        fa = float(np.sum(A64 ** 2))
        assert abs(float(np.sum(r.B ** 2)) - fa) <= 1e-9 * fa
        w = np.linalg.eigvalsh(A64.T @ A64 - r.B.T @ r.B)
        nrm = max(abs(w[0]), abs(w[-1]))
        k = 0
        while k < ell / 2 - 0.5:
            assert nrm <= np.sum(sv2[k:]) / (ell / 2 - 0.5 - k) * (1 + 1e-9)
            k += 1
        for k in range(1, int(np.ceil(ell / 2 - 1))):
            if k < ell / 2 - 1:
                p = oracle.proj_err(A, r.B, k=k)
                assert p["err"] <= (ell - 1) / (ell - 1 - 2 * k) * (1 + 1e-9)


def test_ssd_lossless_when_rank_below_ell():
    """Reading C26: a buffer of rank <= ell-1 (sigma_ell = 0) is compressed losslessly."""
    rng = np.random.default_rng(4)
    ell, d = 7, 19
    A = (rng.standard_normal((200, ell - 1)) @ rng.standard_normal((ell - 1, d))).astype(np.float32)
    r = oracle.sketch(A, ell, "ssd")
    AtA, frob = oracle.gram(A)
    assert np.abs(AtA - r.B.T @ r.B).max() <= 1e-10 * frob
    assert r.delta_total == 0.0


@pytest.mark.parametrize("shards", [1, 3])
def test_cfd_is_fd_plus_delta_on_ell_directions(shards):
    """CFD runs FD and compensates only the final step: B_cfd^T B_cfd -
    B_fd^T B_fd = Delta * (projector onto the final ell directions): ell eigenvalues
    Delta, the rest 0.  With one stream the mass is preserved, ||A||_F^2 = ||B||_F^2, and
    | ||Ax||^2 - ||Bx||^2 | <= Delta."""
    A = _c1()
    ell = 16
    rf = oracle.sketch(A, ell, "fd", n_shards=shards)
    rc = oracle.sketch(A, ell, "cfd", n_shards=shards)
    assert abs(rc.delta_total - rf.delta_total) <= 1e-12 * rf.delta_total
    Dl = rf.delta_total
    w = np.linalg.eigvalsh(rc.B.T @ rc.B - rf.B.T @ rf.B)[::-1]
    np.testing.assert_allclose(w[:ell], Dl, rtol=1e-8)
    assert np.all(np.abs(w[ell:]) <= 1e-8 * Dl)
    A64 = A.astype(np.float64)
    if shards == 1:
        fa = float(np.sum(A64 ** 2))
        assert abs(float(np.sum(rc.B ** 2)) - fa) <= 1e-9 * fa
        m = np.linalg.eigvalsh(A64.T @ A64 - rc.B.T @ rc.B)
        assert max(abs(m[0]), abs(m[-1])) <= Dl * (1 + 1e-9)


# ---------------------------------------------------------------------------
# Hashing / OSNAP (reading C28)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("s", [1, 4])
def test_hash_sketch_is_a_signed_bucket_matrix(s):
    """A = I_n: B = S itself.  Every column has exactly one nonzero per block, of
    magnitude 1/sqrt(s) (PAPER.md:198: one non-zero per column, +-1; :200: s stacked)."""
    n, ell = 200, 16
    S = oracle.hash_sketch(np.eye(n, dtype=np.float32), ell, s=s, seed=3)
    lb = ell // s
    for j in range(s):
        blk = S[j * lb:(j + 1) * lb]
        assert np.all(np.count_nonzero(blk, axis=0) == 1)
        assert np.allclose(np.abs(blk).sum(axis=0), 1.0 / np.sqrt(s), rtol=0, atol=1e-15)


def test_hash_sketch_linear_and_mergeable():
    """B(A) for one call = B(first part) + B(second part, row0 offset), exactly (fp64,
    same summation order), and B is linear in A."""
    A = _c1()
    B = oracle.hash_sketch(A, 16, s=4, seed=9)
    B2 = oracle.hash_sketch(A[:700], 16, s=4, seed=9)
    oracle.hash_sketch(A[700:], 16, s=4, seed=9, row0=700, B=B2)
    assert np.array_equal(B, B2)
    C = oracle.hash_sketch(2.0 * A, 16, s=4, seed=9)
    assert np.array_equal(C, 2.0 * B)


def test_hash_sketch_unbiased_covariance():
    """E[B^T B] = A^T A: over 400 seeds the mean of B^T B approaches A^T A (the
    off-diagonal terms cancel in expectation: independent signs), within 5 standard errors."""
    rng = np.random.default_rng(2)
    A = rng.standard_normal((60, 5)).astype(np.float32)
    AtA = A.astype(np.float64).T @ A.astype(np.float64)
    acc = []
    for seed in range(400):
        B = oracle.hash_sketch(A, 8, s=4, seed=seed)
        acc.append(B.T @ B)
    acc = np.array(acc)
    mean, se = acc.mean(0), acc.std(0) / np.sqrt(len(acc))
    assert np.all(np.abs(mean - AtA) <= 5 * se + 1e-9)


# --------------------------------------------------------------------------
# oracle/alg1_svd.py: Alg. 1 with a library SVD, used for the
# c4 cached results.  Pinned to oracle.c's Gram + Jacobi formulation (independent:
# no shared code, a different factorisation) and to the hand examples / bounds.
# --------------------------------------------------------------------------
from oracle import alg1_svd  # noqa: E402

SVD_VARIANTS = ["fd", "fast_fd", "alpha_fd", "fast_alpha_fd", "isvd", "fast_isvd"]


@pytest.mark.parametrize("variant", SVD_VARIANTS)
def test_alg1_svd_matches_jacobi_oracle_c1(variant):
    A = _c1()
    B, st = alg1_svd.sketch_stream(A, 16, variant, alpha=0.2)
    r = oracle.sketch(A, 16, variant, alpha=0.2)
    assert np.abs(B.T @ B - r.B.T @ r.B).max() < 1e-11 * r.frob_sq
    np.testing.assert_allclose(st, [r.frob_sq, r.delta_total, r.removed, r.n_shrinks, r.rows_seen],
                               rtol=1e-11, atol=1e-11 * r.frob_sq)


@pytest.mark.parametrize("variant", ["fast_fd", "fast_alpha_fd"])
def test_alg1_svd_matches_jacobi_oracle_c4_shard(variant):
    """A c4-shaped stream (d = 1024, ell = 128, L = 256): 400 rows (one buffer ReduceRank + the
    final one), two 200-row shards and their merge."""
    w = fdgen.config("c4")
    A = fdgen.host_rows(w, 0, 400, nthreads=1)
    B, st = alg1_svd.sketch_stream(A, 128, variant, alpha=0.2)
    r = oracle.sketch(A, 128, variant, alpha=0.2, n_shards=2, want_shards=True)
    X, sx = alg1_svd.sketch_stream(A[:200], 128, variant, alpha=0.2)
    Y, sy = alg1_svd.sketch_stream(A[200:], 128, variant, alpha=0.2)
    for S, ref in ((X, r.shards[0]), (Y, r.shards[1])):
        assert np.linalg.norm(S.T @ S - ref.T @ ref, 2) < 1e-11 * r.frob_sq
    M, sm = alg1_svd.merge(X, Y, 128, variant, alpha=0.2)
    assert np.linalg.norm(M.T @ M - r.B.T @ r.B, 2) < 1e-11 * r.frob_sq
    Mo, smo = oracle.merge(np.stack([r.shards[0], r.shards[1]]), 128, variant, alpha=0.2)
    np.testing.assert_allclose(sm[1:4], smo[1:4], rtol=1e-10)
    r1 = oracle.sketch(A, 128, variant, alpha=0.2)
    assert np.linalg.norm(B.T @ B - r1.B.T @ r1.B, 2) < 1e-11 * r1.frob_sq
    assert abs(st[1] - r1.delta_total) < 1e-10 * r1.delta_total and int(st[3]) == r1.n_shrinks


@pytest.mark.parametrize("case", [c for c in _read_golden_rules() if c[0] in ("fd", "isvd")])
def test_alg1_svd_hand_examples(case):
    """The SPEC.md hand examples of the FD / alpha-FD / iSVD rules, on the SVD formulation."""
    rule, alpha, ell, s_in, s_out, delta = case
    L = len(s_in)
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.standard_normal((L + 1, L + 1)))
    Bf = np.diag(s_in) @ Q[:L]
    m = ell if rule == "isvd" else max(1, int(np.floor(alpha * ell + 0.5)))
    B, dl, removed = alg1_svd.reduce_rank(Bf, ell, "isvd" if rule == "isvd" else "fd", m)
    sv = np.linalg.svd(B, compute_uv=False)
    expect = np.zeros(len(sv))
    expect[: len(s_out)] = s_out
    np.testing.assert_allclose(sv ** 2, expect ** 2, atol=1e-12 * max(1.0, max(s_in) ** 2))
    assert abs(dl - delta) < 1e-12 * max(1.0, max(s_in) ** 2)


def test_alg1_svd_bounds_c2_prefix():
    """Lemma 1 / Lemma 3 on the SVD formulation: 0 <= ||Ax||^2 - ||Bx||^2 <= Delta,
    ||A||_F^2 - ||B||_F^2 = ell Delta (FD per-row)."""
    w = fdgen.config("c2")
    A = fdgen.host_rows(w, 0, 600, nthreads=1)
    B, st = alg1_svd.sketch_stream(A, 20, "fd")
    A64 = A.astype(np.float64)
    ev = np.linalg.eigvalsh(A64.T @ A64 - B.T @ B)
    assert ev[0] > -1e-10 * st[0] and ev[-1] <= st[1] * (1 + 1e-10)
    assert abs(st[0] - np.sum(B ** 2) - 20 * st[1]) < 1e-10 * st[0]
