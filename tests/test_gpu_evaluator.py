"""GPU evaluator pieces against exact fp64 references (-m gpu).

fd_cov_gram_partial (tensor-core A^T A, reading E3): each chunk of rows is
column-scaled to 31-bit integers q = round(a 2^(30 - e_j)), split into four int8 digits,
and the digit products of weight 2^48 ... 2^16 are summed exactly in int32.  Per row and
entry the error is bounded by the rounding of q (2^-29 cmax_i cmax_j) and the dropped
digit products of weight <= 2^8 (<= (2^23 + 2^14) 2^-58 cmax_i cmax_j):
    |AtA_gpu - A^T A|_ij <= sum over chunks of n_c 2^-28 cmax_i cmax_j
(cmax = the chunk's column maxima).  A dropped or mis-scaled digit group, a transposed
plane or a wrong chunk exponent breaks this by orders of magnitude.  The reference is
A^T A in fp64 from the exact fp32 products (numpy, test-side).  The Lanczos evaluator is
compared with the oracle's on the same (A, B) in test_gpu_parity.py (relative 1e-6);
here additionally on c3 / c4 / c5 prefixes.
"""
import numpy as np
import pytest

import fdgen
import oracle
from oracle import alg1_svd

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def fd():
    import paper_1501_06561_b200 as m
    return m


def _bound(A, chunk_rows):
    b = np.zeros((A.shape[1], A.shape[1]))
    for r0 in range(0, A.shape[0], chunk_rows):
        c = np.abs(A[r0:r0 + chunk_rows]).max(axis=0).astype(np.float64)
        b += min(chunk_rows, A.shape[0] - r0) * 2.0 ** -28 * np.outer(c, c)
    return b


def _gram(A_host, ld_pad=0):
    n, d = A_host.shape
    At = torch.zeros((n, d + ld_pad), dtype=torch.float32)
    At[:, :d] = torch.from_numpy(A_host)
    Ad = At.cuda()[:, :d]
    G = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    fd().cov_gram_partial(Ad, G)
    torch.cuda.synchronize()
    return G.cpu().numpy()


def _chunk_rows(d):
    # the library's row chunk (fd_syrk_tc.cu syrk_chunk_rows): nsplit * 680 K-blocks of 64
    # rows, capped so the four digit planes of a chunk stay under 512 MiB
    ncb = (d + 127) // 128
    ntiles = ncb * (ncb + 1)          # 128 x 64 tiles of the lower block triangle
    nsplit = max(1, 148 // ntiles)
    by_mem = max(64, (512 << 20) // (ncb * 4 * 128) // 64 * 64)
    return min(nsplit * 680 * 64, by_mem)


@pytest.mark.parametrize("n,d,ld_pad", [(1, 7, 0), (300, 64, 3), (1000, 500, 0), (777, 129, 5), (2048, 1024, 0),
                                        (515, 3072, 4)])
def test_tc_gram_vs_exact(n, d, ld_pad):
    rng = np.random.default_rng(n * 31 + d)
    A = rng.standard_normal((n, d)).astype(np.float32)
    A[:, ::7] *= 1e-3                       # columns of very different scale
    A[n // 2:, 1::5] *= 1e4 if d > 1 else 1
    G = _gram(A, ld_pad)
    A64 = A.astype(np.float64)
    ref = A64.T @ A64
    assert np.all(np.abs(G - ref) <= _bound(A, _chunk_rows(d)) + 1e-300)
    np.testing.assert_array_equal(G, G.T)


@pytest.mark.parametrize("n,d", [(5000, 256), (3000, 1024)])
def test_tc_gram_gaussian_typical_error(n, d):
    """Without intra-column dynamic range the error is ~2^-30 cmax^2 per row, random in sign:
    ||dG||_F ~ 1e-9 ||G||_F (the worst-case bound above is n 2^-28 cmax^2)."""
    A = np.random.default_rng(d).standard_normal((n, d)).astype(np.float32)
    G = _gram(A)
    A64 = A.astype(np.float64)
    ref = A64.T @ A64
    assert np.linalg.norm(G - ref) <= 1e-8 * np.linalg.norm(ref)


def test_tc_gram_multi_chunk_scale_change():
    """Rows spanning several chunks whose column maxima differ by 1e6 (per-chunk exponents)."""
    d = 64
    cr = _chunk_rows(d)
    n = cr + cr // 2 + 77
    rng = np.random.default_rng(5)
    A = rng.standard_normal((n, d)).astype(np.float32)
    A[cr:] *= 1e-6
    A[:cr, 3] *= 1e3
    G = _gram(A)
    A64 = A.astype(np.float64)
    ref = A64.T @ A64
    assert np.all(np.abs(G - ref) <= _bound(A, cr))
    # the small second chunk is not swamped: its own Gram is reproduced
    Gs = _gram(A[cr:])
    ref_s = A64[cr:].T @ A64[cr:]
    assert np.linalg.norm(Gs - ref_s) <= 1e-6 * np.linalg.norm(ref_s)


def test_tc_gram_accumulates_and_nonfinite_is_nan():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((400, 96)).astype(np.float32)
    G = torch.eye(96, dtype=torch.float64, device="cuda")
    fd().cov_gram_partial(torch.from_numpy(A).cuda(), G)
    ref = A.astype(np.float64).T @ A.astype(np.float64) + np.eye(96)
    assert np.all(np.abs(G.cpu().numpy() - ref) <= _bound(A, _chunk_rows(96)) + 1e-12)
    A[17, 5] = np.inf
    G2 = torch.zeros((96, 96), dtype=torch.float64, device="cuda")
    fd().cov_gram_partial(torch.from_numpy(A).cuda(), G2)
    assert torch.isnan(G2).all()


@pytest.mark.parametrize("cfg,rows,ell", [("c3", 6000, 50), ("c4", 20000, 128), ("c5", 40000, 32)])
def test_cov_err_same_B_prefixes(cfg, rows, ell):
    """cov-err of the oracle's own sketch: GPU evaluator vs oracle evaluator, relative 1e-6 (C12)."""
    w = fdgen.config(cfg)
    if w.kind == fdgen.KIND_IMAGE:
        w.xminmax = fdgen.host_minmax(w)
    A = fdgen.host_rows(w, 0, rows)
    B, _ = alg1_svd.sketch_stream(A, ell, "fast_fd")     # any fixed B will do: the evaluator is under test
    B32 = B.astype(np.float32)
    eo = oracle.cov_err(A, B32.astype(np.float64))
    eg = fd().cov_err(torch.from_numpy(A).cuda(), torch.from_numpy(B32).cuda())
    assert abs(eg["err"] - eo["err"]) <= 1e-6 * eo["err"]
    assert abs(eg["lmin"] - eo["lmin"]) <= 1e-6 * eo["err"]
