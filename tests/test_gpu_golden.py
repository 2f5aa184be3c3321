"""Full-size GPU parity against cached oracle results (tests/golden/full_*.npz).

The cached values were written by tests/golden/make_goldens.py, which calls only
`oracle/` (fp64 CPU oracle) and `fdgen` (seeded inputs); nothing here comes from
the CUDA path.  Each case runs the GPU sketch with the same DAG (P_total shard
streams, recursive-halving merge tree; reading C10) on the same seeded rows and
checks the C12 tolerances (reading C12):
  sketch : ||B_gpu^T B_gpu - B_ora^T B_ora||_2 <= 1e-4 ||A||_F^2
  err    : |err_gpu(A, B_gpu) - err_ora(A, B_ora)| <= 1e-3 err_ora + 1e-6
  stats  : frob to 1e-9, shrink count exact, Delta / removed to the sketch tolerance.
Workloads (BASELINE.json configs): c2 per-row at ell 60/80/100
(PAPER.md:539-541), c5 per-row at P_total = 1 (reading C15), c3 at n = 60 000 with
ell 50/100/200, c4 Fast FD and Fast 0.2-FD at the bench's
P_total = 2368 including the 12-level merge tail.
"""
import glob
import json
import os
import sys

import numpy as np
import pytest

import fdgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from oracle_tree import merge_tree  # noqa: E402

SKETCH_TOL = 1e-4
ERR_TOL = 1e-3
EPS32 = 2.0 ** -23


def err_floor(Bo, frob):
    """Absolute floor of the err comparison in fp32 ulps of the sketch (reading C12): storage
    2 eps32 ||B||_F^2 + fp32 arithmetic of B^T B's dominant directions 8 eps32 ||B||_2^2,
    over ||A||_F^2 (round 1 used a flat 1e-6)."""
    return EPS32 * (2.0 * float(np.sum(Bo ** 2)) + 8.0 * float(np.linalg.norm(Bo, 2)) ** 2) / frob
GOLD = sorted(glob.glob(os.path.join(HERE, "golden", "full_*.npz")))


def _id(path):
    return os.path.basename(path)[5:-4]


def spec_norm(M):
    """||M||_2 of a symmetric d x d fp64 matrix (numpy eigvalsh, test-side)."""
    w = np.linalg.eigvalsh((M + M.T) / 2)
    return float(max(abs(w[0]), abs(w[-1])))


_ROWS = {}


def device_rows(cfg, n):
    key = (cfg, n)
    if key not in _ROWS:
        _ROWS.clear()
        torch.cuda.empty_cache()
        w = fdgen.config(cfg)
        assert w.n == n
        gen = fdgen.DeviceGenerator(w)
        A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda")
        gen.fill(A, 0)
        _ROWS[key] = A
    return _ROWS[key]


@pytest.mark.parametrize("path", GOLD, ids=[_id(p) for p in GOLD])
def test_fullsize_parity_vs_cached_oracle(path):
    import paper_1501_06561_b200 as fd
    z = np.load(path)
    prm = json.loads(str(z["params"]))
    Bo = z["B"].astype(np.float64)
    st_o = z["stats"]
    err_o = float(z["err"][0])
    A = device_rows(prm["cfg"], prm["n"])
    sk = fd.Sketcher(prm["d"], prm["ell"], prm["variant"], alpha=prm["alpha"], n_shards=prm["P_total"])
    sk.append(A)
    B, st = sk.sketch()
    torch.cuda.synchronize()
    sk.close()
    frob = st_o[0]
    assert abs(st["frob_sq"] - frob) <= 1e-9 * frob
    assert st["rows_seen"] == prm["n"]
    assert st["n_shrinks"] == int(st_o[3])
    Bg = B.cpu().numpy().astype(np.float64)
    diff = spec_norm(Bg.T @ Bg - Bo.T @ Bo)
    assert diff <= SKETCH_TOL * frob, f"sketch diff {diff / frob:.3e} * frob"
    assert abs(st["delta_total"] - st_o[1]) <= SKETCH_TOL * frob + 1e-5 * st_o[1]
    assert abs(st["removed_mass"] - st_o[2]) <= 2 * SKETCH_TOL * frob
    # Lemma 3 ledger on the GPU side: ||A||_F^2 - ||B||_F^2 = removed
    assert abs((st["frob_sq"] - float(np.sum(Bg ** 2))) - st["removed_mass"]) <= SKETCH_TOL * frob
    eg = fd.cov_err(A, B)["err"]
    ea = err_floor(Bo, frob)
    assert abs(eg - err_o) <= ERR_TOL * err_o + ea, f"err gpu {eg} oracle {err_o} (floor {ea:.2e})"


def test_goldens_present():
    """The cached set covers every workload named in tests/golden/make_goldens.py."""
    sys.path.insert(0, os.path.join(HERE, "golden"))
    import make_goldens
    want = {j["key"] for j in make_goldens.jobs_table()}
    have = {_id(p) for p in GOLD}
    missing = sorted(want - have)
    assert not missing, f"golden files missing: {missing}"


def test_c4_merge_tail_vs_oracle_merge():
    """The c4 merge tail on its own: shards 0..255 of the bench DAG (c4, Fast FD,
    P_total = 2368; all 3543 rows long since 2368 does not divide n: the first 1152
    shards carry one extra row) as a 256-shard handle.  fd_sketch's recursive-halving
    merge (8 levels, merge Gram 2 ell - 2 = 254) against the oracle's tree
    (oracle.merge pairwise over the same tree, tests/oracle_tree.py) fed the GPU's own
    fp32 leaf sketches (fd_shard_sketch)."""
    import paper_1501_06561_b200 as fd
    w = fdgen.config("c4")
    P, ell, count = 2368, 128, 256
    q, r = divmod(w.n, P)
    assert r >= count
    nrows = count * (q + 1)
    gen = fdgen.DeviceGenerator(w)
    A = torch.empty((nrows, w.d), dtype=torch.float32, device="cuda")
    gen.fill(A, 0)
    sk = fd.Sketcher(w.d, ell, "fast_fd", n_shards=count)
    sk.append(A)
    Bg, _ = sk.sketch(stats=False)
    S = torch.stack([sk.shard_sketch(s) for s in range(count)])
    torch.cuda.synchronize()
    sk.close()
    del A
    Sh = S.cpu().numpy().astype(np.float64)
    Bo, _ = merge_tree(Sh, ell, "fast_fd")
    frob = float(np.sum(Sh ** 2))   # mass entering the tree
    Bgn = Bg.cpu().numpy().astype(np.float64)
    M = Bgn.T @ Bgn - Bo.T @ Bo
    diff = float(np.max(np.abs(np.linalg.eigvalsh((M + M.T) / 2))))
    assert diff <= SKETCH_TOL * frob, f"merge-tail diff {diff / frob:.3e} * ||S||_F^2"
