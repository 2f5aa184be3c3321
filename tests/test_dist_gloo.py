"""The N>1 host path on CPU: world_size-2 torch.distributed (gloo) runs of the
row partition, the sketch all_gather + merge plumbing and the evaluator's Gram
all_reduce (paper_1501_06561_b200/dist.py), with the CPU oracle standing in for
the per-rank CUDA sketch (test infrastructure only).

Checks reading C10: the g-rank result equals the single-process oracle at the
same P_total (the merge DAG depends on P_total only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fdgen
import oracle
from paper_1501_06561_b200.dist import gather_and_merge, local_range, reduce_gram, reduce_hash

WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, P_total, ell, variant, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        A = fdgen.host_rows(fdgen.config("c1"))
        r0, r1 = local_range(A.shape[0], rank, WORLD, P_total)
        # per-rank sketch of its rows with P_total / world shards (oracle stands in
        # for fd_append_rows + fd_sketch on the GPU)
        r = oracle.sketch(A[r0:r1], ell, variant, n_shards=P_total // WORLD)
        st = dict(frob_sq=r.frob_sq, delta_total=r.delta_total, removed_mass=r.removed,
                  n_shrinks=r.n_shrinks, rows_seen=r.rows_seen)

        def merge_fn(S):
            B, mst = oracle.merge(S.numpy().astype(np.float64), ell, variant)
            return torch.from_numpy(B), dict(delta_total=mst[1], removed_mass=mst[2], n_shrinks=mst[3])

        B, tot = gather_and_merge(torch.from_numpy(r.B), st, merge_fn)
        AtA_p, _ = oracle.gram(A[r0:r1])
        AtA, frob = reduce_gram(torch.from_numpy(AtA_p), frob_fn=lambda G: torch.diagonal(G).sum().item())
        np.save(os.path.join(out_dir, f"B{rank}.npy"), B.numpy())
        np.save(os.path.join(out_dir, f"G{rank}.npy"), AtA.numpy())
        np.save(os.path.join(out_dir, f"s{rank}.npy"),
                np.array([tot["frob_sq"], tot["delta_total"], tot["removed_mass"], tot["n_shrinks"],
                          tot["rows_seen"], frob]))
    finally:
        dist.destroy_process_group()


def test_local_range_partition():
    for n in (0, 1, 7, 2000, 8388608):
        for g in (1, 2, 3, 8):
            rs = [local_range(n, r, g) for r in range(g)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(g - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def _split(n, P):
    q, r = divmod(n, P)
    return [q + (1 if s < r else 0) for s in range(P)]


@pytest.mark.parametrize("n,P,g", [(8388608, 2368, 8), (8388608, 2368, 2), (2003, 4, 2), (60000, 296, 8),
                                   (7, 8, 4), (1000, 24, 3)])
def test_local_range_is_shard_aligned(n, P, g):
    """Each rank's rows are exactly the global shards [r P/g, (r+1) P/g) of the
    1-GPU split (reading C10), and fd_append_rows' split of the rank's range into
    P/g shards reproduces their sizes: the g-rank DAG is the 1-GPU DAG at P_total
    also when P_total does not divide n."""
    glob = _split(n, P)
    off = 0
    for r in range(g):
        a, b = local_range(n, r, g, P)
        assert a == off
        loc = _split(b - a, P // g)
        assert loc == glob[r * (P // g):(r + 1) * (P // g)]
        off = b
    assert off == n
    with pytest.raises(ValueError):
        local_range(n, 0, g, P + 1 if (P + 1) % g else P + 2)


@pytest.mark.parametrize("variant", ["fast_fd", "alpha_fd"])
@pytest.mark.parametrize("P_total", [4, 6])
def test_two_rank_gloo_matches_single_process(tmp_path, variant, P_total):
    ell = 16
    mp.start_processes(_worker, args=(_port(), P_total, ell, variant, str(tmp_path)), nprocs=WORLD,
                       start_method="spawn", join=True)
    A = fdgen.host_rows(fdgen.config("c1"))
    ref = oracle.sketch(A, ell, variant, n_shards=P_total)
    G, frob = oracle.gram(A)
    for rank in range(WORLD):
        B = np.load(tmp_path / f"B{rank}.npy")
        s = np.load(tmp_path / f"s{rank}.npy")
        # same DAG -> same sketch (fp64 oracle on both sides: rounding-order only)
        assert np.abs(B.T @ B - ref.B.T @ ref.B).max() <= 1e-10 * ref.frob_sq
        assert abs(s[0] - ref.frob_sq) <= 1e-12 * ref.frob_sq
        assert abs(s[1] - ref.delta_total) <= 1e-10 * ref.frob_sq
        assert abs(s[2] - ref.removed) <= 1e-10 * ref.frob_sq
        assert int(s[3]) == ref.n_shrinks and int(s[4]) == A.shape[0]
        Gr = np.load(tmp_path / f"G{rank}.npy")
        assert np.abs(Gr - G).max() <= 1e-12 * frob
        assert abs(s[5] - frob) <= 1e-12 * frob
    # both ranks hold the identical sketch (deterministic local merge, no broadcast)
    assert np.array_equal(np.load(tmp_path / "B0.npy"), np.load(tmp_path / "B1.npy"))


def _hash_worker(rank, port, ell, s_blocks, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        A = fdgen.host_rows(fdgen.config("c1"))
        r0, r1 = local_range(A.shape[0] - 3, rank, WORLD)   # ragged split
        # the oracle stands in for fd_hash_sketch(row0 = r0) on the GPU
        Bp = oracle.hash_sketch(A[r0:r1], ell, s=s_blocks, seed=7, row0=r0)
        B = reduce_hash(torch.from_numpy(Bp))
        np.save(os.path.join(out_dir, f"H{rank}.npy"), B.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("s_blocks", [1, 4])
def test_two_rank_gloo_hash_merge_is_a_sum(tmp_path, s_blocks):
    """Hashing / OSNAP across ranks: ranks hash their rows by
    global row index and all_reduce the fp64 accumulators; the result is the single-process
    sketch of the same rows (sums reordered by rank only)."""
    ell = 16
    mp.start_processes(_hash_worker, args=(_port(), ell, s_blocks, str(tmp_path)), nprocs=WORLD,
                       start_method="spawn", join=True)
    A = fdgen.host_rows(fdgen.config("c1"))
    n = A.shape[0] - 3
    ref = oracle.hash_sketch(A[:n], ell, s=s_blocks, seed=7)
    scale = np.abs(ref).max()
    H0, H1 = np.load(tmp_path / "H0.npy"), np.load(tmp_path / "H1.npy")
    assert np.abs(H0 - ref).max() <= 1e-13 * scale
    assert np.array_equal(H0, H1)
    # a rank that ignored its row offset would hash different buckets
    wrong = oracle.hash_sketch(A[n // 2:n], ell, s=s_blocks, seed=7, row0=0)
    right = oracle.hash_sketch(A[n // 2:n], ell, s=s_blocks, seed=7, row0=n // 2)
    assert np.abs(wrong - right).max() > 1e-3 * scale
