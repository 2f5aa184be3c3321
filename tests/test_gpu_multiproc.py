"""The multi-process path with real CUDA on both sides.

Two processes share the one GPU of the test box (their kernels never wait on each
other: each sketches its own rows, then the host gathers).  Rank r sketches the rows
of the global shards [r P/2, (r+1) P/2) (dist.local_range; P does not divide n here,
the case ADVICE round 1 found) with the CUDA Sketcher, the ell x d sketches are
all-gathered over gloo (host copies), and every rank merges them with the CUDA
fd_merge (dist.gather_and_merge).  The result must equal the one-process sketch with
the same P_total (reading C10: the DAG depends on P_total only) and the oracle run
with the same DAG.
"""
import os
import socket

import numpy as np
import pytest

import fdgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, cfg, n, ell, variant, P, out_dir):
    import torch.distributed as dist

    import paper_1501_06561_b200 as fd
    from paper_1501_06561_b200.dist import dist_sketch, local_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        torch.cuda.set_device(0)
        w = fdgen.config(cfg, n=n)
        r0, r1 = local_range(w.n, rank, WORLD, P)
        A = torch.empty((r1 - r0, w.d), dtype=torch.float32, device="cuda")
        fdgen.DeviceGenerator(w).fill(A, r0)
        sk = fd.Sketcher(w.d, ell, variant, n_shards=P // WORLD)
        sk.append(A)
        B, st = dist_sketch(sk)
        # evaluator: partial Grams summed over the ranks (gloo all_reduce on host copies)
        AtA = torch.zeros((w.d, w.d), dtype=torch.float64, device="cuda")
        fd.cov_gram_partial(A, AtA)
        G = AtA.cpu()
        dist.all_reduce(G)
        frob = float(torch.diagonal(G).sum())
        e = fd.cov_err_from_gram(G.cuda(), B, frob)
        np.save(os.path.join(out_dir, f"B{rank}.npy"), B.cpu().numpy())
        np.save(os.path.join(out_dir, f"s{rank}.npy"),
                np.array([st["frob_sq"], st["delta_total"], st["removed_mass"], st["n_shrinks"], st["rows_seen"],
                          e["err"]]))
        sk.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,n,ell,variant,P", [("c2", 10000, 40, "fast_fd", 6), ("c1", 2000, 16, "fd", 2)])
def test_two_process_cuda_sketch_matches_single_process(tmp_path, cfg, n, ell, variant, P):
    import torch.multiprocessing as mp

    import paper_1501_06561_b200 as fd
    mp.start_processes(_worker, args=(_port(), cfg, n, ell, variant, P, str(tmp_path)), nprocs=WORLD,
                       start_method="spawn", join=True)
    w = fdgen.config(cfg, n=n)
    A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda")
    fdgen.DeviceGenerator(w).fill(A, 0)
    sk = fd.Sketcher(w.d, ell, variant, n_shards=P)
    sk.append(A)
    B1, st1 = sk.sketch()
    B1 = B1.cpu().numpy().astype(np.float64)
    sk.close()
    e1 = fd.cov_err(A, torch.from_numpy(B1.astype(np.float32)).cuda())["err"]
    An = A.cpu().numpy()
    ro = oracle.sketch(An, ell, variant, n_shards=P)
    frob = ro.frob_sq
    for rank in range(WORLD):
        B = np.load(tmp_path / f"B{rank}.npy").astype(np.float64)
        s = np.load(tmp_path / f"s{rank}.npy")
        # same DAG, same kernels: the one-process sketch up to fp32 rounding order
        M = B.T @ B - B1.T @ B1
        assert np.max(np.abs(np.linalg.eigvalsh((M + M.T) / 2))) <= 1e-6 * frob
        Mo = B.T @ B - ro.B.T @ ro.B
        assert np.max(np.abs(np.linalg.eigvalsh((Mo + Mo.T) / 2))) <= 1e-4 * frob
        assert abs(s[0] - frob) <= 1e-9 * frob
        assert int(s[3]) == ro.n_shrinks and int(s[4]) == w.n
        assert abs(s[1] - ro.delta_total) <= 1e-4 * frob + 1e-5 * ro.delta_total
        assert abs(s[5] - e1) <= 1e-6 * e1 + 1e-9
    assert np.array_equal(np.load(tmp_path / "B0.npy"), np.load(tmp_path / "B1.npy"))
