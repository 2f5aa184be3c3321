#!/usr/bin/env python
"""Write the cached oracle results the full-size GPU parity tests compare against.

TEST INFRASTRUCTURE.  Calls only `oracle/` (the fp64 CPU oracle) and `fdgen`
(the seeded input generator, which holds none of the method's arithmetic); no
value here comes from the CUDA path.  Output: tests/golden/full_<key>.npz with
  B        the oracle's root sketch (ell x d), stored as fp32 (the C12 sketch
           tolerance is 1e-4 ||A||_F^2; fp32 storage perturbs B^T B by ~1e-7 of it)
  stats    [frob_sq, Delta, removed, n_shrinks, rows_seen]   (oracle.sketch's order)
  err      cov-err of the fp64 oracle B, lmax, lmin (both / ||A||_F^2)
and the run parameters (cfg, variant, ell, alpha, P_total).

Workloads ("next round" item 1; BASELINE.json configs):
  c2 per-row FD / 0.2-FD / iSVD at ell in {60, 80, 100}, P_total = 1 (Fig. 5 :668-678)
  c5 per-row FD / 0.2-FD / iSVD at ell = 32, P_total = 1 (config 5; PAPER.md:543 intent)
  c3 Fast FD / Fast 0.2-FD at ell in {50, 100, 200}, P_total = 296 (CIFAR-10 stand-in)
  c4 Fast FD / Fast 0.2-FD at ell = 128, P_total = 2368 (the bench configuration)

A sharded run (P_total > 1) is computed shard by shard: shard s is
`oracle.sketch(rows of shard s, n_shards=1)` -- the same stream + final
ReduceRank that `oracle.sketch(A, n_shards=P)` runs for it (C10 ranges
floor(n/P) + (s < n mod P)) -- cached under .golden_cache/ so the long runs
resume, then merged with tests/oracle_tree.merge_tree (the oracle's own
recursive-halving tree, pinned to oracle.merge in test_oracle_pins.py).  The
cov-err's A^T A is oracle.gram over fixed row chunks, summed in chunk order.

c4 (64 000 ReduceRanks of 256 x 1024 per variant) runs on oracle/alg1_svd.py,
Alg. 1 with a library SVD as the paper itself runs it: the
Jacobi oracle needs ~1.3 s per ReduceRank there (~7 CPU hours per variant), the
SVD formulation ~0.05 s.  It is pinned to oracle.c's sketch and merge to fp64
rounding in tests/test_oracle_pins.py (test_alg1_svd_*); shards and the tree run
in worker threads with single-threaded BLAS.

    python tests/golden/make_goldens.py [--only KEY[,KEY..]] [--threads T]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import sys
import time

# single-threaded BLAS: the parallelism is over shards / tree nodes
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import fdgen  # noqa: E402
import oracle  # noqa: E402
from oracle import alg1_svd  # noqa: E402
from oracle_tree import merge_tree  # noqa: E402

CACHE = os.path.join(ROOT, ".golden_cache")
OUT = os.path.join(ROOT, "tests", "golden")
C3_P = 296
C4_P = 2368
GRAM_CHUNK = 131072


def jobs_table():
    J = []
    for ell in (60, 80, 100):
        for v in ("fd", "alpha_fd", "isvd"):
            J.append(dict(key=f"c2_{v}_l{ell}_p1", cfg="c2", variant=v, ell=ell, alpha=0.2, P=1))
    for v in ("fd", "alpha_fd", "isvd"):
        J.append(dict(key=f"c5_{v}_l32_p1", cfg="c5", variant=v, ell=32, alpha=0.2, P=1))
    for ell in (50, 100, 200):
        for v in ("fast_fd", "fast_alpha_fd"):
            J.append(dict(key=f"c3_{v}_l{ell}_p{C3_P}", cfg="c3", variant=v, ell=ell, alpha=0.2, P=C3_P))
    for v in ("fast_fd", "fast_alpha_fd"):
        J.append(dict(key=f"c4_{v}_l128_p{C4_P}", cfg="c4", variant=v, ell=128, alpha=0.2, P=C4_P,
                      engine="svd"))
    return J


def workload(cfg):
    w = fdgen.config(cfg)
    if w.kind == fdgen.KIND_IMAGE:
        path = os.path.join(CACHE, f"{cfg}_minmax.json")
        if os.path.exists(path):
            w.xminmax = tuple(json.load(open(path)))
        else:
            w.xminmax = fdgen.host_minmax(w)
            os.makedirs(CACHE, exist_ok=True)
            json.dump(list(w.xminmax), open(path, "w"))
    return w


def shard_range(n, P, s):
    q, r = divmod(n, P)
    return s * q + min(s, r), q + (1 if s < r else 0)


def shard_task(job, w, s):
    d = os.path.join(CACHE, job["key"])
    path = os.path.join(d, f"shard_{s:05d}.npz")
    if os.path.exists(path):
        return s
    r0, nr = shard_range(w.n, job["P"], s)
    A = fdgen.host_rows(w, r0, nr, nthreads=1)
    if job.get("engine") == "svd":
        B, st = alg1_svd.sketch_stream(A, job["ell"], job["variant"], alpha=job["alpha"])
    else:
        res = oracle.sketch(A, job["ell"], job["variant"], alpha=job["alpha"], n_shards=1, nthreads=1)
        B = res.B
        st = np.array([res.frob_sq, res.delta_total, res.removed, res.n_shrinks, res.rows_seen])
    tmp = path + ".tmp.npz"
    np.savez(tmp, B=B, stats=st)
    os.replace(tmp, path)
    return s


def gram_task(cfg, w, c):
    d = os.path.join(CACHE, f"{cfg}_gram")
    path = os.path.join(d, f"chunk_{c:05d}.npz")
    if os.path.exists(path):
        return c
    r0 = c * GRAM_CHUNK
    nr = min(GRAM_CHUNK, w.n - r0)
    A = fdgen.host_rows(w, r0, nr, nthreads=1)
    G, f = oracle.gram(A, nthreads=1)
    tmp = path + ".tmp.npz"
    np.savez(tmp, G=G, frob=np.array([f]))
    os.replace(tmp, path)
    return c


def full_gram(cfg, w, ex):
    os.makedirs(os.path.join(CACHE, f"{cfg}_gram"), exist_ok=True)
    nch = (w.n + GRAM_CHUNK - 1) // GRAM_CHUNK
    list(ex.map(lambda c: gram_task(cfg, w, c), range(nch)))
    G = np.zeros((w.d, w.d))
    f = 0.0
    for c in range(nch):
        z = np.load(os.path.join(CACHE, f"{cfg}_gram", f"chunk_{c:05d}.npz"))
        G += z["G"]
        f += float(z["frob"][0])
    return G, f


def err_from_gram(G, frob, B):
    """cov-err from A^T A: oracle's extreme eigenvalues of A^T A - B^T B."""
    M = G - B.T @ B
    hi, lo = oracle.sym_extremes(M, jacobi_max=1024, kmax=512)
    return max(abs(hi), abs(lo)) / frob, hi / frob, lo / frob


def run_job(job, threads, log):
    out = os.path.join(OUT, f"full_{job['key']}.npz")
    if os.path.exists(out):
        log(f"{job['key']}: exists")
        return
    t0 = time.time()
    w = workload(job["cfg"])
    with cf.ThreadPoolExecutor(threads) as ex:
        if job["P"] == 1:
            A = fdgen.host_rows(w, 0, w.n)
            res = oracle.sketch(A, job["ell"], job["variant"], alpha=job["alpha"], n_shards=1, nthreads=1)
            B = res.B
            stats = np.array([res.frob_sq, res.delta_total, res.removed, res.n_shrinks, res.rows_seen])
            e = oracle.cov_err(A, B, nthreads=threads)
            err, lmax, lmin = e["err"], e["lmax"], e["lmin"]
        else:
            os.makedirs(os.path.join(CACHE, job["key"]), exist_ok=True)
            P = job["P"]
            done = 0
            for s in ex.map(lambda s: shard_task(job, w, s), range(P)):
                done += 1
                if done % 64 == 0:
                    log(f"{job['key']}: {done}/{P} shards, {time.time() - t0:.0f} s")
            S = np.empty((P, job["ell"], w.d))
            stats = np.zeros(5)
            for s in range(P):
                z = np.load(os.path.join(CACHE, job["key"], f"shard_{s:05d}.npz"))
                S[s] = z["B"]
                stats += z["stats"]
            mf = None
            if job.get("engine") == "svd":
                mf = lambda X, Y: alg1_svd.merge(X, Y, job["ell"], job["variant"], alpha=job["alpha"])  # noqa: E731
            B, mst = merge_tree(S, job["ell"], job["variant"], alpha=job["alpha"], nthreads=threads, merge_fn=mf)
            stats[1:4] += mst[1:4]
            del S
            G, f = full_gram(job["cfg"], w, ex)
            assert abs(f - stats[0]) <= 1e-9 * f, (f, stats[0])
            err, lmax, lmin = err_from_gram(G, stats[0], B)
    np.savez_compressed(out, B=B.astype(np.float32), stats=stats, err=np.array([err, lmax, lmin]),
                        params=json.dumps(dict(cfg=job["cfg"], variant=job["variant"], ell=job["ell"],
                                               alpha=job["alpha"], P_total=job["P"], n=w.n, d=w.d)))
    log(f"{job['key']}: err {err:.6g} lmin {lmin:.3g} shrinks {int(stats[3])} in {time.time() - t0:.0f} s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--threads", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    a = ap.parse_args()
    only = set(x for x in a.only.split(",") if x)

    def log(msg):
        print(time.strftime("%H:%M:%S"), msg, flush=True)

    jobs = [j for j in jobs_table() if not only or j["key"] in only or j["cfg"] in only]
    small = [j for j in jobs if j["P"] == 1]
    # per-row P = 1 jobs are single-threaded chains: run them side by side
    with cf.ThreadPoolExecutor(a.threads) as ex:
        list(ex.map(lambda j: run_job(j, 1, log), small))
    for j in jobs:
        if j["P"] > 1:
            run_job(j, a.threads, log)


if __name__ == "__main__":
    main()
