"""Multi-GPU plumbing (one process per GPU, torch.distributed).

Rows are split evenly across ranks; each rank sketches its rows with
P_local = P_total / world shards (so the shard DAG depends only on P_total,
reading C10), then the per-rank sketches are all-gathered (NCCL over
NVLink/NVSwitch) and every rank runs the same recursive-halving merge tree
locally (fd_merge) — deterministic, no broadcast.  The evaluator's d x d
partial Grams are summed with one all_reduce.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

STAT_KEYS = ("frob_sq", "delta_total", "removed_mass", "n_shrinks", "rows_seen")


def local_range(n: int, rank: int, world: int, n_shards_total: int | None = None):
    """Contiguous row range of `rank`: the rows of the global shards
    [rank P_local, (rank+1) P_local), P_local = P_total / world, with the global
    shard sizes floor(n/P_total) + (s < n mod P_total) of reading C10.  The rank's
    fd_append_rows then splits its range into exactly those P_local shards, so the
    g-rank DAG is the 1-GPU DAG at the same P_total for every n (not only when
    P_total divides n).  P_total defaults to world (one shard per rank)."""
    P = world if n_shards_total is None else int(n_shards_total)
    if P < 1 or P % world:
        raise ValueError(f"P_total={P} must be a positive multiple of world={world}")
    q, r = divmod(n, P)
    pl = P // world
    s0, s1 = rank * pl, (rank + 1) * pl
    return s0 * q + min(s0, r), s1 * q + min(s1, r)


def gather_and_merge(B_local, stats_local: dict, merge_fn, group=None):
    """all_gather the per-rank sketches and merge them with `merge_fn`
    ((world x ell x d) tensor -> (B, merge_stats)); stats are summed across ranks
    and the merge's own delta / removed / shrinks are added."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return B_local, dict(stats_local)
    nccl = dist.get_backend(group) == "nccl"
    if nccl:
        gathered = torch.empty((world,) + tuple(B_local.shape), dtype=B_local.dtype, device=B_local.device)
        dist.all_gather_into_tensor(gathered, B_local.contiguous(), group=group)
    else:  # gloo: list form of the same gather on host copies, result back on B's device
        Bh = B_local.detach().to("cpu").contiguous()
        gh = torch.empty((world,) + tuple(Bh.shape), dtype=Bh.dtype)
        dist.all_gather(list(gh.unbind(0)), Bh, group=group)
        gathered = gh.to(B_local.device)
    vec = torch.tensor([float(stats_local[k]) for k in STAT_KEYS], dtype=torch.float64,
                       device=B_local.device if nccl else "cpu")
    dist.all_reduce(vec, group=group)
    B, mst = merge_fn(gathered)
    out = {k: float(v) for k, v in zip(STAT_KEYS, vec.tolist())}
    if mst:
        out["delta_total"] += mst["delta_total"]
        out["removed_mass"] += mst["removed_mass"]
        out["n_shrinks"] += mst["n_shrinks"]
    out["n_shrinks"] = int(out["n_shrinks"])
    out["rows_seen"] = int(out["rows_seen"])
    return B, out


def dist_sketch(sketcher, group=None):
    """Sketch of the rows appended on all ranks (every rank returns the same B)."""
    B_local, st = sketcher.sketch(stats=True)
    return gather_and_merge(B_local, st, lambda S: sketcher.merge(S, stats=True), group)


def reduce_gram(AtA, group=None, frob_fn=None):
    """Sum the per-rank d x d fp64 partial Grams in place (one all_reduce);
    returns (AtA, ||A||_F^2 = trace(AtA)).  `frob_fn` computes the trace (libfd's
    fd_cov_frob_from_gram for device Grams; the CPU gloo tests pass their own)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(AtA, group=group)
    if frob_fn is None:
        from . import cov_frob_from_gram as frob_fn
    return AtA, float(frob_fn(AtA))


def dist_cov_err(A_local, B, group=None, proj_k=0):
    """cov-err of B for the row-sharded A (sum of partial Grams by all_reduce); with
    proj_k > 0 also proj-err at k = proj_k from the same A^T A."""
    from . import cov_err_from_gram, cov_gram_partial, proj_err_from_gram
    d = B.shape[1]
    AtA = torch.zeros((d, d), dtype=torch.float64, device=B.device)
    cov_gram_partial(A_local, AtA)
    AtA, frob = reduce_gram(AtA, group)
    out = cov_err_from_gram(AtA, B, frob)
    if proj_k > 0:
        out["proj_err"] = proj_err_from_gram(AtA, B, frob, k=proj_k)["err"]
    return out


def reduce_hash(B, group=None):
    """Merge of the Hashing / OSNAP sketches: the sketch is
    linear in the rows, B = S A = sum over ranks of S[:, rows_r] A[rows_r], so with every
    rank hashing its rows by their GLOBAL index (fd_hash_sketch's row0 = the rank's first
    row) the merge is one all_reduce(SUM) of the ell x d fp64 accumulators, in place."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(B, group=group)
    return B
