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


def local_range(n: int, rank: int, world: int):
    """Contiguous row range of `rank` (sizes floor(n/world) + (rank < n mod world))."""
    q, r = divmod(n, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def gather_and_merge(B_local, stats_local: dict, merge_fn, group=None):
    """all_gather the per-rank sketches and merge them with `merge_fn`
    ((world x ell x d) tensor -> (B, merge_stats)); stats are summed across ranks
    and the merge's own delta / removed / shrinks are added."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return B_local, dict(stats_local)
    gathered = torch.empty((world,) + tuple(B_local.shape), dtype=B_local.dtype, device=B_local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(gathered, B_local.contiguous(), group=group)
    else:  # gloo (CPU tests): list form of the same gather
        dist.all_gather(list(gathered.unbind(0)), B_local.contiguous(), group=group)
    vec = torch.tensor([float(stats_local[k]) for k in STAT_KEYS], dtype=torch.float64, device=B_local.device)
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


def reduce_gram(AtA, group=None):
    """Sum the per-rank d x d fp64 partial Grams in place (one all_reduce);
    returns (AtA, ||A||_F^2 = trace(AtA))."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(AtA, group=group)
    return AtA, float(torch.diagonal(AtA).sum().item())


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
