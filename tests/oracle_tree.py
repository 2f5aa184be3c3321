"""Thread-parallel evaluation of the oracle's recursive-halving merge tree.

TEST INFRASTRUCTURE (calls only `oracle/`).  `oracle.merge(S)` walks the tree of
DESIGN.md reading C10 (node [lo, hi) splits at lo + ceil((hi-lo)/2)) serially;
this helper evaluates the SAME tree, one `oracle.merge` of a pair per internal
node, with every node of one height in parallel (ctypes releases the GIL).
`tests/test_oracle_pins.py::test_parallel_tree_equals_oracle_merge` pins it to
`oracle.merge` on small counts (identical bytes).
"""
from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np

import oracle


def _build(lo, hi, nodes):
    """Post-order node list; returns (index of [lo, hi), its height)."""
    if hi - lo == 1:
        nodes.append(("leaf", lo, 0))
        return len(nodes) - 1, 0
    mid = lo + (hi - lo + 1) // 2
    a, ha = _build(lo, mid, nodes)
    b, hb = _build(mid, hi, nodes)
    h = 1 + max(ha, hb)
    nodes.append(("node", (a, b), h))
    return len(nodes) - 1, h


def merge_tree(sketches, ell, variant, alpha=None, nthreads=0, progress=None, merge_fn=None):
    """Root of the recursive-halving tree over `sketches` (count x ell x d, fp64 or fp32)
    with pairwise `oracle.merge` (or `merge_fn(X, Y) -> (B, stats5)`, e.g.
    oracle.alg1_svd.merge).  Returns (B, stats5) with stats5 = the merges' own
    [0, Delta, removed, n_shrinks, 0] summed (as `oracle.merge` reports them)."""
    S = np.asarray(sketches)
    count = S.shape[0]
    nodes = []
    root, H = _build(0, count, nodes)
    val = [None] * len(nodes)
    st_sum = np.zeros(5)
    for i, (kind, arg, h) in enumerate(nodes):
        if kind == "leaf":
            val[i] = np.ascontiguousarray(S[arg], dtype=np.float64)
    nthreads = nthreads or (os.cpu_count() or 1)

    def run(i):
        a, b = nodes[i][1]
        if merge_fn is not None:
            B, st = merge_fn(val[a], val[b])
        else:
            B, st = oracle.merge(np.stack([val[a], val[b]]), ell, variant, alpha=alpha)
        return i, B, st

    with cf.ThreadPoolExecutor(nthreads) as ex:
        for h in range(1, H + 1):
            todo = [i for i, nd in enumerate(nodes) if nd[0] == "node" and nd[2] == h]
            for i, B, st in ex.map(run, todo):
                val[i] = B
                st_sum += st
            if progress:
                progress(h, H, len(todo))
    return val[root], st_sum
