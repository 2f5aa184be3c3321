"""Evaluator timing on c4 (CUDA events): tensor-core A^T A, cov-err Lanczos, proj-err."""
import sys
import time
sys.path.insert(0, '.')
import torch
import fdgen
import paper_1501_06561_b200 as m

w = fdgen.config("c4")
gen = fdgen.DeviceGenerator(w)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda")
gen.fill(A, 0)
B = A[:128].contiguous()
AtA = torch.zeros((w.d, w.d), dtype=torch.float64, device="cuda")


def timed(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); t0 = time.perf_counter(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    print(name, "events ms", [round(a, 2) for a, _ in ts], "wall ms", [round(b, 2) for _, b in ts], flush=True)


timed("cov_gram_partial (c4)", lambda: (AtA.zero_(), m.cov_gram_partial(A, AtA)))
frob = m.cov_frob_from_gram(AtA)
timed("cov_err_from_gram", lambda: m.cov_err_from_gram(AtA, B, frob))
timed("proj_err_from_gram", lambda: m.proj_err_from_gram(AtA, B, frob, k=10))
