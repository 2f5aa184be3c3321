"""Small cases covering every kernel path, for compute-sanitizer --tool memcheck:
per-row fp64 (N <= 160), legacy fp32 eig (N = 32), tridiagonal-kernel path
(32 < N <= 256: tcgen05 Gram, trd, lean eig, bt), large-N global-memory eig
(N = 400), merges, host-input staging, the evaluator."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1501_06561_b200 as m

rng = np.random.default_rng(0)
cases = [(600, 64, 16, "fd", 1), (600, 64, 16, "fast_fd", 2), (900, 200, 40, "fast_alpha_fd", 3),
         (700, 100, 20, "fast_isvd", 2), (1300, 96, 200, "fast_fd", 2), (500, 48, 24, "alpha_fd", 2)]
for n, d, ell, v, P in cases:
    A = (rng.standard_normal((n, d)) * np.linspace(3, 0.1, d)).astype(np.float32)
    Ad = torch.from_numpy(A).cuda()
    sk = m.Sketcher(d, ell, v, n_shards=P)
    sk.append(Ad[: n // 2])
    sk.append(torch.from_numpy(A[n // 2:]).pin_memory())
    B, st = sk.sketch()
    e = m.cov_err(Ad, B)
    torch.cuda.synchronize()
    print(v, n, d, ell, P, "shrinks", st["n_shrinks"], "err", round(e["err"], 6), flush=True)
    sk.close()
print("sanitize case ok")
