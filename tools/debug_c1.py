import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle, fdgen, paper_1501_06561_b200 as m
np.set_printoptions(precision=6, linewidth=160)
A = fdgen.host_rows(fdgen.config("c1"))
ell, d, variant = 16, 64, sys.argv[1] if len(sys.argv) > 1 else "fd"
def diff_at(n):
    sk = m.Sketcher(d, ell, variant)
    sk.append(torch.from_numpy(A[:n]).cuda())
    B, st = sk.sketch()
    Bg = B.cpu().numpy().astype(np.float64)
    r = oracle.sketch(A[:n], ell, variant)
    return np.abs(Bg.T @ Bg - r.B.T @ r.B).max() / r.frob_sq, Bg, r, st
for n in [20, 50, 100, 200, 400, 800, 1200, 1600, 2000]:
    dd, Bg, r, st = diff_at(n)
    print(n, f"{dd:.2e}", st['delta_total'], r.delta_total)
lo, hi = 16, 2000
while hi - lo > 1:
    mid = (lo + hi) // 2
    if diff_at(mid)[0] > 1e-5: hi = mid
    else: lo = mid
print("first bad n", hi)
dd, Bg, r, st = diff_at(hi)
print("gpu sv", np.linalg.svd(Bg, compute_uv=False))
print("ora sv", np.linalg.svd(r.B, compute_uv=False))
dd0, Bg0, r0, st0 = diff_at(hi - 1)
print("prev ora sv", np.linalg.svd(r0.B, compute_uv=False))
# the buffer Gram at the failing step = [B_prev (ell-1 rows); a_n]
Bf = np.vstack([r0.B[:ell-1], A[hi-1:hi].astype(np.float64)])
w = np.linalg.eigvalsh(Bf @ Bf.T)[::-1]
print("eig of failing Gram", w)
np.save("gpurun_out/c1_fail_gram.npy", Bf)
