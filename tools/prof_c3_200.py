"""c3 ell=200 (P_total=296) sketch for ncu captures of the fused N=398 eig kernel:
    ncu --set full -k regex:eig_kernel -s <skip> -c 1 python tools/prof_c3_200.py"""
import sys
import torch
sys.path.insert(0, '.')
import fdgen
import paper_1501_06561_b200 as m

w = fdgen.config("c3")
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda")
fdgen.DeviceGenerator(w).fill(A)
sk = m.Sketcher(w.d, 200, "fast_fd", n_shards=296)
sk.append(A)
B, st = sk.sketch()
torch.cuda.synchronize()
print("ok", st["n_shrinks"])
