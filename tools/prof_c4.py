"""One c4 bench step (P = 1184 shard streams, fast_fd, ell = 128) for ncu captures:
    ncu --set full -k regex:<kernel> -s <skip> -c 1 python tools/prof_c4.py"""
import sys
import torch
sys.path.insert(0, '.')
import fdgen
import paper_1501_06561_b200 as m

w = fdgen.config("c4")
gen = fdgen.DeviceGenerator(w)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda")
gen.fill(A)
sk = m.Sketcher(w.d, 128, "fast_fd", n_shards=2368)
sk.append(A)
B, st = sk.sketch()
torch.cuda.synchronize()
print("ok", st["n_shrinks"])
