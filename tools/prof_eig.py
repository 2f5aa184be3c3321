import sys, torch
sys.path.insert(0, '.')
import fdgen, paper_1501_06561_b200 as m
w = fdgen.config("c4", n=148 * 1500)
gen = fdgen.DeviceGenerator(w)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda"); gen.fill(A)
sk = m.Sketcher(w.d, 128, "fast_fd", n_shards=148)
sk.append(A); B, st = sk.sketch(); torch.cuda.synchronize(); print("ok", st["n_shrinks"])
