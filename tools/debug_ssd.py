"""GPU vs oracle SSD on c2 prefixes (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import fdgen, oracle
import paper_1501_06561_b200 as m
A = fdgen.host_rows(fdgen.config("c2"))
def sn(M):
    w = np.linalg.eigvalsh((M + M.T) / 2); return max(abs(w[0]), abs(w[-1]))
for ell in (16, 20, 24):
    for n in (40, 200, 1000, 3000):
        An = A[:n]
        sk = m.Sketcher(An.shape[1], ell, "ssd")
        sk.append(torch.from_numpy(An).cuda())
        B, st = sk.sketch()
        Bg = B.cpu().numpy().astype(np.float64)
        sk.close()
        r = oracle.sketch(An, ell, "ssd")
        frob = r.frob_sq
        print(ell, n, "diff/frob %.3e" % (sn(Bg.T @ Bg - r.B.T @ r.B) / frob),
              "mass gpu %.6e ora %.6e" % (np.sum(Bg ** 2) / frob, np.sum(r.B ** 2) / frob),
              "delta gpu %.6e ora %.6e" % (st["delta_total"], r.delta_total), flush=True)
