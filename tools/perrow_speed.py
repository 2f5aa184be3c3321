"""Per-row kernel throughput (c1/c2/c5 per-row variants at P_total = 1): rows/s."""
import sys, time
import torch
sys.path.insert(0, ".")
import fdgen
import paper_1501_06561_b200 as fd

for cfg, ell, v in [("c1", 16, "fd"), ("c2", 20, "fd"), ("c2", 100, "fd"), ("c2", 100, "ssd"), ("c2", 100, "cfd"),
                    ("c5", 32, "fd"), ("c5", 32, "isvd")]:
    w = fdgen.config(cfg)
    A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda")
    fdgen.DeviceGenerator(w).fill(A, 0)
    sk = fd.Sketcher(w.d, ell, v, n_shards=1)
    sk.append(A); sk.sketch(); torch.cuda.synchronize()
    sk.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sk.append(A); B, st = sk.sketch(stats=False); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{cfg} ell={ell} {v}: {w.n / (ms / 1e3):.4g} rows/s ({ms:.1f} ms)", flush=True)
    sk.close()
