"""Per-row kernel phase clocks (CTA 0 of stream 0; FD_DEBUG_EIG=1): cycles per row per phase."""
import ctypes, os, sys
os.environ["FD_DEBUG_EIG"] = "1"
import torch
sys.path.insert(0, ".")
import fdgen
import paper_1501_06561_b200 as fd
L = fd.lib()
L.fd_debug_eig_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
names = ["partials", "cluster-sync1", "gather+cfd", "sort+deflate", "roots", "roots-sync+gather", "loewner+rule",
         "WtT+norms", "recon"]
for cfg, ell, v in [("c1", 16, "fd"), ("c2", 20, "fd"), ("c2", 100, "fd"), ("c5", 32, "fd")]:
    w = fdgen.config(cfg)
    n = min(w.n, 20000)
    A = torch.empty((n, w.d), dtype=torch.float32, device="cuda")
    fdgen.DeviceGenerator(w).fill(A, 0)
    sk = fd.Sketcher(w.d, ell, v, n_shards=1)
    sk.append(A)
    torch.cuda.synchronize()
    tr = (ctypes.c_longlong * 32)()
    L.fd_debug_eig_trace(sk.h, tr)
    rows = max(1, tr[9])
    tot = sum(tr[i] for i in range(9))
    print(f"{cfg} ell={ell} {v}: {tot / rows:.0f} cycles/row over {rows} rows; " +
          ", ".join(f"{names[i]} {tr[i] / rows:.0f}" for i in range(9)) +
          f"; warp-0 secular iterations/row {tr[10] / rows:.1f} (max {tr[11]}), K/row {tr[12] / rows:.1f}", flush=True)
    sk.close()
