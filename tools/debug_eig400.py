"""Phase clocks of the fused eig_kernel (CTA 0, FD_DEBUG_EIG) on c3-shaped problems (N = 2 ell)."""
import os, sys, ctypes, torch
os.environ["FD_DEBUG_EIG"] = "1"
sys.path.insert(0, '.')
import fdgen, paper_1501_06561_b200 as m
L = m._lib.lib()
L.fd_debug_eig_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
w = fdgen.config("c3")
gen = fdgen.DeviceGenerator(w)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda"); gen.fill(A)
for ell, P in [(200, 296), (100, 296)]:
    sk = m.Sketcher(w.d, ell, "fast_fd", n_shards=P)
    sk.profile(True)
    sk.append(A)
    sk.sketch(stats=False)
    torch.cuda.synchronize()
    tr = (ctypes.c_longlong * 32)()
    L.fd_debug_eig_trace(sk.h, tr)
    prof = sk.profile_read()
    t = list(tr)
    names = ["load", "tridiag", "bisect", "rule+clusters", "invit", "backtransform"]
    cnt = max(t[10], 1)
    ph = {names[i]: t[i + 1] / cnt for i in range(6)}
    print(ell, "N", t[9], "problems(block0)", t[10], "avg clusters", t[7] / cnt, "max cluster", t[8],
          {k: f"{v/1.9e3:.1f}us" for k, v in ph.items()}, flush=True)
    print("   per kernel ms:", {k: (round(v[0], 2), v[1]) for k, v in prof.items()}, flush=True)
    sk.close()
