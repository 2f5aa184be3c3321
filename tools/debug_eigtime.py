import os, sys, ctypes, numpy as np, torch
os.environ["FD_DEBUG_EIG"] = "1"
sys.path.insert(0, '.')
import fdgen, paper_1501_06561_b200 as m
L = m._lib.lib()
L.fd_debug_eig_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
w = fdgen.config("c4", n=int(sys.argv[1]) if len(sys.argv) > 1 else 148*7085)
gen = fdgen.DeviceGenerator(w)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda"); gen.fill(A)
for variant, ell, P in [("fast_fd", 128, 148), ("fast_fd", 64, 148), ("fd", 32, 148)]:
    sk = m.Sketcher(w.d, ell, variant, n_shards=P)
    sk.profile(True)
    sk.append(A[: P * 2000] if variant == "fd" else A)
    tr = (ctypes.c_longlong * 32)()
    L.fd_debug_eig_trace(sk.h, tr)
    prof = sk.profile_read()
    t = list(tr)
    names = ["load", "tridiag", "bisect", "rule+clusters", "invit", "backtransform"]
    cnt = max(t[10], 1)
    ph = {names[i]: t[i + 1] / cnt for i in range(6)}
    print(variant, ell, "N", t[9], "problems(block0)", t[10], "avg clusters", t[7] / cnt, "max cluster", t[8], {k: f"{v/1.9e3:.1f}us" for k, v in ph.items()})
    print("   invit sub-phases us (solves, small-cluster MGS, block CGS):", [round(t[i] / cnt / 1.9e3, 1) for i in (16, 17, 18)])
    print("   per kernel ms:", {k: (round(v[0], 2), v[1]) for k, v in prof.items()})
    sk.close()
