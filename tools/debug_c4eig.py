"""Phase times + cluster statistics of the eig kernel (CTA 0) on the bench config."""
import os, sys, ctypes, torch
os.environ["FD_DEBUG_EIG"] = "1"
sys.path.insert(0, '.')
import fdgen, paper_1501_06561_b200 as m
L = m._lib.lib()
L.fd_debug_eig_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
P = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
w = fdgen.config("c4")
gen = fdgen.DeviceGenerator(w)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda"); gen.fill(A)
sk = m.Sketcher(w.d, 128, "fast_fd", n_shards=P)
sk.profile(True)
sk.append(A)
tr = (ctypes.c_longlong * 32)()
L.fd_debug_eig_trace(sk.h, tr)
prof = sk.profile_read()
t = list(tr)
names = ["load", "tridiag", "bisect", "rule+clusters", "invit", "backtransform"]
cnt = max(t[10], 1)
print("P", P, "N", t[9], "problems(block0)", cnt, "avg clusters", t[7] / cnt, "max cluster", t[8],
      {names[i]: f"{t[i + 1] / cnt / 1.965e3:.1f}us" for i in range(6)})
print("per kernel ms:", {k: (round(v[0], 2), v[1]) for k, v in prof.items()})
print("invit sub-phases us/problem: solves %.1f warpMGS %.1f blockCGS %.1f" % tuple(t[k] / cnt / 1.965e3 for k in (16, 17, 18)))
