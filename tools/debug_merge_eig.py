"""eig phase clocks (CTA 0) of the finalize + merge-tree launches of a c4 sketch."""
import os, sys, ctypes, torch
os.environ["FD_DEBUG_EIG"] = "1"
sys.path.insert(0, '.')
import fdgen, paper_1501_06561_b200 as m
L = m._lib.lib()
L.fd_debug_eig_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
P = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
w = fdgen.config("c4")
gen = fdgen.DeviceGenerator(w)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda"); gen.fill(A)
sk = m.Sketcher(w.d, 128, "fast_fd", n_shards=P)
sk.append(A)
t0 = (ctypes.c_longlong * 32)(); L.fd_debug_eig_trace(sk.h, t0)
sk.profile(True); sk.profile_read()
B, st = sk.sketch()
prof = sk.profile_read()
t1 = (ctypes.c_longlong * 32)(); L.fd_debug_eig_trace(sk.h, t1)
d = [a - b for a, b in zip(list(t1), list(t0))]
cnt = max(d[10], 1)
names = ["load", "tridiag", "bisect", "rule+clusters", "invit", "backtransform"]
print("sketch(): problems(block0)", cnt, "max cluster", t1[8], {names[i]: f"{d[i + 1] / cnt / 1.965e3:.1f}us" for i in range(6)})
print("invit sub-phases us/problem: solves %.1f warpMGS %.1f blockCGS %.1f" % tuple(d[k] / cnt / 1.965e3 for k in (16, 17, 18)))
print("sketch() per kernel ms:", {k: (round(v[0], 2), v[1]) for k, v in prof.items()})
