"""Phase clocks of trd_kernel (CTA 0, FD_DEBUG_EIG): P1 (update+publish), P3 (reflector+SYMV), P4 (reduce)."""
import os, sys, ctypes, torch
os.environ["FD_DEBUG_EIG"] = "1"
sys.path.insert(0, '.')
import fdgen, paper_1501_06561_b200 as m
L = m._lib.lib()
L.fd_debug_eig_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
w = fdgen.config("c4", n=148 * 8 * 1000)
gen = fdgen.DeviceGenerator(w)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda"); gen.fill(A)
sk = m.Sketcher(w.d, 128, "fast_fd", n_shards=1184)
sk.append(A)
tr = (ctypes.c_longlong * 32)()
L.fd_debug_eig_trace(sk.h, tr)
t = list(tr)
steps = max(t[14], 1)
print("steps", steps, {"P1": t[11] / steps, "P3": t[12] / steps, "P4": t[13] / steps}, "cycles per step")
q = steps / 4
print("cycles per step by i range [0,64) [64,128) [128,192) [192,254):", [round(t[20 + k] / q) for k in range(4)])
