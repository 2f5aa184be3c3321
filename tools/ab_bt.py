"""A/B of the back-transform: tcgen05 bt_tc_kernel (default) vs FP32 SIMT bt_kernel (FD_SIMT_BT):
sketch difference ||B1^T B1 - B2^T B2||_2 / ||A||_F^2 and cov-err on c4-shaped data, plus a c2 case vs the oracle."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import fdgen, oracle, paper_1501_06561_b200 as m

def run(A, ell, v, P, simt):
    if simt: os.environ["FD_SIMT_BT"] = "1"
    else: os.environ.pop("FD_SIMT_BT", None)
    sk = m.Sketcher(A.shape[1], ell, v, n_shards=P)
    sk.profile(True)
    sk.append(A)
    B, st = sk.sketch()
    prof = sk.profile_read()
    sk.close()
    return B, st, prof

w = fdgen.config("c4", n=2368 * 600)
A = torch.empty((w.n, w.d), dtype=torch.float32, device="cuda"); fdgen.DeviceGenerator(w).fill(A)
for v in ("fast_fd", "fast_alpha_fd"):
    B1, s1, p1 = run(A, 128, v, 2368, False)
    B2, s2, p2 = run(A, 128, v, 2368, True)
    b1 = B1.double().cpu().numpy(); b2 = B2.double().cpu().numpy()
    D = b1.T @ b1 - b2.T @ b2
    ev = np.linalg.eigvalsh((D + D.T) / 2)
    e1 = m.cov_err(A, B1)["err"]; e2 = m.cov_err(A, B2)["err"]
    print(f"c4 n={w.n} {v}: sketch diff {max(abs(ev[0]), abs(ev[-1])) / s1['frob_sq']:.2e}, err tc {e1:.6e} simt {e2:.6e} rel {(e1-e2)/e2:+.2e}; "
          f"bt ms tc {p1['bt'][0]:.2f} simt {p2['bt'][0]:.2f}", flush=True)
Ah = fdgen.host_rows(fdgen.config("c2"))
Ad = torch.from_numpy(Ah).cuda()
for ell in (40, 100):
    r = oracle.sketch(Ah, ell, "fast_fd")
    eo = oracle.cov_err(Ah, r.B)["err"]
    for simt in (False, True):
        B, st, _ = run(Ad, ell, "fast_fd", 1, simt)
        Bg = B.cpu().numpy().astype(np.float64)
        D = Bg.T @ Bg - r.B.T @ r.B
        ev = np.linalg.eigvalsh((D + D.T) / 2)
        eg = m.cov_err(Ad, B)["err"]
        print(f"c2 ell={ell} {'simt' if simt else 'tc  '}: diff {max(abs(ev[0]), abs(ev[-1])) / r.frob_sq:.2e} err_rel {(eg - eo) / eo:+.2e}", flush=True)
