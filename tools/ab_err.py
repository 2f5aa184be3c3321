"""A/B of GEMM paths: sketch diff and cov-err deviation vs the oracle (c1, c2)."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import fdgen, oracle, paper_1501_06561_b200 as m
cases = [("c1", 16, "fast_fd"), ("c2", 40, "fast_fd"), ("c2", 100, "fast_fd"), ("c2", 100, "fast_alpha_fd"), ("c2", 20, "fd")]
data = {c: fdgen.host_rows(fdgen.config(c)) for c in ("c1", "c2")}
for cfg, ell, v in cases:
    A = data[cfg]
    r = oracle.sketch(A, ell, v)
    eo = oracle.cov_err(A, r.B)["err"]
    sk = m.Sketcher(A.shape[1], ell, v)
    Ad = torch.from_numpy(A).cuda()
    sk.append(Ad); B, st = sk.sketch()
    Bg = B.cpu().numpy().astype(np.float64)
    D = Bg.T @ Bg - r.B.T @ r.B
    w = np.linalg.eigvalsh((D + D.T) / 2)
    eg = m.cov_err(Ad, B)["err"]
    led = (st["frob_sq"] - (Bg ** 2).sum() - st["removed_mass"]) / r.frob_sq
    print(f"{os.environ.get('TAG','')} {cfg} ell={ell} {v}: diff {max(abs(w[0]), abs(w[-1]))/r.frob_sq:.2e}  err_rel {(eg-eo)/eo:+.2e}  ledger {led:+.2e}", flush=True)
    sk.close()
