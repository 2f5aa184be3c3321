import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle, paper_1501_06561_b200 as m
np.set_printoptions(precision=5, linewidth=150)
rng = np.random.default_rng(0)
for ell, d, variant in [(4, 8, "fd"), (4, 8, "fast_fd"), (16, 64, "fd")]:
    A = (rng.standard_normal((200, d)) * np.linspace(2, 0.2, d)).astype(np.float32)
    for n in list(range(ell, ell + 8)) + [3 * ell, 100, 200]:
        sk = m.Sketcher(d, ell, variant)
        sk.append(torch.from_numpy(A[:n]).cuda())
        B, st = sk.sketch()
        Bg = B.cpu().numpy().astype(np.float64)
        r = oracle.sketch(A[:n], ell, variant)
        diff = np.abs(Bg.T @ Bg - r.B.T @ r.B).max() / r.frob_sq
        print(f"ell={ell} {variant} n={n}: diff {diff:.2e} delta {st['delta_total']:.5g}/{r.delta_total:.5g} shrinks {st['n_shrinks']}/{r.n_shrinks} frob {st['frob_sq']:.5g}/{r.frob_sq:.5g}")
        if diff > 1e-5:
            print("  sv gpu", np.linalg.svd(Bg, compute_uv=False)[:6]); print("  sv ora", np.linalg.svd(r.B, compute_uv=False)[:6])
            break
