"""Diagnostic: one ReduceRank (batched, n = 2*ell rows) GPU vs oracle, several sizes."""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle, paper_1501_06561_b200 as m
np.set_printoptions(precision=5, linewidth=150)
for ell, d, variant, nrows in [(2, 4, "fd", 2), (4, 8, "fd", 4), (4, 8, "fast_fd", 8), (8, 16, "fast_fd", 16), (16, 64, "fd", 16), (32, 64, "fast_fd", 64), (128, 300, "fast_fd", 256)]:
    rng = np.random.default_rng(ell)
    A = (rng.standard_normal((nrows, d)) * np.linspace(2, 0.2, d)).astype(np.float32)
    sk = m.Sketcher(d, ell, variant)
    sk.append(torch.from_numpy(A).cuda())
    B, st = sk.sketch()
    Bg = B.cpu().numpy().astype(np.float64)
    r = oracle.sketch(A, ell, variant)
    sg = np.linalg.svd(Bg, compute_uv=False); so = np.linalg.svd(r.B, compute_uv=False)
    diff = np.abs(Bg.T @ Bg - r.B.T @ r.B).max() / r.frob_sq
    print(f"ell={ell} d={d} {variant} n={nrows}: maxdiff/frob={diff:.2e} delta gpu {st['delta_total']:.6g} ora {r.delta_total:.6g} removed {st['removed_mass']:.6g} {r.removed:.6g} shrinks {st['n_shrinks']} {r.n_shrinks}")
    if diff > 1e-5:
        print("  sv gpu", sg[:8]); print("  sv ora", so[:8])
        print("  row norms gpu", np.linalg.norm(Bg, axis=1)[:8])
        print("  gram offdiag max", np.abs(Bg @ Bg.T - np.diag(np.diag(Bg @ Bg.T))).max())
