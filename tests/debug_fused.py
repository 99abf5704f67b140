"""Debug helper (GPU): compare fused solve_apply with optimize_field + apply_field."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_09582_b200 as glu
g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "glu_golden.npz"))
img = g["mix67x45_s4/high"]
high = torch.from_numpy(img).cuda()
low, grid = glu.grid_downsample(high, 4)
for mode in (glu.Mode.Fast, glu.Mode.Exact, glu.Mode.Gnu):
    f = glu.optimize_field(high, low, grid, None, mode)
    a = glu.apply_field(f, low).cpu().numpy()
    b, pf = glu.solve_apply(high, low, grid, low, None, mode, keep_params=True)
    b = b.cpu().numpy()
    P = f.numpy(); P2 = pf.numpy()
    bad = np.argwhere((a != b).any(axis=2))
    print(mode, "params equal", P.tobytes() == P2.tobytes(), "mismatching px", len(bad))
    L = low.cpu().numpy().reshape(-1, 3)
    for (y, x) in bad[:5]:
        p = P[y, x]
        print(" ", y, x, p, "apply", a[y, x], "fused", b[y, x], "La", L[p["a"]], "Lb", L[p["b"]])
