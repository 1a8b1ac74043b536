"""Per-operator deviation of the CUDA path from the reference's golden vectors (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_19959_b200 as sv  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
g = np.load(os.path.join(G, "basis_1d.npz"))
for p in range(1, 6):
    b = sv.DGBasis(p)
    A, B = sv.sldg1d.overlap_pairs_device(b, g[f"p{p}_fracs"])
    print(f"overlap p{p}: max|dA| {np.abs(A - g[f'p{p}_A']).max():.3e} "
          f"max|dB| {np.abs(B - g[f'p{p}_B']).max():.3e}  minv {np.abs(b.mass_inv - g[f'p{p}_mass_inv']).max():.3e}")
x = np.load(os.path.join(G, "xside.npz"))
for nx in (16, 64):
    xg = sv.XGrid(nx, 2, 4.0 * np.pi)
    plan = sv.precompute_x_matrices(xg, x[f"nx{nx}_speeds"], 0.05)
    fd = torch.from_numpy(x[f"nx{nx}_f"].copy()).cuda()
    sv.advect_x(fd, plan)
    ref = x[f"nx{nx}_out"]
    d = np.abs(fd.cpu().numpy() - ref)
    print(f"advect_x nx{nx}: max abs {d.max():.3e}  max rel-to-row-max "
          f"{(d.max(axis=1) / np.abs(ref).max(axis=1)).max():.3e}")
s = np.load(os.path.join(G, "sweeps.npz"))
for k in range(int(s["n_cases"])):
    dim, nb, lv, p, fs = (int(v) for v in s[f"s{k}_cfg"])
    bc = str(s[f"s{k}_bc"])
    m = sv.build_mesh(dim, nb, lv, 6.0)
    b = sv.DGBasis(p)
    plan = sv.build_sweep_plan(m, sv.classify_conforming(sv.extract_pencils(m, 0), m, bc),
                               sv.build_permutation(b, dim), b)
    f = np.random.default_rng(int(s[f"s{k}_seed"])).standard_normal((plan.n_dofs, 2))
    fd = torch.from_numpy(f).cuda()
    sv.advect_velocity(fd, s[f"s{k}_speeds"], float(s[f"s{k}_dt"]), plan, bc=bc, force_slow=bool(fs))
    ref = s[f"s{k}_out"]
    d = np.abs(fd.cpu().numpy() - ref)
    print(f"advect_v case {k} d{dim} b{nb} l{lv} p{p} {bc} slow={fs}: max abs {d.max():.3e} "
          f"rel {d.max() / np.abs(ref).max():.3e}")
