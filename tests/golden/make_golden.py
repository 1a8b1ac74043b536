"""Generate golden fixtures by running the REFERENCE package (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Everything is produced by the reference's own
public API (sldg_vlasov), seeded with np.random.default_rng; the fixtures pin
both the oracle (oracle/sldg_oracle.py) and the CUDA path.  /root/reference
does not exist on the GPU box, so only the .npz files travel.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

import sldg_vlasov as sv  # noqa: E402
from sldg_vlasov import driver as drv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def basis_and_1d():
    out = {}
    rng = np.random.default_rng(2024)
    for p in range(1, 6):
        b = sv.DGBasis(p)
        out[f"p{p}_nodes"] = b.nodes
        out[f"p{p}_weights"] = b.weights
        out[f"p{p}_gauss_nodes"] = b.gauss_nodes
        out[f"p{p}_gauss_weights"] = b.gauss_weights
        out[f"p{p}_mass_inv"] = b.mass_inv
        out[f"p{p}_diff"] = b.diff
        fr = np.concatenate([[0.0, 0.5, 1e-17, float(np.nextafter(1.0, 0.0)) - 1e-16],
                             rng.random(6)])
        fr = fr[(fr >= 0) & (fr < 1)]
        out[f"p{p}_fracs"] = fr
        out[f"p{p}_A"] = np.array([sv.overlap_pair(b, a).same for a in fr])
        out[f"p{p}_B"] = np.array([sv.overlap_pair(b, a).neighbor for a in fr])
    # decompose_shift incl. the one-ulp fold and negative speeds
    sp = np.concatenate([rng.uniform(-50, 50, 40), [0.0, -0.25, 2.3, 6.0, -6.0]])
    dt = np.concatenate([rng.uniform(1e-3, 2.0, 40), [1.0, 1.0, 1.0, 1.0, 1.0]])
    w = np.concatenate([rng.uniform(1e-3, 3.0, 40), [1.0, 1.0, 1.0, 1.0, 1.0]])
    # fold case: ratio just below an integer by < 1 ulp
    sp = np.append(sp, float(np.nextafter(3.0, 0.0)))
    dt = np.append(dt, 1.0)
    w = np.append(w, 1.0)
    ds = [sv.decompose_shift(a, b_, c) for a, b_, c in zip(sp, dt, w)]
    out["shift_speed"], out["shift_dt"], out["shift_width"] = sp, dt, w
    out["shift_n"] = np.array([d.n_shift for d in ds], dtype=np.int64)
    out["shift_frac"] = np.array([d.frac for d in ds])
    # apply_update on random pencils, both bcs, large shifts
    cases = []
    for k in range(24):
        p = int(rng.integers(1, 6))
        n = int(rng.integers(3, 9))
        b = sv.DGBasis(p)
        vals = rng.standard_normal((2, n, p + 1))
        disp = float(rng.uniform(-2.5 * n, 2.5 * n))
        bc = "periodic" if k % 3 else "absorbing"
        d = sv.decompose_shift(disp, 1.0, 1.0)
        res = sv.apply_update(vals, d, sv.overlap_pair(b, d.frac), bc)
        out[f"upd{k}_p"] = np.array(p)
        out[f"upd{k}_bc"] = np.array(bc)
        out[f"upd{k}_disp"] = np.array(disp)
        out[f"upd{k}_vals"] = vals
        out[f"upd{k}_out"] = res
        cases.append(k)
    out["n_upd"] = np.array(len(cases))
    save("basis_1d.npz", **out)


MESHES = [(3, 4, 0), (3, 4, 1), (3, 4, 2), (3, 3, 1), (3, 3, 2), (1, 16, 0), (3, 6, 1),
          (3, 5, 2)]


def meshes_and_plans():
    out = {}
    for dim, nb, lv in MESHES:
        tag = f"d{dim}_b{nb}_l{lv}"
        m = sv.build_mesh(dim, nb, lv, 6.0)
        out[f"{tag}_levels"] = m.levels
        out[f"{tag}_lo"] = m.lo
        out[f"{tag}_width"] = m.width
        for bc in ("absorbing", "periodic"):
            for d in range(dim):
                ps = sv.classify_conforming(sv.extract_pencils(m, d), m, bc)
                k = f"{tag}_{bc}_dir{d}"
                out[f"{k}_offsets"] = ps.offsets
                out[f"{k}_cell_ids"] = ps.cell_ids
                out[f"{k}_weights"] = ps.weights
                out[f"{k}_conforming"] = ps.conforming
                if d == 0:
                    for p in (1, 2, 3):
                        b = sv.DGBasis(p)
                        perm = sv.build_permutation(b, dim)
                        plan = sv.build_sweep_plan(m, ps, perm, b)
                        kk = f"{k}_p{p}"
                        out[f"{kk}_n_groups"] = np.array(len(plan.groups))
                        out[f"{kk}_layout"] = np.array([(g.n_lines, g.n_cells)
                                                        for g in plan.groups])
                        out[f"{kk}_gather"] = np.concatenate([g.gather.ravel()
                                                              for g in plan.groups])
                        out[f"{kk}_simple"] = np.array([g.simple for g in plan.groups])
    save("meshes_plans.npz", **out)


def sweeps():
    """advect_velocity on small AMR/uniform plans, hybrid and forced-slow."""
    out = {}
    rng = np.random.default_rng(1002)
    cases = [(3, 4, 1, 3), (3, 4, 2, 3), (3, 4, 1, 2), (3, 3, 1, 2), (1, 16, 0, 3),
             (3, 3, 2, 1)]
    idx = 0
    for dim, nb, lv, p in cases:
        m = sv.build_mesh(dim, nb, lv, 6.0)
        b = sv.DGBasis(p)
        perm = sv.build_permutation(b, dim)
        for bc in ("absorbing", "periodic"):
            ps = sv.classify_conforming(sv.extract_pencils(m, 0), m, bc)
            plan = sv.build_sweep_plan(m, ps, perm, b)
            ncol = 2
            seed = 1000 + idx
            # inputs are regenerated from the seed by the tests (not stored)
            f = np.random.default_rng(seed).standard_normal((plan.n_dofs, ncol))
            speeds = rng.uniform(-1.5, 1.5, size=ncol)
            speeds[1] *= 20.0   # large shift: exercises wrap / multi-cell feet
            dt = 0.1
            for fs in (False, True):
                g = f.copy()
                sv.advect_velocity(g, speeds, dt, plan, bc=bc, force_slow=fs)
                k = f"s{idx}"
                out[f"{k}_cfg"] = np.array([dim, nb, lv, p, int(fs)])
                out[f"{k}_bc"] = np.array(bc)
                out[f"{k}_seed"] = np.array(seed)
                out[f"{k}_speeds"] = speeds
                out[f"{k}_dt"] = np.array(dt)
                out[f"{k}_out"] = g
                idx += 1
    # one pencil-level case from test_vsweep (_amr_pencil), random speeds
    out["n_cases"] = np.array(idx)
    save("sweeps.npz", **out)


def xside():
    out = {}
    rng = np.random.default_rng(77)
    L = 4.0 * np.pi
    for nx in (16, 64):
        xg = sv.XGrid(nx, 2, L)
        speeds = np.concatenate([rng.uniform(-6, 6, 10), [0.0, 3.0 * xg.h / 0.05]])
        f = rng.standard_normal((len(speeds), xg.n_dofs))
        plan = sv.precompute_x_matrices(xg, speeds, 0.05)
        g = f.copy()
        sv.advect_x(g, plan)
        out[f"nx{nx}_speeds"] = speeds
        out[f"nx{nx}_f"] = f
        out[f"nx{nx}_out"] = g
        ps = sv.PoissonSolver(xg)
        x = xg.dof_coords
        rho = 1.0 + 0.05 * np.sin(0.5 * x) + 0.02 * np.cos(1.5 * x) + 1e-3 * rng.random(x.size)
        phi = ps.solve(rho)
        out[f"nx{nx}_rho"] = rho
        out[f"nx{nx}_phi"] = phi
        out[f"nx{nx}_E"] = ps.electric_field(phi)
        vw = rng.random(50)
        ff = rng.standard_normal((50, xg.n_dofs))
        out[f"nx{nx}_vw"] = vw
        out[f"nx{nx}_ff"] = ff
        out[f"nx{nx}_rho_of_ff"] = sv.compute_rho(ff, vw)
    save("xside.npz", **out)


def poisson_large():
    """Poisson solve + E at the x resolutions of configs 4 and 5 (N_x = 128, 256, 512): the
    device path applies the leading block of the augmented system's inverse, the reference
    LU (xfield.py:146,163); both are ~3e-13 from the exact solution of the discrete system
    at N_x = 512."""
    out = {}
    rng = np.random.default_rng(512)
    for nx in (128, 256, 512):
        xg = sv.XGrid(nx, 2, 4.0 * np.pi)
        ps = sv.PoissonSolver(xg)
        x = xg.dof_coords
        for k, eps in enumerate((0.01, 0.3)):
            rho = 1.0 + eps * np.cos(0.5 * x) + 0.02 * np.sin(1.5 * x) + 1e-4 * rng.random(x.size)
            phi = ps.solve(rho)
            out[f"nx{nx}_{k}_rho"] = rho
            out[f"nx{nx}_{k}_phi"] = phi
            out[f"nx{nx}_{k}_E"] = ps.electric_field(phi)
    save("poisson.npz", **out)


def simulations():
    """Short Strang runs: diagnostics per step + sampled coefficients."""
    out = {}
    rng = np.random.default_rng(5)
    cfgs = {
        "cfg1": dict(dim=3, n_base=16, levels=0, degree=1, n_x=16, n_steps=3),
        "cfg3": dict(dim=3, n_base=4, levels=1, degree=2, n_x=64, n_steps=5),
        "cfg4": dict(dim=3, n_base=4, levels=2, degree=3, n_x=128, n_steps=3),
        "q3l1p": dict(dim=3, n_base=4, levels=1, degree=3, n_x=16, n_steps=4, bc="periodic"),
        "v1": dict(dim=1, n_base=16, levels=0, degree=2, n_x=16, n_steps=5),
    }
    for name, kw in cfgs.items():
        cfg = drv.SimConfig(**kw)
        sim = drv.Simulation(cfg)
        recs = [sim.diagnostics(sim.field_solve())]
        for _ in range(cfg.n_steps):
            recs.append(sim.step())
        arr = np.array([[r.t, r.e_max, r.m0, r.m1, r.m2, r.e_field, r.e_total] for r in recs])
        n = sim.f.size
        sample = np.sort(rng.choice(n, size=min(4000, n), replace=False))
        out[f"{name}_records"] = arr
        out[f"{name}_sample_idx"] = sample
        out[f"{name}_sample_val"] = sim.f.ravel()[sample]
        out[f"{name}_fmax"] = np.array(np.abs(sim.f).max())
        out[f"{name}_colsum"] = sim.f.sum(axis=0)
        out[f"{name}_rowsum"] = sim.f.sum(axis=1)
    save("simulations.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["basis", "meshes", "sweeps", "x", "poisson", "sim"]
    if "basis" in which:
        basis_and_1d()
    if "meshes" in which:
        meshes_and_plans()
    if "sweeps" in which:
        sweeps()
    if "x" in which:
        xside()
    if "poisson" in which:
        poisson_large()
    if "sim" in which:
        simulations()
