"""Pin the CPU oracle (oracle/sldg_oracle.py) against the reference's golden vectors.

The fixtures in tests/golden/ were produced by the reference package itself
(tests/golden/make_golden.py).  CPU only.
"""
import numpy as np
import pytest

from oracle import sldg_oracle as so


def test_basis_constants(golden):
    g = golden("basis_1d.npz")
    for p in range(1, 6):
        b = so.Basis(p)
        np.testing.assert_allclose(b.nodes, g[f"p{p}_nodes"], atol=1e-15, rtol=0)
        np.testing.assert_allclose(b.weights, g[f"p{p}_weights"], atol=1e-15, rtol=0)
        np.testing.assert_array_equal(b.gq, g[f"p{p}_gauss_nodes"])
        np.testing.assert_allclose(b.mass_inv, g[f"p{p}_mass_inv"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(b.diff, g[f"p{p}_diff"], rtol=1e-13, atol=1e-13)


def test_overlap_pairs(golden):
    g = golden("basis_1d.npz")
    for p in range(1, 6):
        b = so.Basis(p)
        for k, a in enumerate(g[f"p{p}_fracs"]):
            A, B = so.overlap_mats(b, float(a))
            np.testing.assert_allclose(A, g[f"p{p}_A"][k], atol=1e-13, rtol=0)
            np.testing.assert_allclose(B, g[f"p{p}_B"][k], atol=1e-13, rtol=0)


def test_split_shift_bit_exact(golden):
    g = golden("basis_1d.npz")
    for s, d, w, n, fr in zip(g["shift_speed"], g["shift_dt"], g["shift_width"],
                              g["shift_n"], g["shift_frac"]):
        nn, ff = so.split_shift(float(s), float(d), float(w))
        assert nn == n and ff == fr


def test_uniform_update(golden):
    g = golden("basis_1d.npz")
    for k in range(int(g["n_upd"])):
        p = int(g[f"upd{k}_p"])
        b = so.Basis(p)
        n, a = so.split_shift(float(g[f"upd{k}_disp"]), 1.0, 1.0)
        A, B = so.overlap_mats(b, a)
        out = so.uniform_update(g[f"upd{k}_vals"], n, A, B, str(g[f"upd{k}_bc"]))
        np.testing.assert_allclose(out, g[f"upd{k}_out"], atol=1e-13, rtol=0)


def test_brute_projection_matches_update():
    rng = np.random.default_rng(5)
    for _ in range(10):
        p = int(rng.integers(1, 5))
        n = int(rng.integers(3, 7))
        b = so.Basis(p)
        u = rng.standard_normal((n, p + 1))
        disp = rng.uniform(-2.0 * n, 2.0 * n)
        bc = so.PERIODIC if rng.random() < 0.6 else so.ABSORBING
        ns, a = so.split_shift(disp, 1.0, 1.0)
        A, B = so.overlap_mats(b, a)
        got = so.uniform_update(u, ns, A, B, bc)
        assert np.abs(got - so.brute_projection(u, disp, 1.0, b, bc)).max() <= 1e-12


MESHES = [(3, 4, 0), (3, 4, 1), (3, 4, 2), (3, 3, 1), (3, 3, 2), (1, 16, 0), (3, 6, 1),
          (3, 5, 2)]


@pytest.mark.parametrize("dim,nb,lv", MESHES)
def test_mesh_pencils_plans(golden, dim, nb, lv):
    g = golden("meshes_plans.npz")
    tag = f"d{dim}_b{nb}_l{lv}"
    m = so.make_mesh(dim, nb, lv, 6.0)
    np.testing.assert_array_equal(m.levels, g[f"{tag}_levels"])
    np.testing.assert_array_equal(m.lo, g[f"{tag}_lo"])
    np.testing.assert_array_equal(m.width, g[f"{tag}_width"])
    for bc in ("absorbing", "periodic"):
        for d in range(dim):
            k = f"{tag}_{bc}_dir{d}"
            ps = so.mark_conforming(so.make_pencils(m, d), bc)
            np.testing.assert_array_equal(ps.offsets, g[f"{k}_offsets"])
            np.testing.assert_array_equal(ps.cell_ids, g[f"{k}_cell_ids"])
            np.testing.assert_array_equal(ps.weights, g[f"{k}_weights"])
            np.testing.assert_array_equal(ps.conforming, g[f"{k}_conforming"])
            if d == 0:
                for p in (1, 2, 3):
                    plan = so.make_plan(m, ps, p)
                    kk = f"{k}_p{p}"
                    assert len(plan.groups) == int(g[f"{kk}_n_groups"])
                    lay = np.array([(gr.n_lines, gr.n_cells) for gr in plan.groups])
                    np.testing.assert_array_equal(lay, g[f"{kk}_layout"])
                    np.testing.assert_array_equal(
                        np.concatenate([gr.gather.ravel() for gr in plan.groups]),
                        g[f"{kk}_gather"])


def _sweep_case(g, i):
    k = f"s{i}"
    dim, nb, lv, p, fs = [int(v) for v in g[f"{k}_cfg"]]
    bc = str(g[f"{k}_bc"])
    m = so.make_mesh(dim, nb, lv, 6.0)
    plan = so.make_plan(m, so.mark_conforming(so.make_pencils(m, 0), bc), p)
    speeds = g[f"{k}_speeds"]
    f = np.random.default_rng(int(g[f"{k}_seed"])).standard_normal((plan.n_dofs, len(speeds)))
    return plan, f, speeds, float(g[f"{k}_dt"]), bc, bool(fs), g[f"{k}_out"]


def test_sweeps(golden):
    g = golden("sweeps.npz")
    for i in range(int(g["n_cases"])):
        plan, f, speeds, dt, bc, fs, ref = _sweep_case(g, i)
        so.advect_v(f, speeds, dt, plan, bc, fs)
        scale = np.abs(ref).max()
        assert np.abs(f - ref).max() <= 1e-13 * scale, f"case {i}"


def test_xside(golden):
    g = golden("xside.npz")
    for nx in (16, 64):
        xg = so.XGrid(nx, 2, 4.0 * np.pi)
        f = g[f"nx{nx}_f"].copy()
        so.advect_x(f, so.x_plan(xg, g[f"nx{nx}_speeds"], 0.05), nx)
        np.testing.assert_allclose(f, g[f"nx{nx}_out"], atol=1e-13, rtol=0)
        ps = so.Poisson(xg)
        phi = ps.solve(g[f"nx{nx}_rho"])
        np.testing.assert_allclose(phi, g[f"nx{nx}_phi"], atol=1e-14, rtol=0)
        np.testing.assert_allclose(ps.efield(phi), g[f"nx{nx}_E"], atol=1e-13, rtol=0)
        np.testing.assert_allclose(so.rho(g[f"nx{nx}_ff"], g[f"nx{nx}_vw"]),
                                   g[f"nx{nx}_rho_of_ff"], atol=1e-13, rtol=0)


SIMS = {
    "cfg1": dict(dim=3, n_base=16, levels=0, degree=1, n_x=16, n_steps=3),
    "cfg3": dict(dim=3, n_base=4, levels=1, degree=2, n_x=64, n_steps=5),
    "cfg4": dict(dim=3, n_base=4, levels=2, degree=3, n_x=128, n_steps=3),
    "q3l1p": dict(dim=3, n_base=4, levels=1, degree=3, n_x=16, n_steps=4, bc="periodic"),
    "v1": dict(dim=1, n_base=16, levels=0, degree=2, n_x=16, n_steps=5),
}

# records(0).e_max known answers from SURVEY.md §8(c) (reference run, IC only).
# rho - mean(rho) is ~1e-2 of rho, so the summation order of the N_v-term
# reduction alone moves E at the ~1e-12 relative level (the survey's numbers
# came from a differently threaded BLAS): compare at 1e-11.
EMAX0 = {"cfg1": 0.020255538263257728, "cfg3": 0.020064331750957558,
         "cfg4": 0.020015337693626376}


@pytest.mark.parametrize("name", list(SIMS))
def test_simulation(golden, name):
    g = golden("simulations.npz")
    kw = dict(SIMS[name])
    n_steps = kw.pop("n_steps")
    sim = so.Sim(**kw)
    recs = [sim.diagnostics(sim.field_solve())]
    for _ in range(n_steps):
        recs.append(sim.step())
    arr = np.array([[r[k] for k in ("t", "e_max", "m0", "m1", "m2", "e_field", "e_total")]
                    for r in recs])
    ref = g[f"{name}_records"]
    np.testing.assert_allclose(arr[:, [0, 2, 4, 6]], ref[:, [0, 2, 4, 6]], rtol=1e-12)
    assert np.abs(arr[:, 1] - ref[:, 1]).max() <= 1e-12 * ref[0, 1]
    assert np.abs(arr[:, 3] - ref[:, 3]).max() <= 1e-12 * abs(ref[:, 2]).max()
    fmax = float(g[f"{name}_fmax"])
    got = sim.f.ravel()[g[f"{name}_sample_idx"]]
    assert np.abs(got - g[f"{name}_sample_val"]).max() <= 1e-12 * fmax
    if name in EMAX0:
        assert abs(arr[0, 1] - EMAX0[name]) <= 1e-11 * EMAX0[name]


def test_fit_oracle():
    t = np.arange(0.0, 20.0 + 1e-12, 0.1)
    rate, npk = so.peak_run_fit(t, np.exp(-0.1533 * t) * np.abs(np.cos(1.4156 * t)))
    assert rate is not None and abs(rate + 0.1533) <= 1e-3
    rate, npk = so.peak_run_fit(t, np.exp(-0.2 * t))
    assert rate is None and npk < 2


def test_poisson_large_nx(golden):
    """N_x = 128 / 256 / 512 Poisson + E (configs 4 and 5) against the reference."""
    g = golden("poisson.npz")
    for nx in (128, 256, 512):
        ps = so.Poisson(so.XGrid(nx, 2, 4.0 * np.pi))
        for k in range(2):
            phi = ps.solve(g[f"nx{nx}_{k}_rho"])
            np.testing.assert_allclose(phi, g[f"nx{nx}_{k}_phi"], rtol=0,
                                       atol=1e-14 * np.abs(g[f"nx{nx}_{k}_phi"]).max())
            e = ps.efield(phi)
            np.testing.assert_allclose(e, g[f"nx{nx}_{k}_E"], rtol=0,
                                       atol=1e-14 * np.abs(g[f"nx{nx}_{k}_E"]).max())


def test_coefficient_goldens_consistent(golden):
    """The multi-step reference runs (coeffs_*.npz) carry the records of run_*.npz."""
    import os
    for name in ("cfg1", "cfg3", "cfg4", "cfg2"):
        path = os.path.join(os.path.dirname(__file__), "golden", f"coeffs_{name}.npz")
        if not os.path.exists(path):
            continue
        c = golden(f"coeffs_{name}.npz")
        r = golden(f"run_{name}.npz")
        np.testing.assert_allclose(c["records"][:, 2], r["records"][:, 2], rtol=1e-12)
        assert c["records"].shape == r["records"].shape


@pytest.mark.parametrize("nb,lv", [(4, 2), (3, 2), (5, 2), (4, 1)])
def test_area_weights_product_equals_oracle(nb, lv):
    """weights="area": the product's vectorised builder and the oracle's
    per-pencil scan give identical weights, and every cell's weights sum to one."""
    import paper_2603_19959_b200 as sv
    m = sv.build_mesh(3, nb, lv, 6.0)
    ps = sv.extract_pencils(m, 0, "area")
    om = so.make_mesh(3, nb, lv, 6.0)
    ops = so.make_pencils(om, 0, "area")
    np.testing.assert_array_equal(ps.cell_ids, ops.cell_ids)
    np.testing.assert_array_equal(ps.weights, ops.weights)
    tot = np.bincount(ps.cell_ids, weights=ps.weights)
    assert np.abs(tot - 1.0).max() <= 4.5e-16
    cnt = sv.extract_pencils(m, 0)
    np.testing.assert_array_equal(ps.weights == 1.0, cnt.weights == 1.0)
