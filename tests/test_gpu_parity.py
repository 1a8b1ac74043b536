"""CUDA path vs the reference's golden vectors and the CPU oracle (needs a B200).

Tolerances: fp64 coefficients within 1e-12 relative to max|ref| (the
north-star bar); bitwise where the reference is bitwise (zero speeds, x
integer shifts, determinism).
"""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_19959_b200 as sv  # noqa: E402
from oracle import sldg_oracle as so  # noqa: E402

DEV = torch.device("cuda", 0)
TOL = 1e-12


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(DEV)


def plan_for(dim, nb, lv, p, bc):
    m = sv.build_mesh(dim, nb, lv, 6.0)
    b = sv.DGBasis(p)
    ps = sv.classify_conforming(sv.extract_pencils(m, 0), m, bc)
    return sv.build_sweep_plan(m, ps, sv.build_permutation(b, dim), b), m, b


def test_library_loaded_from_tree():
    from paper_2603_19959_b200 import _capi
    lib = _capi.lib()
    assert lib.sldg_version() >= 10000
    assert _capi.LIB_PATH.endswith("paper_2603_19959_b200/_lib/libsldg.so")


def test_overlap_pairs_golden(golden):
    g = golden("basis_1d.npz")
    for p in range(1, 6):
        b = sv.DGBasis(p)
        A, B = sv.sldg1d.overlap_pairs_device(b, g[f"p{p}_fracs"])
        np.testing.assert_allclose(A, g[f"p{p}_A"], atol=1e-13, rtol=0)
        np.testing.assert_allclose(B, g[f"p{p}_B"], atol=1e-13, rtol=0)
        # alpha == 0 is the exact identity pair
        z = np.nonzero(g[f"p{p}_fracs"] == 0.0)[0]
        assert np.array_equal(A[z[0]], np.eye(p + 1)) and not B[z[0]].any()


def test_level_matrices_match_host_split():
    b = sv.DGBasis(3)
    lm = sv.precompute_level_matrices(b, 0.5, 1.0, 1.0, 2)
    assert lm.n_shift[0] == 0 and abs(lm.frac[0] - 0.5) < 1e-15
    assert lm.n_shift[1] == 1 and lm.frac[1] == 0.0
    for p in range(1, 6):
        b = sv.DGBasis(p)
        lm = sv.precompute_level_matrices(b, 0.731, 0.1, 1.3, 3)
        for pair in lm.pairs:
            assert np.abs(b.weights @ (pair.same + pair.neighbor) - b.weights).max() < 1e-12


def test_device_split_shift_bit_exact(golden):
    """k_level_mats' decompose_shift equals Python's bit for bit (incl. the 1-ulp fold)."""
    import ctypes as C

    from paper_2603_19959_b200 import _capi
    g = golden("basis_1d.npz")
    plan, _, _ = plan_for(1, 4, 0, 1, "periodic")
    for s, d, w, n, fr in zip(g["shift_speed"], g["shift_dt"], g["shift_width"],
                              g["shift_n"], g["shift_frac"]):
        # width of level 0 is the plan's base width; rescale speed so speed*dt/width matches
        pl, _, _ = plan_for(1, 4, 0, 1, "periodic")
        pl.base_width = float(w)
        pl._dev = {}
        sp = dev([s])
        ns = torch.empty(1, dtype=torch.int64, device=DEV)
        fr_d = torch.empty(1, dtype=torch.float64, device=DEV)
        mats = torch.empty(2 * 4, dtype=torch.float64, device=DEV)
        _capi.check(_capi.lib().sldg_level_matrices(pl.device_handle(), sp.data_ptr(), 1,
                                                     float(d), ns.data_ptr(), fr_d.data_ptr(),
                                                     mats.data_ptr(), None))
        assert int(ns.item()) == int(n) and float(fr_d.item()) == float(fr)


SWEEP_CASES = list(range(24))


def _sweep_case(g, i):
    k = f"s{i}"
    dim, nb, lv, p, fs = [int(v) for v in g[f"{k}_cfg"]]
    bc = str(g[f"{k}_bc"])
    plan, _, _ = plan_for(dim, nb, lv, p, bc)
    speeds = g[f"{k}_speeds"]
    f = np.random.default_rng(int(g[f"{k}_seed"])).standard_normal((plan.n_dofs, len(speeds)))
    return plan, f, speeds, float(g[f"{k}_dt"]), bc, bool(fs), g[f"{k}_out"]


@pytest.mark.parametrize("case", SWEEP_CASES)
def test_advect_velocity_golden(golden, case):
    g = golden("sweeps.npz")
    if case >= int(g["n_cases"]):
        pytest.skip("no such case")
    plan, f, speeds, dt, bc, fs, ref = _sweep_case(g, case)
    fd = dev(f)
    out = sv.advect_velocity(fd, speeds, dt, plan, bc=bc, force_slow=fs)
    assert out is fd
    got = fd.cpu().numpy()
    assert np.abs(got - ref).max() <= TOL * np.abs(ref).max(), f"case {case}"
    # numpy in / numpy out path gives the same bits
    fh = f.copy()
    sv.advect_velocity(fh, speeds, dt, plan, bc=bc, force_slow=fs)
    assert np.array_equal(fh, got)


@pytest.mark.parametrize("bc", ["absorbing", "periodic"])
@pytest.mark.parametrize("dim,nb,lv,p", [(3, 4, 1, 3), (3, 4, 2, 3), (3, 3, 1, 2),
                                          (3, 5, 2, 2), (3, 8, 0, 2), (1, 16, 0, 4),
                                          (3, 4, 0, 5)])
def test_advect_velocity_vs_oracle(bc, dim, nb, lv, p):
    rng = np.random.default_rng(100 + nb * 10 + lv + p)
    plan, m, b = plan_for(dim, nb, lv, p, bc)
    om = so.make_mesh(dim, nb, lv, 6.0)
    oplan = so.make_plan(om, so.mark_conforming(so.make_pencils(om, 0), bc), p)
    ncol = 40
    f = rng.standard_normal((plan.n_dofs, ncol))
    speeds = rng.uniform(-1.5, 1.5, size=ncol)
    speeds[3] = 0.0
    speeds[5] *= 25.0
    speeds[7] = 0.021 / 0.1 * 0.5    # Landau-sized shift
    ref = so.advect_v(f.copy(), speeds, 0.1, oplan, bc)
    fd = dev(f)
    sv.advect_velocity(fd, speeds, 0.1, plan, bc=bc)
    got = fd.cpu().numpy()
    assert np.abs(got - ref).max() <= TOL * np.abs(ref).max()
    assert np.array_equal(got[:, 3], f[:, 3])        # zero speed: untouched bits
    refs = so.advect_v(f.copy(), speeds, 0.1, oplan, bc, force_slow=True)
    fs = dev(f)
    sv.advect_velocity(fs, speeds, 0.1, plan, bc=bc, force_slow=True)
    assert np.abs(fs.cpu().numpy() - refs).max() <= TOL * np.abs(refs).max()
    # hybrid == forced slow within 1e-12 (acceptance C2, vsweep.py tests 171-182)
    assert np.abs(got - fs.cpu().numpy()).max() <= 1e-12 * max(1.0, np.abs(f).max())


def test_advect_velocity_errors():
    plan, _, _ = plan_for(3, 4, 1, 3, "absorbing")
    f = torch.zeros((plan.n_dofs, 3), dtype=torch.float64, device=DEV)
    with pytest.raises(sv.SweepError):
        sv.advect_velocity(f, np.ones(4), 0.1, plan)
    with pytest.raises(ValueError):
        sv.advect_velocity(f, np.ones(3), 0.1, plan, bc="reflecting")
    before = f.clone()
    assert sv.advect_velocity(f, np.zeros(3), 0.1, plan) is f
    assert torch.equal(f, before)


def test_advect_velocity_deterministic_and_tile_invariant():
    """Bitwise run-to-run, and a column's result is independent of the other columns."""
    plan, _, _ = plan_for(3, 6, 1, 2, "absorbing")
    rng = np.random.default_rng(7)
    f = rng.standard_normal((plan.n_dofs, 96))
    sp = rng.uniform(-2.0, 2.0, 96) * 0.1
    a, b_ = dev(f), dev(f)
    sv.advect_velocity(a, sp, 0.1, plan)
    sv.advect_velocity(b_, sp, 0.1, plan)
    assert torch.equal(a, b_)
    sub = dev(f[:, 10:13])
    sv.advect_velocity(sub, sp[10:13], 0.1, plan)
    assert torch.equal(sub, a[:, 10:13])


def test_advect_velocity_mass_periodic():
    plan, m, b = plan_for(3, 4, 1, 3, "periodic")
    perm = sv.build_permutation(b, 3)
    w = sv.velocity_dof_weights(m, b, perm)
    rng = np.random.default_rng(61)
    f = rng.standard_normal((plan.n_dofs, 3))
    m0 = w @ f
    fd = dev(f)
    sv.advect_velocity(fd, np.array([0.31, -0.9, 0.02]), 0.1, plan, bc="periodic")
    m1 = w @ fd.cpu().numpy()
    assert np.abs((m1 - m0) / m0).max() <= 1e-12


def test_xside_golden(golden):
    g = golden("xside.npz")
    for nx in (16, 64):
        xg = sv.XGrid(nx, 2, 4.0 * np.pi)
        plan = sv.precompute_x_matrices(xg, g[f"nx{nx}_speeds"], 0.05)
        fd = dev(g[f"nx{nx}_f"])
        sv.advect_x(fd, plan)
        got = fd.cpu().numpy()
        np.testing.assert_allclose(got, g[f"nx{nx}_out"], atol=1e-13, rtol=0)
        # zero-speed row untouched; integer shift row an exact roll
        np.testing.assert_array_equal(got[-2], g[f"nx{nx}_f"][-2])
        np.testing.assert_array_equal(
            got[-1], np.roll(g[f"nx{nx}_f"][-1].reshape(nx, 3), 3, axis=0).ravel())
        ps = sv.PoissonSolver(xg)
        phi = ps.solve(dev(g[f"nx{nx}_rho"]))
        np.testing.assert_allclose(phi.cpu().numpy(), g[f"nx{nx}_phi"], atol=1e-13, rtol=0)
        e = ps.electric_field(phi)
        np.testing.assert_allclose(e.cpu().numpy(), g[f"nx{nx}_E"], atol=1e-12, rtol=0)
        r = sv.compute_rho(dev(g[f"nx{nx}_ff"]), g[f"nx{nx}_vw"])
        np.testing.assert_allclose(r.cpu().numpy(), g[f"nx{nx}_rho_of_ff"], atol=1e-13, rtol=0)


def test_advect_x_vs_oracle_large_shifts():
    rng = np.random.default_rng(3)
    for nx, p in ((16, 2), (64, 2), (32, 3), (8, 1)):
        xg = sv.XGrid(nx, p, 4.0 * np.pi)
        sp = np.concatenate([rng.uniform(-40, 40, 30), [0.0, 0.0, 1.0]])
        f = rng.standard_normal((len(sp), xg.n_dofs))
        ref = so.advect_x(f.copy(), so.x_plan(so.XGrid(nx, p, 4.0 * np.pi), sp, 0.05), nx)
        fd = dev(f)
        sv.advect_x(fd, sv.precompute_x_matrices(xg, sp, 0.05))
        assert np.abs(fd.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()


SIMS = {
    "cfg1": dict(dim=3, n_base=16, levels=0, degree=1, n_x=16, n_steps=3),
    "cfg3": dict(dim=3, n_base=4, levels=1, degree=2, n_x=64, n_steps=5),
    "cfg4": dict(dim=3, n_base=4, levels=2, degree=3, n_x=128, n_steps=3),
    "q3l1p": dict(dim=3, n_base=4, levels=1, degree=3, n_x=16, n_steps=4, bc="periodic"),
    "v1": dict(dim=1, n_base=16, levels=0, degree=2, n_x=16, n_steps=5),
}


@pytest.mark.parametrize("name", list(SIMS))
def test_simulation_golden(golden, name):
    g = golden("simulations.npz")
    kw = dict(SIMS[name])
    sim = sv.Simulation(sv.SimConfig(**kw))
    recs = [sim.diagnostics(sim.field_solve())]
    for _ in range(kw["n_steps"]):
        recs.append(sim.step())
    arr = np.array([[r.t, r.e_max, r.m0, r.m1, r.m2, r.e_field, r.e_total] for r in recs])
    ref = g[f"{name}_records"]
    np.testing.assert_allclose(arr[:, [0, 2, 4, 6]], ref[:, [0, 2, 4, 6]], rtol=1e-12)
    assert np.abs(arr[:, 1] - ref[:, 1]).max() <= 1e-10 * ref[0, 1]
    assert np.abs(arr[:, 3] - ref[:, 3]).max() <= 1e-12 * abs(ref[:, 2]).max()
    f = sim.f.cpu().numpy()
    fmax = float(g[f"{name}_fmax"])
    got = f.ravel()[g[f"{name}_sample_idx"]]
    assert np.abs(got - g[f"{name}_sample_val"]).max() <= TOL * fmax
    np.testing.assert_allclose(f.sum(axis=0), g[f"{name}_colsum"], rtol=1e-11)


@pytest.mark.parametrize("amr_fused", ["off", "on"])
def test_run_matches_step_loop(amr_fused, monkeypatch):
    """run() pipelines the steps (advance); the step loop does not.  With the separate
    passes the two are bit-identical; the one-pass AMR step composes X.X into one stencil
    (re-association only, ~1e-16 relative per step)."""
    monkeypatch.setenv("SLDG_AMR_FUSED", amr_fused)
    cfg = sv.SimConfig(dim=3, n_base=4, levels=1, degree=2, n_x=16, n_steps=6)
    res = sv.run(cfg)
    sim = sv.Simulation(cfg)
    recs = [sim.diagnostics(sim.field_solve())] + [sim.step() for _ in range(6)]
    for a, b_ in zip(res.records, recs):
        if amr_fused == "off":
            assert a == b_
        else:
            np.testing.assert_allclose(np.array(dataclasses.astuple(a)),
                                       np.array(dataclasses.astuple(b_)), rtol=1e-11, atol=1e-13)


def test_nonfinite_aborts_with_step_index():
    cfg = sv.SimConfig(dim=1, n_base=16, levels=0, degree=2, n_x=16, n_steps=2)
    sim = sv.Simulation(cfg)
    sim.f[:] = float("inf")
    with pytest.raises(RuntimeError, match="step 0"):
        sim.run()


def _small_sim(**kw):
    base = dict(dim=3, n_base=6, levels=1, degree=2, n_x=24, n_steps=4)
    base.update(kw)
    return sv.Simulation(sv.SimConfig(**base))


def test_fused_x_passes_bitwise():
    """XX == X;X bit for bit; fused rho/moments equal the standalone reductions to 1e-14."""
    from paper_2603_19959_b200.xfield import advect_x_fused_into, advect_x_into
    sim = _small_sim()
    f0 = sim.f.clone()
    a, b_ = torch.empty_like(f0), torch.empty_like(f0)
    advect_x_into(f0, a, sim.x_plan)
    advect_x_into(a, b_, sim.x_plan)
    c = torch.empty_like(f0)
    mom = torch.empty(3, dtype=torch.float64, device=DEV)
    rho = torch.empty(f0.shape[1], dtype=torch.float64, device=DEV)
    advect_x_fused_into(f0, c, sim.x_plan, 2, mom=sim._mom_args(mom), rho=(sim._vw, rho))
    assert torch.equal(b_, c)
    ref_m = sv.moments(a, sim.vweights, sim.vcoords, sim.xgrid.dof_weights)
    assert np.allclose(mom.cpu().numpy(), ref_m, rtol=1e-13, atol=1e-13 * abs(ref_m[0]))
    ref_rho = sv.compute_rho(b_, sim.vweights)
    assert torch.allclose(rho, ref_rho, rtol=1e-13, atol=0)
    d = torch.empty_like(f0)
    advect_x_fused_into(f0, d, sim.x_plan, 1, rho=(sim._vw, rho))
    assert torch.equal(d, a)


def test_pipelined_advance_matches_steps_bitwise():
    s1, s2 = _small_sim(), _small_sim()
    recs = [s1.step() for _ in range(4)]
    table = s2.advance(4).cpu().numpy()
    for r, row in zip(recs, table):
        assert (r.e_max, r.e_field, r.m0, r.m1, r.m2) == tuple(float(v) for v in row)
    assert torch.equal(s1.f, s2.f)


def test_step_host_roundtrip():
    s1, s2 = _small_sim(), _small_sim()
    fh = s2.f.cpu().numpy().copy()
    r1 = s1.step()
    r2 = s2.step_host(fh)
    assert r1 == r2
    assert np.array_equal(fh, s1.f.cpu().numpy())


@pytest.mark.parametrize("nx,px", [(8, 1), (16, 2), (24, 3), (64, 2), (128, 3), (40, 2)])
def test_fused_x_geometries(nx, px):
    """Every fused-x geometry (lanes per row, cells per lane) against the plain pass."""
    from paper_2603_19959_b200.xfield import advect_x_fused_into, advect_x_into
    sim = _small_sim(n_x=nx, degree_x=px, n_base=4, levels=1)
    rng = np.random.default_rng(nx)
    f0 = dev(rng.standard_normal(tuple(sim.f.shape)))
    a, b_ = torch.empty_like(f0), torch.empty_like(f0)
    advect_x_into(f0, a, sim.x_plan)
    advect_x_into(a, b_, sim.x_plan)
    ref = so.advect_x(f0.cpu().numpy(), so.x_plan(so.XGrid(nx, px, sim.config.length),
                                                   sim.vcoords[:, 0], 0.5 * sim.config.dt), nx)
    assert np.abs(a.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()
    c = torch.empty_like(f0)
    mom = torch.empty(3, dtype=torch.float64, device=DEV)
    rho = torch.empty(f0.shape[1], dtype=torch.float64, device=DEV)
    advect_x_fused_into(f0, c, sim.x_plan, 2, mom=sim._mom_args(mom), rho=(sim._vw, rho))
    assert torch.equal(b_, c)
    ref_m = np.array(sv.moments(a, sim.vweights, sim.vcoords, sim.xgrid.dof_weights))
    assert np.abs(mom.cpu().numpy() - ref_m).max() <= 1e-12 * np.abs(ref_m).max()
    ref_rho = sv.compute_rho(b_, sim.vweights)
    assert torch.allclose(rho, ref_rho, rtol=1e-12, atol=1e-14)


def test_slab_x_kernel_matches_periodic():
    """Slab update with margins filled from the periodic neighbours == periodic update."""
    import ctypes as C

    from paper_2603_19959_b200 import _capi, shard
    from paper_2603_19959_b200._device import current_stream
    from paper_2603_19959_b200.xfield import advect_x_into
    rng = np.random.default_rng(11)
    nx, p = 32, 2
    o = p + 1
    xg = sv.XGrid(nx, p, 4.0 * np.pi)
    sp = np.concatenate([rng.uniform(-6, 6, 40), [0.0]])
    plan = sv.precompute_x_matrices(xg, sp, 0.05)
    fg = rng.standard_normal((len(sp), nx * o))
    full = torch.empty((len(sp), nx * o), dtype=torch.float64, device=DEV)
    advect_x_into(dev(fg), full, plan)
    hl, hr = shard.x_halo_cells(xg.h, sp, 0.05)
    assert (hl, hr) == plan.halo()
    for c0, nl in ((0, 8), (8, 8), (24, 8), (5, 11)):
        lw, rw = shard.margin_dofs(hl, o), shard.margin_dofs(hr, o)
        width = lw + nl * o + rw
        ext = np.zeros((len(sp), width))
        cells = [(c0 - hl + k) % nx for k in range(hl + nl + hr)]
        blk = np.concatenate([fg[:, c * o:(c + 1) * o] for c in cells], axis=1)
        ext[:, lw - hl * o:lw + (nl + hr) * o] = blk
        e_d = dev(ext)
        out = torch.zeros_like(e_d)
        _capi.check(_capi.lib().sldg_advect_x_slab(
            plan.device_handle(), e_d[:, lw - hl * o:].data_ptr(), width, hl, hr, nl,
            out[:, lw:].data_ptr(), width, current_stream()))
        got = out[:, lw:lw + nl * o].cpu().numpy()
        assert np.array_equal(got, full[:, c0 * o:(c0 + nl) * o].cpu().numpy())


def test_sharded_world1_matches_simulation():
    from paper_2603_19959_b200.shard import ShardedSimulation
    cfg = sv.SimConfig(dim=3, n_base=4, levels=1, degree=2, n_x=16, n_steps=3)
    a = sv.Simulation(cfg)
    b = ShardedSimulation(cfg, 0, 1)
    ra = [a.step() for _ in range(3)]
    rb = [b.step() for _ in range(3)]
    fa, fb = a.f.cpu().numpy(), b.f.cpu().numpy()
    assert np.abs(fa - fb).max() <= 1e-13 * np.abs(fa).max()
    for x, y in zip(ra, rb):
        assert abs(x.m0 - y.m0) <= 1e-13 * abs(x.m0)
        assert abs(x.e_max - y.e_max) <= 1e-11 * abs(x.e_max)


FUSED_CASES = [dict(dim=3, n_base=8, levels=0, degree=2, n_x=32),
               dict(dim=3, n_base=16, levels=0, degree=1, n_x=16),
               dict(dim=3, n_base=6, levels=0, degree=3, n_x=24, bc="periodic"),
               dict(dim=3, n_base=8, levels=0, degree=2, n_x=64, degree_x=1),
               # the compile-time 64-cell row of the headline shape (Q2, p_x = 2)
               dict(dim=3, n_base=6, levels=0, degree=2, n_x=64),
               dict(dim=3, n_base=5, levels=0, degree=2, n_x=64, bc="periodic")]


@pytest.mark.parametrize("kw", FUSED_CASES)
def test_fused_step_matches_unfused_and_oracle(kw):
    a = sv.Simulation(sv.SimConfig(**kw, n_steps=4))
    assert a.fused_step_supported(), "uniform mesh must take the one-pass step"
    b = sv.Simulation(sv.SimConfig(**kw, n_steps=4))
    b._fused_ok = False
    ta = a.advance(4).cpu().numpy()
    tb = b.advance(4).cpu().numpy()
    fa, fb = a.f.cpu().numpy(), b.f.cpu().numpy()
    assert np.abs(fa - fb).max() <= 1e-13 * np.abs(fb).max()
    np.testing.assert_allclose(ta[:, 2:], tb[:, 2:], rtol=1e-13, atol=1e-13 * abs(tb[0, 2]))
    np.testing.assert_allclose(ta[:, :2], tb[:, :2], rtol=1e-10)
    ref = so.Sim(**kw)
    recs = [ref.step() for _ in range(4)]
    assert np.abs(fa - ref.f).max() <= 1e-12 * np.abs(ref.f).max()
    for row, r in zip(ta, recs):
        assert abs(row[2] - r["m0"]) <= 1e-12 * abs(r["m0"])
        assert abs(row[0] - r["e_max"]) <= 1e-10 * recs[0]["e_max"]


@pytest.mark.parametrize("kw", FUSED_CASES[:3] + FUSED_CASES[4:])
def test_fused_last_step_mode_vs_unfused_and_oracle(kw):
    """Simulation.step() on a fused-eligible plan: leading X + field chain + the fused
    kernel's last-step mode (V + trailing X + moments) == the 3-pass step."""
    a = sv.Simulation(sv.SimConfig(**kw, n_steps=2))
    b = sv.Simulation(sv.SimConfig(**kw, n_steps=2))
    b._fused_ok = False
    ref = so.Sim(**kw)
    for k in range(2):
        ra, rb, rr = a.step(), b.step(), ref.step()
        fa, fb = a.f.cpu().numpy(), b.f.cpu().numpy()
        assert np.abs(fa - fb).max() <= 1e-13 * np.abs(fb).max()
        assert np.abs(fa - ref.f).max() <= 1e-12 * np.abs(ref.f).max()
        assert abs(ra.m0 - rb.m0) <= 1e-13 * abs(rb.m0)
        assert abs(ra.m2 - rr["m2"]) <= 1e-12 * abs(rr["m2"])
        if k == 0:   # same state, same rho: the field chain equals the separate kernels
            assert ra.e_max == rb.e_max and ra.e_field == rb.e_field
        assert abs(ra.e_max - rr["e_max"]) <= 1e-10 * abs(rr["e_max"])


def test_run_uses_fused_step_and_matches_step_loop():
    cfg = sv.SimConfig(dim=3, n_base=8, levels=0, degree=2, n_x=32, n_steps=5)
    res = sv.run(cfg)
    sim = sv.Simulation(cfg)
    recs = [sim.diagnostics(sim.field_solve())] + [sim.step() for _ in range(5)]
    for x, y in zip(res.records, recs):
        assert abs(x.m0 - y.m0) <= 1e-13 * abs(y.m0)
        assert abs(x.e_max - y.e_max) <= 1e-10 * abs(recs[0].e_max)


@pytest.mark.parametrize("direction", [1, 2])
@pytest.mark.parametrize("nb,lv,p,bc", [(4, 1, 2, "absorbing"), (4, 1, 3, "periodic"),
                                        (6, 0, 2, "absorbing"), (5, 2, 1, "periodic")])
def test_sweep_other_directions_vs_oracle(direction, nb, lv, p, bc):
    """v_y / v_z sweeps: plans for directions 1 and 2 use the same kernels."""
    rng = np.random.default_rng(direction * 100 + nb + lv + p)
    m = sv.build_mesh(3, nb, lv, 6.0)
    b = sv.DGBasis(p)
    ps = sv.classify_conforming(sv.extract_pencils(m, direction), m, bc)
    plan = sv.build_sweep_plan(m, ps, sv.build_permutation(b, 3), b)
    om = so.make_mesh(3, nb, lv, 6.0)
    oplan = so.make_plan(om, so.mark_conforming(so.make_pencils(om, direction), bc), p)
    f = rng.standard_normal((plan.n_dofs, 34))
    speeds = rng.uniform(-1.5, 1.5, 34) * 0.2
    speeds[2] = 0.0
    speeds[4] *= 30.0
    ref = so.advect_v(f.copy(), speeds, 0.1, oplan, bc)
    fd = dev(f)
    sv.advect_velocity(fd, speeds, 0.1, plan, bc=bc)
    got = fd.cpu().numpy()
    assert np.abs(got - ref).max() <= TOL * np.abs(ref).max()
    assert np.array_equal(got[:, 2], f[:, 2])


@pytest.mark.parametrize("bc", ["absorbing", "periodic"])
@pytest.mark.parametrize("emax", [0.02, 9.0, 40.0])
def test_fused_step_any_shift_matches_separate_passes(bc, emax):
    """k_step_fused with E large enough that the v-shift leaves {-1, 0} (the kernel's
    global-load path instead of the TMA ring) == advect_v followed by the X.X pass."""
    kw = dict(dim=3, n_base=6, levels=0, degree=2, n_x=32, bc=bc)
    a = sv.Simulation(sv.SimConfig(**kw, n_steps=1))
    b = sv.Simulation(sv.SimConfig(**kw, n_steps=1))
    assert a.fused_step_supported()
    rng = np.random.default_rng(int(emax * 10))
    e = dev(rng.uniform(-emax, emax, a.f.shape[1]))
    e[3] = 0.0
    f0 = dev(rng.standard_normal(tuple(a.f.shape)))
    a.f.copy_(f0)
    b.f.copy_(f0)
    out_a = torch.empty(3, dtype=torch.float64, device=DEV)
    out_b = torch.empty(3, dtype=torch.float64, device=DEV)
    a._fused_step(e, out_a)
    b._advect_v(e)
    b._xx(out_b)
    fa, fb = a.f.cpu().numpy(), b.f.cpu().numpy()
    assert np.abs(fa - fb).max() <= 1e-13 * np.abs(fb).max()
    np.testing.assert_allclose(out_a.cpu().numpy(), out_b.cpu().numpy(), rtol=1e-12,
                               atol=1e-12 * abs(float(out_b[0])))
    np.testing.assert_allclose(a._rho.cpu().numpy(), b._rho.cpu().numpy(), rtol=1e-12,
                               atol=1e-12 * float(b._rho.abs().max()))


@pytest.mark.parametrize("p,nx", [(2, 32), (1, 24)])
def test_slab_tiles_kernel_matches_periodic(p, nx):
    """Row-tile slab kernel (whole padded rows staged, halo-relative sources) == the
    periodic update on the slab's columns, bitwise; its rho epilogue == rho of them."""
    import ctypes as C

    from paper_2603_19959_b200 import _capi, shard
    from paper_2603_19959_b200._device import current_stream
    from paper_2603_19959_b200.xfield import advect_x_into
    cfg = sv.SimConfig(dim=3, n_base=4, levels=1, degree=p, n_x=nx, degree_x=2, n_steps=1)
    sim = sv.Simulation(cfg)
    o = sim.xgrid.degree + 1
    rng = np.random.default_rng(nx + p)
    fg = rng.standard_normal(tuple(sim.f.shape))
    full = torch.empty_like(sim.f)
    advect_x_into(dev(fg), full, sim.x_plan)
    sp = sim.vcoords[:, 0]
    hl, hr = shard.x_halo_cells(sim.xgrid.h, sp, 0.5 * cfg.dt)
    w = dev(sim.vweights)
    for c0, nl in ((0, 8), (8, 8), (nx - 8, 8), (3, 10)):
        lw, rw = shard.margin_dofs(hl, o), shard.margin_dofs(hr, o)
        width = lw + nl * o + rw
        width += width & 1
        ext = np.zeros((fg.shape[0], width))
        cells = [(c0 - hl + k) % nx for k in range(hl + nl + hr)]
        blk = np.concatenate([fg[:, c * o:(c + 1) * o] for c in cells], axis=1)
        ext[:, lw - hl * o:lw + (nl + hr) * o] = blk
        e_d = dev(ext)
        out = torch.zeros_like(e_d)
        nb = C.c_size_t()
        _capi.check(_capi.lib().sldg_advect_x_slab_tiles_scratch(
            sim.x_plan.device_handle(), nl, width, C.byref(nb)))
        scr = torch.empty(nb.value, dtype=torch.uint8, device=DEV)
        rho = torch.empty(nl * o, dtype=torch.float64, device=DEV)
        _capi.check(_capi.lib().sldg_advect_x_slab_tiles(
            sim.x_plan.device_handle(), e_d.data_ptr(), width, lw - hl * o, hl, hr, nl,
            out.data_ptr(), width, lw, 1, 0, fg.shape[0], 0, w.data_ptr(), None, None, None,
            None, rho.data_ptr(), scr.data_ptr(), current_stream()))
        got = out[:, lw:lw + nl * o].cpu().numpy()
        ref = full[:, c0 * o:(c0 + nl) * o].cpu().numpy()
        assert np.array_equal(got, ref), (c0, nl)
        r_ref = sim.vweights @ ref
        assert np.abs(rho.cpu().numpy() - r_ref).max() <= 1e-13 * np.abs(r_ref).max()


@pytest.mark.parametrize("p,nx", [(2, 32), (3, 24)])
def test_slab_xx_kernel_matches_periodic_xx(p, nx):
    """n_apply = 2 on a slab (doubled halos, the intermediate's halo cells formed in the
    kernel) == the periodic X.X pass on the slab's columns, bitwise, in row chunks whose
    rho / moments accumulate in call order."""
    import ctypes as C

    from paper_2603_19959_b200 import _capi
    from paper_2603_19959_b200._device import current_stream
    from paper_2603_19959_b200.xfield import advect_x_fused_into
    cfg = sv.SimConfig(dim=3, n_base=4, levels=1, degree=p, n_x=nx, degree_x=2, n_steps=1)
    sim = sv.Simulation(cfg)
    o = sim.xgrid.degree + 1
    rng = np.random.default_rng(nx * p)
    fg = rng.standard_normal(tuple(sim.f.shape))
    full = torch.empty_like(sim.f)
    advect_x_fused_into(dev(fg), full, sim.x_plan, 2)
    hl1, hr1 = sim.x_plan.halo()
    hl, hr = max(2, 2 * hl1), max(1, 2 * hr1)
    w = dev(sim.vweights)
    n_rows = fg.shape[0]
    cut = (n_rows // (p + 1) ** 3 // 2) * (p + 1) ** 3
    for c0, nl in ((0, 12), (nx - 12, 12), (5, 13)):
        if max(hl, hr) > nl:
            continue
        lw, rw = hl * o + (hl * o) % 2, hr * o + (hr * o) % 2
        width = lw + nl * o + rw
        width += width & 1
        ext = np.zeros((n_rows, width))
        cells = [(c0 - hl + k) % nx for k in range(hl + nl + hr)]
        ext[:, lw - hl * o:lw + (nl + hr) * o] = np.concatenate(
            [fg[:, c * o:(c + 1) * o] for c in cells], axis=1)
        e_d = dev(ext)
        out = torch.zeros_like(e_d)
        nb = C.c_size_t()
        _capi.check(_capi.lib().sldg_advect_x_slab_tiles_scratch(
            sim.x_plan.device_handle(), nl, width, C.byref(nb)))
        scr = torch.empty(nb.value, dtype=torch.uint8, device=DEV)
        rho = torch.empty(nl * o, dtype=torch.float64, device=DEV)
        for i, (r0, r1) in enumerate(((0, cut), (cut, n_rows))):
            _capi.check(_capi.lib().sldg_advect_x_slab_tiles(
                sim.x_plan.device_handle(), e_d.data_ptr(), width, lw - hl * o, hl, hr, nl,
                out.data_ptr(), width, lw, 2, r0, r1 - r0, i, w.data_ptr(), None, None, None,
                None, rho.data_ptr(), scr.data_ptr(), current_stream()))
        got = out[:, lw:lw + nl * o].cpu().numpy()
        ref = full[:, c0 * o:(c0 + nl) * o].cpu().numpy()
        assert np.array_equal(got, ref), (c0, nl)
        r_ref = sim.vweights @ ref
        assert np.abs(rho.cpu().numpy() - r_ref).max() <= 1e-13 * np.abs(r_ref).max()


def test_fused_step_advice():
    """The library advises the one-pass step for the headline shape (two CTAs per SM, no
    spills) and not for shapes whose kernel spills or runs one CTA per SM; the default
    policy follows the advice, "force" / "off" override it."""
    import ctypes as C

    from paper_2603_19959_b200 import _capi

    def advice(**kw):
        s = sv.Simulation(sv.SimConfig(**kw, n_steps=1))
        adv = C.c_int32(-1)
        _capi.check(_capi.lib().sldg_step_fused_advice(
            s.sweep_plan.device_handle(), s.x_plan.device_handle(), s.f.shape[1],
            s.f.stride(0), C.byref(adv)))
        return adv.value, s

    yes, s = advice(dim=3, n_base=4, levels=0, degree=2, n_x=64)
    assert yes == 1
    s.fused_policy = "auto"
    assert s.fused_step_supported()
    no, s = advice(dim=3, n_base=4, levels=0, degree=2, n_x=64, degree_x=3)
    assert no == 0
    s.fused_policy = "auto"
    assert not s.fused_step_supported()
    s2 = sv.Simulation(sv.SimConfig(dim=3, n_base=4, levels=0, degree=2, n_x=64, n_steps=1))
    s2.fused_policy = "off"
    assert not s2.fused_step_supported()


@pytest.mark.parametrize("kw", [dict(dim=3, n_base=8, levels=0, degree=2, n_x=32),
                                dict(dim=3, n_base=4, levels=1, degree=2, n_x=16)])
def test_advance_graph_matches_advance_bitwise(kw):
    """advance() replayed from a captured CUDA graph (fused pipeline on the uniform mesh,
    separate passes on the AMR mesh) gives the eager results bit for bit, across both
    state-buffer parities and repeated replays."""
    a = sv.Simulation(sv.SimConfig(**kw, n_steps=3))
    b = sv.Simulation(sv.SimConfig(**kw, n_steps=3))
    for n in (3, 3, 2, 3, 2, 3):
        ta = a.advance(n).cpu().numpy()
        tb = b.advance_graph(n).cpu().numpy()
        assert np.array_equal(ta, tb)
        assert torch.equal(a.f, b.f)


@pytest.mark.parametrize("bc", ["absorbing", "periodic"])
@pytest.mark.parametrize("dim,nb,lv,p", [(3, 8, 1, 2), (3, 6, 2, 3), (3, 8, 0, 2)])
@pytest.mark.parametrize("ncol", [64, 200, 520])
def test_sweep_schedules_bitwise(monkeypatch, bc, dim, nb, lv, p, ncol):
    """The pencil walk (k_sweep_stream) + per-cell worklist and the worklist alone
    (k_vclassify -> k_vitems for every entry) give the same bits; both match the oracle.
    64 columns: whole-row cells (one 1-D bulk copy); 200 (Q3: 96-column tiles, the last
    partly out of range) and 520 (Q2: 256-column tiles): 2-D tensor-map boxes, zero-filled
    past the last column."""
    rng = np.random.default_rng(300 + nb + lv + p + ncol)
    plan, _, _ = plan_for(dim, nb, lv, p, bc)
    f = rng.standard_normal((plan.n_dofs, ncol))
    speeds = rng.uniform(-1.5, 1.5, size=ncol) * 0.2
    speeds[9] = 0.0
    outs = {}
    for sched in ("walk", "items"):
        monkeypatch.setenv("SLDG_SWEEP_SCHEDULE", sched)
        fd = dev(f)
        sv.advect_velocity(fd, speeds, 0.1, plan, bc=bc)
        torch.cuda.synchronize()
        outs[sched] = fd.cpu().numpy()
    assert np.array_equal(outs["walk"], outs["items"])
    assert np.array_equal(outs["items"][:, 9], f[:, 9])
    if ncol != 64:   # the worklist alone is oracle-checked at 64 columns
        return
    om = so.make_mesh(dim, nb, lv, 6.0)
    oplan = so.make_plan(om, so.mark_conforming(so.make_pencils(om, 0), bc), p)
    ref = so.advect_v(f.copy(), speeds, 0.1, oplan, bc)
    assert np.abs(outs["items"] - ref).max() <= TOL * np.abs(ref).max()


@pytest.mark.parametrize("weights", ["count", "area"])
def test_duplicate_pencils_swept_once(monkeypatch, weights):
    """Duplicate whole-fast pencils (identical cell lists) are swept once and their
    targets written with the write-back formula (per-duplicate weights, plan order): the
    walk with the deduplication, the walk without it (SLDG_SWEEP_DEDUP=0: every duplicate
    through the scratch slots) and the worklist give the same bits; the oracle agrees."""
    rng = np.random.default_rng(77)
    m = sv.build_mesh(3, 8, 2, 6.0)
    b = sv.DGBasis(2)
    ps = sv.classify_conforming(sv.extract_pencils(m, 0, weights), m, "absorbing")
    plan = sv.build_sweep_plan(m, ps, sv.build_permutation(b, 3), b)
    ncol = 64
    f = rng.standard_normal((plan.n_dofs, ncol))
    speeds = rng.uniform(-1.5, 1.5, size=ncol) * 0.2
    speeds[5] = 0.0
    outs = {}
    for key, sched, dd in (("dedup", "walk", "1"), ("slots", "walk", "0"), ("items", "items", "1")):
        monkeypatch.setenv("SLDG_SWEEP_SCHEDULE", sched)
        monkeypatch.setenv("SLDG_SWEEP_DEDUP", dd)
        fd = dev(f)
        sv.advect_velocity(fd, speeds, 0.1, plan, bc="absorbing")
        torch.cuda.synchronize()
        outs[key] = fd.cpu().numpy()
    assert np.array_equal(outs["dedup"], outs["slots"])
    assert np.array_equal(outs["dedup"], outs["items"])
    om = so.make_mesh(3, 8, 2, 6.0)
    oplan = so.make_plan(om, so.mark_conforming(so.make_pencils(om, 0, weights), "absorbing"), 2)
    ref = so.advect_v(f.copy(), speeds, 0.1, oplan, "absorbing")
    assert np.abs(outs["dedup"] - ref).max() <= TOL * np.abs(ref).max()
