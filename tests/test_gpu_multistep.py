"""Multi-step parity and conservation on the GPU (needs a B200).

* Coefficients after 1, 5, 50 and 200 Strang steps against the REFERENCE's own runs
  (tests/golden/coeffs_<cfg>.npz, made by tests/golden/make_golden_coeffs.py with
  sldg_vlasov.driver.Simulation): SURVEY.md §8(c) protocol (2), the north-star bar
  "coefficients within 1e-12 of the CPU reference", normwise (÷ max|f|) and per coefficient
  (÷ |f|) wherever |f| >= 1e-3 max|f| (a pure relative test is ill-posed for Maxwellian-tail
  coefficients of ~1e-10).  The steps run through the pipelined path
  run() uses (k_step_fused on uniform meshes, the AMR passes otherwise).
* Per-step mass conservation with periodic velocity bc, mirroring the reference's
  test_mass_and_momentum_invariants_per_step (pkg/tests/test_driver.py:92-101), on the
  fused path, the AMR worklist path, and with two AMR levels in "area" weight mode
  (the reference's 1/n_c weights lose ~3e-6 of the mass per step there).
* The Poisson solve + E at N_x = 128, 256, 512 against the reference (tests/golden/poisson.npz).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_19959_b200 as sv  # noqa: E402
from oracle import sldg_oracle as so  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DEV = torch.device("cuda", 0)
COEF_CFGS = {
    "cfg1": dict(dim=3, n_base=16, levels=0, degree=1, n_x=16),
    "cfg2": dict(dim=3, n_base=32, levels=0, degree=2, n_x=64),
    "cfg3": dict(dim=3, n_base=4, levels=1, degree=2, n_x=64),
    "cfg4": dict(dim=3, n_base=4, levels=2, degree=3, n_x=128),
}


def _compare(f, g, n, tol=1e-12):
    """Normwise <= 1e-12 max|f| at every saved step; per coefficient (|f| >= 1e-3 max|f|)
    <= 1e-12 over the first 5 steps and <= 1e-11 after 50 / 200 steps.  The per-coefficient
    difference grows by ~2.5e-14 per step at config 2 (7e-12 after 200 steps, normwise
    1.2e-13): every step rounds in a different order than numpy/BLAS, and the smallest
    coefficients of the band carry the most cancellation.  The reference's own dynamics do
    not amplify differences: seeding its state with 1e-16 relative noise, or swapping its LU
    Poisson solve for this build's explicit inverse, moves the same metric by < 6e-15 after
    50 steps."""
    idx = g["sample_idx"]
    ref = g[f"s{n}_val"]
    fmax = float(g[f"s{n}_fmax"])
    got = f.ravel()[idx]
    err = np.abs(got - ref)
    assert err.max() <= tol * fmax, f"step {n}: normwise {err.max() / fmax:.3e}"
    big = np.abs(ref) >= 1e-3 * fmax
    assert big.sum() > 100
    rel = (err[big] / np.abs(ref[big])).max()
    assert rel <= (tol if n <= 5 else 10 * tol), f"step {n}: per-coefficient {rel:.3e}"
    np.testing.assert_allclose(f.sum(axis=0), g[f"s{n}_colsum"], rtol=1e-11)
    return err.max() / fmax, rel


@pytest.mark.parametrize("name", list(COEF_CFGS))
def test_coefficients_match_reference_multistep(name):
    path = os.path.join(HERE, f"coeffs_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"no reference coefficient run for {name}")
    g = np.load(path)
    save_at = [int(n) for n in g["save_at"]]
    sim = sv.Simulation(sv.SimConfig(**COEF_CFGS[name], n_steps=max(save_at)))
    ref_rec = g["records"]
    done = 0
    tables = []
    for n in save_at:
        tables.append(sim.advance(n - done).cpu().numpy())
        done = n
        _compare(sim.f.cpu().numpy(), g, n)
    table = np.concatenate(tables)
    # records [max|E|, e_field, m0, m1, m2] vs the reference's (t, e_max, m0, m1, m2, e_field)
    ref = ref_rec[1:len(table) + 1]
    np.testing.assert_allclose(table[:, 2], ref[:, 2], rtol=1e-12)
    np.testing.assert_allclose(table[:, 4], ref[:, 4], rtol=1e-12)
    assert np.abs(table[:, 0] - ref[:, 1]).max() <= 1e-10 * ref_rec[0, 1]


def _periodic_mass_series(sim, n):
    table = sim.advance(n).cpu().numpy()
    m0 = table[:, 2]
    return np.abs(np.diff(m0)) / np.abs(m0[:-1]), table[:, 3]


@pytest.mark.parametrize("kw", [
    dict(dim=3, n_base=8, levels=0, degree=2, n_x=64),     # k_step_fused
    dict(dim=3, n_base=4, levels=1, degree=3, n_x=16),     # AMR worklist + write-back
    dict(dim=3, n_base=6, levels=1, degree=2, n_x=24),
])
def test_periodic_mass_invariant_per_step(kw):
    sim = sv.Simulation(sv.SimConfig(**kw, bc="periodic", n_steps=10))
    dm, m1 = _periodic_mass_series(sim, 10)
    # reference test_driver.py:92-101 asserts 1e-12; round-off here is a few ulp
    assert dm.max() <= 4e-15, dm
    assert np.abs(m1).max() <= 1e-10


def test_two_level_amr_mass_area_weights():
    """with two AMR levels the reference's 1/n_c pencil weights lose mass;
    the conservative "area" weights keep it to round-off.  Both modes match the oracle."""
    kw = dict(dim=3, n_base=4, levels=2, degree=3, n_x=16, bc="periodic", n_steps=4)
    drift = {}
    for mode in ("count", "area"):
        sim = sv.Simulation(sv.SimConfig(**kw, pencil_weights=mode))
        dm, _ = _periodic_mass_series(sim, 4)
        drift[mode] = dm.max()
        ref = so.Sim(dim=3, n_base=4, levels=2, degree=3, n_x=16, bc="periodic",
                     pencil_weights=mode)
        for _ in range(4):
            ref.step()
        f = sim.f.cpu().numpy()
        assert np.abs(f - ref.f).max() <= 1e-12 * np.abs(ref.f).max()
    assert drift["count"] > 1e-8          # the reference's known non-conservation
    assert drift["area"] <= 4e-15, drift


def test_poisson_large_nx_golden():
    g = np.load(os.path.join(HERE, "poisson.npz"))
    for nx in (128, 256, 512):
        ps = sv.PoissonSolver(sv.XGrid(nx, 2, 4.0 * np.pi))
        for k in range(2):
            rho = torch.from_numpy(g[f"nx{nx}_{k}_rho"]).to(DEV)
            phi = ps.solve(rho)
            e = ps.electric_field(phi).cpu().numpy()
            rphi, re_ = g[f"nx{nx}_{k}_phi"], g[f"nx{nx}_{k}_E"]
            assert np.abs(phi.cpu().numpy() - rphi).max() <= 1e-12 * np.abs(rphi).max()
            assert np.abs(e - re_).max() <= 1e-12 * np.abs(re_).max()
