"""The reference's pure pencil-level functions on the device (needs a B200):
apply_update, projection_oracle, generalized_overlap, weighted_writeback and
sweep_pencil against the reference's golden vectors and the CPU oracle.
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

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-12


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300)


def test_apply_update_matches_reference_goldens():
    g = np.load(os.path.join(GOLD, "basis_1d.npz"))
    for k in range(int(g["n_upd"])):
        p, bc, disp = int(g[f"upd{k}_p"]), str(g[f"upd{k}_bc"]), float(g[f"upd{k}_disp"])
        b = sv.DGBasis(p)
        d = sv.decompose_shift(disp, 1.0, 1.0)
        out = sv.apply_update(g[f"upd{k}_vals"], d, sv.overlap_pair(b, d.frac), bc)
        assert rel(out, g[f"upd{k}_out"]) <= TOL, (k, p, bc)


def test_apply_update_device_tensor_and_errors():
    b = sv.DGBasis(2)
    d = sv.decompose_shift(0.7, 1.0, 1.0)
    pair = sv.overlap_pair(b, d.frac)
    v = np.random.default_rng(3).standard_normal((4, 6, 3))
    host = sv.apply_update(v, d, pair, "periodic")
    dv = sv.apply_update(torch.from_numpy(v).cuda(), d, pair, "periodic")
    assert dv.is_cuda and np.array_equal(dv.cpu().numpy(), host)
    with pytest.raises(ValueError):
        sv.apply_update(v[0, 0], d, pair)
    with pytest.raises(ValueError):
        sv.apply_update(v, d, pair, "reflecting")


@pytest.mark.parametrize("p,n,disp,bc", [(1, 5, 0.37, "periodic"), (2, 6, -2.61, "periodic"),
                                         (3, 4, 9.3, "periodic"), (2, 7, 1.8, "absorbing"),
                                         (4, 5, -0.45, "absorbing")])
def test_projection_oracle_vs_oracle_and_apply_update(p, n, disp, bc):
    rng = np.random.default_rng(p * 10 + n)
    b, ob = sv.DGBasis(p), so.Basis(p)
    width = 0.75
    v = rng.standard_normal((n, p + 1))
    got = sv.projection_oracle(v, disp, width, b, bc)
    assert rel(got, so.brute_projection(v, disp, width, ob, bc)) <= 1e-13
    # the SLDG update is the exact projection of the translated solution
    d = sv.decompose_shift(disp, 1.0, width)
    upd = sv.apply_update(v, d, sv.overlap_pair(b, d.frac), bc)
    assert rel(got, upd) <= 1e-11


def test_generalized_overlap_vs_oracle():
    rng = np.random.default_rng(11)
    for p in (1, 2, 3, 5):
        b, ob = sv.DGBasis(p), so.Basis(p)
        for _ in range(12):
            dw = float(rng.choice([0.25, 0.5, 1.0]))
            sw = float(rng.choice([0.25, 0.5, 1.0]))
            dlo, slo = float(rng.uniform(-2, 2)), float(rng.uniform(-2, 2))
            disp = float(rng.uniform(-1.5, 1.5))
            g = sv.generalized_overlap(b, dlo, dw, slo, sw, disp)
            m, vl, vr = so.general_overlap(ob, dlo, dw, slo, sw, disp)
            assert (g.lo, g.hi) == (vl, vr)
            assert np.abs(g.matrix - m).max() <= 1e-13 * max(np.abs(m).max(), 1.0)
    with pytest.raises(ValueError):
        sv.generalized_overlap(sv.DGBasis(2), 0.0, 0.0, 0.0, 1.0, 0.1)


def test_weighted_writeback_bitwise_vs_oracle():
    rng = np.random.default_rng(5)
    n = 400
    f = rng.standard_normal(n)
    gather = np.concatenate([np.arange(n), rng.integers(0, n, 700)])
    weights = np.where(rng.random(gather.size) < 0.4, 1.0,
                       rng.choice([0.5, 0.25, 1.0 / 3.0], gather.size))
    values = rng.standard_normal(gather.size)
    got = sv.weighted_writeback(f, gather, weights, values)
    assert np.array_equal(got, so.writeback(f, gather, weights, values))
    with pytest.raises(sv.SweepError):
        sv.weighted_writeback(f, gather[gather != 7], weights[gather != 7],
                              values[gather != 7])


@pytest.mark.parametrize("nb,lv,p,bc,force", [(4, 1, 2, "absorbing", False),
                                               (4, 2, 1, "periodic", False),
                                               (3, 1, 3, "periodic", True),
                                               (6, 0, 2, "absorbing", False)])
def test_sweep_pencil_vs_oracle(nb, lv, p, bc, force):
    rng = np.random.default_rng(nb * 7 + lv + p)
    m = sv.build_mesh(3, nb, lv, 6.0)
    b, ob = sv.DGBasis(p), so.Basis(p)
    ps = sv.classify_conforming(sv.extract_pencils(m, 0), m, bc)
    n_levels = int(m.levels.max()) + 1
    for q in range(0, ps.n_pencils, max(1, ps.n_pencils // 5)):
        sl = ps.pencil_slice(q)
        lo, w = ps.lowers[sl], ps.widths[sl]
        lev, conf = ps.levels[sl], ps.conforming[sl]
        vals = rng.standard_normal((3, 2, len(lo), p + 1))
        speed, dt = float(rng.uniform(-4, 4)), 0.1
        lm = sv.precompute_level_matrices(b, speed, dt, m.base_width, n_levels)
        got = sv.sweep_pencil(vals, lo, w, lev, conf, speed, dt, lm, bc, 6.0, b, force)
        lsh = so.level_shifts(ob, speed, dt, m.base_width, n_levels)
        ref = so.pencil_update(vals, lo, w, lev, conf, speed, dt, lsh, bc, 6.0, ob, force)
        assert got.shape == vals.shape
        assert rel(got, ref) <= TOL, (q, speed)
    with pytest.raises(sv.SweepError):
        sv.sweep_pencil(np.zeros((2, 3)), lo, w, lev, conf, 1.0, dt, lm, bc, 6.0, b)
