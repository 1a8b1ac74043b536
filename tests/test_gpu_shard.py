"""Sharded steps on one B200: the ranks' own advance() generators run in lockstep
(shard.Collectives.lockstep services their exchange points on one device, with the
arithmetic the NCCL driver uses), compared with the single-device Simulation.

x-slabs (ShardedSimulation, the AMR path): per-row upwind halos packed
and unpacked by libsldg, the trailing + leading half x-steps as one X.X pass after one
exchange of doubled halos, row-chunked.  Pencils (PencilShardedSimulation, uniform
meshes): the rank-order sum of the partials is the only exchange.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_19959_b200 as sv  # noqa: E402
from paper_2603_19959_b200 import _capi, shard  # noqa: E402
from paper_2603_19959_b200._device import current_stream  # noqa: E402

DEV = torch.device("cuda", 0)
SLAB_CASES = [dict(dim=3, n_base=4, levels=1, degree=2, n_x=24),                # cfg3 shape
              dict(dim=3, n_base=4, levels=2, degree=3, n_x=32),                # cfg4 shape
              dict(dim=3, n_base=4, levels=1, degree=2, n_x=24, bc="periodic"),
              dict(dim=3, n_base=4, levels=0, degree=1, n_x=32, degree_x=1)]


def _slab_run(kw, world, n_steps, n_chunks=3):
    sims = [shard.ShardedSimulation(sv.SimConfig(**kw, n_steps=n_steps), r, world,
                                    n_chunks=n_chunks) for r in range(world)]
    tabs = [torch.empty((n_steps, 5), dtype=torch.float64, device=DEV) for _ in sims]
    shard.Collectives.lockstep([s.advance_steps(n_steps, t) for s, t in zip(sims, tabs)])
    f = np.concatenate([s.f.cpu().numpy() for s in sims], axis=1)
    return f, [t.cpu().numpy() for t in tabs], sims


@pytest.mark.parametrize("kw", SLAB_CASES)
@pytest.mark.parametrize("world", [1, 2, 3])
def test_slab_ranks_in_lockstep_match_simulation(kw, world):
    n_steps = 4
    ref = sv.Simulation(sv.SimConfig(**kw, n_steps=n_steps))
    tr = ref.advance(n_steps).cpu().numpy()
    fr = ref.f.cpu().numpy()
    f, tabs, sims = _slab_run(kw, world, n_steps)
    assert np.abs(f - fr).max() <= 1e-13 * np.abs(fr).max()
    for t in tabs:   # every rank holds the same global diagnostics
        np.testing.assert_array_equal(t, tabs[0])
    np.testing.assert_allclose(tabs[0][:, 2:], tr[:, 2:], rtol=1e-12, atol=1e-13 * abs(tr[0, 2]))
    assert np.abs(tabs[0][:, 0] - tr[:, 0]).max() <= 1e-11 * tr[0, 0]


def test_slab_run_is_deterministic_and_chunk_count_only_changes_sums():
    kw = SLAB_CASES[1]
    f1, t1, _ = _slab_run(kw, 2, 3)
    f2, t2, _ = _slab_run(kw, 2, 3)
    np.testing.assert_array_equal(f1, f2)
    np.testing.assert_array_equal(t1[0], t2[0])
    f3, t3, _ = _slab_run(kw, 2, 3, n_chunks=1)
    assert np.abs(f3 - f1).max() <= 1e-13 * np.abs(f1).max()


def _halo_layout(sim, n_apply):
    """(wl, wr) cells per row from the x plan's shifts (host restatement of halo.cu)."""
    g = sim.x_plan.groups
    wl = np.zeros(len(g), dtype=np.int64)
    wr = np.zeros(len(g), dtype=np.int64)
    for k, grp in enumerate(g):
        n, a = grp.decomp.n_shift, grp.decomp.frac
        if n == 0 and a == 0.0:
            continue
        if n >= 0:
            wl[k] = n_apply * (n + 1)
        else:
            wr[k] = n_apply * -n
    inv = sim.x_plan.inverse
    return wl[inv], wr[inv]


@pytest.mark.parametrize("n_apply", [1, 2])
def test_halo_pack_unpack_rows(n_apply):
    kw = dict(dim=3, n_base=4, levels=1, degree=2, n_x=24)
    s = shard.ShardedSimulation(sv.SimConfig(**kw, n_steps=1), 0, 2)
    hp = s.halo1 if n_apply == 1 else s.halo2
    o, lw, nl = s.o, s.lw, s.n_local
    rng = np.random.default_rng(n_apply)
    buf = torch.from_numpy(rng.standard_normal(tuple(s._F.shape))).to(DEV)
    wl, wr = _halo_layout(s, n_apply)
    n_rows = buf.shape[0]
    e = hp.extent(0, n_rows)
    assert e[1] == int(wl.sum()) * o and e[3] == int(wr.sum()) * o
    assert hp.reach_l == wl.max() and hp.reach_r == wr.max()
    to_r = torch.zeros(max(e[1], 1), dtype=torch.float64, device=DEV)
    to_l = torch.zeros(max(e[3], 1), dtype=torch.float64, device=DEV)
    lib = _capi.lib()
    r_mid = (n_rows // 27 // 2) * 27
    for r0, r1 in ((0, r_mid), (r_mid, n_rows)):   # two chunks
        ex = hp.extent(r0, r1)
        _capi.check(lib.sldg_halo_pack(hp.h, buf.data_ptr(), s.width, lw, r0, r1,
                                       to_r[ex[0]:].data_ptr(), to_l[ex[2]:].data_ptr(),
                                       current_stream()))
    b = buf.cpu().numpy()
    want_r = np.concatenate([b[r, lw + (nl - wl[r]) * o:lw + nl * o] for r in range(n_rows)])
    want_l = np.concatenate([b[r, lw:lw + wr[r] * o] for r in range(n_rows)])
    np.testing.assert_array_equal(to_r.cpu().numpy()[:e[1]], want_r)
    np.testing.assert_array_equal(to_l.cpu().numpy()[:e[3]], want_l)
    # unpack: the neighbours' data lands in this slab's margins, nothing else changes
    out = buf.clone()
    _capi.check(lib.sldg_halo_unpack(hp.h, out.data_ptr(), s.width, lw, 0, n_rows,
                                     to_r.data_ptr(), to_l.data_ptr(), current_stream()))
    ob = out.cpu().numpy()
    exp = b.copy()
    for r in range(n_rows):
        if wl[r]:
            exp[r, lw - wl[r] * o:lw] = b[r, lw + (nl - wl[r]) * o:lw + nl * o]
        if wr[r]:
            exp[r, lw + nl * o:lw + (nl + wr[r]) * o] = b[r, lw:lw + wr[r] * o]
    np.testing.assert_array_equal(ob, exp)


@pytest.mark.parametrize("kw", [dict(dim=3, n_base=6, levels=0, degree=2, n_x=32),
                                dict(dim=3, n_base=5, levels=0, degree=1, n_x=16, bc="periodic")])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_pencil_ranks_in_lockstep_match_simulation(kw, world):
    n_steps = 3
    ref = sv.Simulation(sv.SimConfig(**kw, n_steps=n_steps))
    tr = ref.advance(n_steps).cpu().numpy()
    sims = [shard.PencilShardedSimulation(sv.SimConfig(**kw, n_steps=n_steps), r, world)
            for r in range(world)]
    tabs = [torch.empty((n_steps, 5), dtype=torch.float64, device=DEV) for _ in sims]
    shard.Collectives.lockstep([s.advance_steps(n_steps, t) for s, t in zip(sims, tabs)])
    rows = [s.owned_rows() for s in sims]
    allr = np.concatenate(rows)
    assert len(np.unique(allr)) == len(allr) == sims[0].f.shape[0]   # disjoint cover
    fref = ref.f.cpu().numpy()
    for s, r in zip(sims, rows):
        got = s.f.cpu().numpy()[r]
        assert np.abs(got - fref[r]).max() <= 1e-13 * np.abs(fref).max()
    for t in tabs:
        tt = t.cpu().numpy()
        np.testing.assert_array_equal(tt, tabs[0].cpu().numpy())
        np.testing.assert_allclose(tt[:, 2:], tr[:, 2:], rtol=1e-13, atol=1e-13 * abs(tr[0, 2]))
        np.testing.assert_allclose(tt[:, :2], tr[:, :2], rtol=1e-10)
    with pytest.raises(NotImplementedError):
        sims[0].step_host(None)


def test_slab_run_driver_matches_lockstep():
    """ShardedSimulation.advance() at world 1 goes through Collectives.run -- the NCCL
    driver's CUDA-stream path (halo exchange and unpack on the communication stream, the
    X.X chunks waiting on their events) -- and gives the lockstep driver's bits."""
    kw = SLAB_CASES[1]
    a = shard.ShardedSimulation(sv.SimConfig(**kw, n_steps=3), 0, 1, n_chunks=3)
    ta = a.advance(3).cpu().numpy()
    f, tabs, _ = _slab_run(kw, 1, 3)
    np.testing.assert_array_equal(a.f.cpu().numpy(), f)
    np.testing.assert_array_equal(ta, tabs[0])
