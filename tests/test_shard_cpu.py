"""Multi-rank x-slab logic on CPU: world_size 2 (and 3) over gloo.

The device kernels cannot run here, so the slab x-update is evaluated with the
oracle's 1D SLDG math, indexed exactly like the CUDA slab kernel
(xfield.cu k_advect_x, slab mode: source cell = cell + halo_l - n).  What is
under test is the product's host logic: partition, halo widths, the P2P
exchange into the margins, the rho all-gather and the rank-order sums.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sldg_oracle as so
from paper_2603_19959_b200 import shard


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def slab_update(ext, hl, n_local, o, groups_per_row):
    """Oracle math on a margin buffer: out[cell] = A u[cell+hl-n] + B u[cell+hl-n-1]."""
    n_rows = ext.shape[0]
    out = np.empty((n_rows, n_local * o))
    for r in range(n_rows):
        n, a, A, B = groups_per_row[r]
        u = ext[r].reshape(-1, o)
        if n == 0 and a == 0.0:
            out[r] = u[hl:hl + n_local].ravel()
            continue
        for c in range(n_local):
            out[r, c * o:(c + 1) * o] = A @ u[c + hl - n] + B @ u[c + hl - n - 1]
    return out


def _worker(rank, world, port, nx, p, speeds, f_glob, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = p + 1
        xg = so.XGrid(nx, p, 4.0 * np.pi)
        dt = 0.05
        part = shard.SlabPartition(nx, world)
        nl, c0 = part.local(rank), part.start(rank)
        hl, hr = shard.x_halo_cells(xg.h, speeds, dt)
        ex = shard.HaloExchanger(rank, world, hl, hr, o, nl)
        width = ex.lw + nl * o + ex.rw
        buf = torch.zeros((len(speeds), width), dtype=torch.float64)
        buf[:, ex.lw:ex.lw + nl * o] = torch.from_numpy(f_glob[:, c0 * o:(c0 + nl) * o])
        ex.exchange(buf)
        b = buf.numpy()
        # halo margins must equal the periodic neighbours' cells
        for k in range(hl):
            gc = (c0 - hl + k) % nx
            np.testing.assert_array_equal(b[:, ex.lw - hl * o + k * o:ex.lw - hl * o + (k + 1) * o],
                                          f_glob[:, gc * o:(gc + 1) * o])
        for k in range(hr):
            gc = (c0 + nl + k) % nx
            s0 = ex.lw + nl * o + k * o
            np.testing.assert_array_equal(b[:, s0:s0 + o], f_glob[:, gc * o:(gc + 1) * o])
        groups = []
        for sp in speeds:
            n, a = so.split_shift(float(sp), dt, xg.h)
            A, B = so.overlap_mats(xg.basis, a)
            groups.append((n, a, A, B))
        ext = b[:, ex.lw - hl * o:ex.lw + (nl + hr) * o]
        out = slab_update(ext, hl, nl, o, groups)
        # rho all-gather and the rank-order sum
        w = np.linspace(0.5, 1.5, len(speeds))
        rho_loc = torch.from_numpy(w @ out)
        rho = shard.allgather_segments(rho_loc, [n * o for n in part.counts()])
        tot = shard.sum_in_rank_order(torch.tensor([float(out.sum()), float(rank), 1.0]))
        result_q.put((rank, c0, out, rho.numpy(), tot.numpy(), (hl, hr)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nx,p", [(2, 16, 2), (3, 24, 1), (2, 12, 3)])
def test_sharded_x_advection_matches_global(world, nx, p):
    rng = np.random.default_rng(world * 100 + nx)
    speeds = np.concatenate([rng.uniform(-6.0, 6.0, 9), [0.0, 40.0 * 4.0 * np.pi / nx]])
    xg = so.XGrid(nx, p, 4.0 * np.pi)
    hl, hr = shard.x_halo_cells(xg.h, speeds, 0.05)
    if max(hl, hr) > nx // world:
        speeds = speeds[:-1]
    f_glob = rng.standard_normal((len(speeds), nx * (p + 1)))
    ref = so.advect_x(f_glob.copy(), so.x_plan(xg, speeds, 0.05), nx)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nx, p, speeds, f_glob, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    o = p + 1
    got = np.concatenate([r[2] for r in res], axis=1)
    # slab update with exchanged halos == global periodic update, bit for bit
    # (same operands, same order: python matmul on the same blocks)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14 * np.abs(ref).max())
    w = np.linspace(0.5, 1.5, len(speeds))
    for r in res:
        np.testing.assert_allclose(r[3], w @ got, rtol=1e-13)
        assert r[4][1] == sum(range(world)) and r[4][2] == world
    assert res[0][5][0] >= 1


def test_partition_and_halo_widths():
    p = shard.SlabPartition(10, 4)
    assert p.counts() == [3, 3, 2, 2] and p.start(2) == 6 and sum(p.counts()) == 10
    h = 4.0 * np.pi / 512
    hl, hr = shard.x_halo_cells(h, np.linspace(-6, 6, 145), 0.05)
    # cfg5 grid: max |v| dt/2 / h = 6*0.05/0.0245 = 12.2 cells
    assert hl == 13 and hr == 13
    with pytest.raises(ValueError):
        shard.HaloExchanger(0, 2, 5, 1, 3, 4)
    assert shard.margin_dofs(3, 3) == 10 and shard.margin_dofs(2, 3) == 6


@pytest.mark.parametrize("n_items,cells,world", [(3072, 32, 8), (50, 5, 3), (7, 4, 8), (9, 2, 2)])
def test_pencil_item_ranges_cover_whole_items(n_items, cells, world):
    """Pencil sharding: the ranks' tile shares are contiguous, disjoint, cover every
    tile, start and end on item boundaries, and differ by at most one item."""
    spans = [shard.item_tile_range(n_items * cells, cells, r, world) for r in range(world)]
    pos = 0
    for t0, cnt in spans:
        assert t0 == pos and t0 % cells == 0 and cnt % cells == 0
        pos += cnt
    assert pos == n_items * cells
    sizes = [c // cells for _, c in spans]
    assert max(sizes) - min(sizes) <= 1
