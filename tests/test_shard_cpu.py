"""Multi-rank host logic of the sharded steps on CPU: world_size 2 and 3 over gloo.

The device kernels cannot run here, so the per-row halo pack / unpack is restated on
the host (the layout of csrc/halo.cu) and the two device reductions are replaced by
host stand-ins inside the worker processes.  What is under test is the product's
exchange layer, shard.Collectives.run servicing an advance() generator's requests:
the P2P halo exchange on the periodic ring into the margins, the rho all-gather in rank
order, the rank-order sum; plus the slab partition and the pencil item ranges.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_19959_b200 import shard


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _np_ordered_sum(parts, out):
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    out.copy_(acc)
    return out


def _np_gather_index(src, idx, out):
    out.copy_(src[idx])
    return out


def _widths(rng, n_rows, reach):
    """Per-row upwind halo widths like halo.cu: one side per row (or none)."""
    side = rng.integers(0, 3, n_rows)            # 0 identity, 1 left-reaching, 2 right
    w = rng.integers(1, reach + 1, n_rows)
    return np.where(side == 1, w, 0), np.where(side == 2, w, 0)


def _worker(rank, world, port, f_glob, nx, o, wl, wr, result_q):
    """One rank: its slab of f_glob in a [margin | local | margin] buffer; the per-row
    upwind halo packed on the host (the layout of halo.cu), exchanged by
    Collectives.run, unpacked by the 'after' callback; then an all-gather of a rho
    segment and a rank-order sum, all through the product's Collectives."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard.ordered_sum = _np_ordered_sum          # device kernels -> host stand-ins
        shard.gather_index = _np_gather_index
        part = shard.SlabPartition(nx, world)
        nl, c0 = part.local(rank), part.start(rank)
        hl, hr = int(wl.max()), int(wr.max())
        lw, rw = shard.margin_dofs(hl, o), shard.margin_dofs(hr, o)
        n_rows = f_glob.shape[0]
        buf = np.zeros((n_rows, lw + nl * o + rw))
        buf[:, lw:lw + nl * o] = f_glob[:, c0 * o:(c0 + nl) * o]
        to_r = torch.from_numpy(np.concatenate(
            [buf[r, lw + (nl - wl[r]) * o:lw + nl * o] for r in range(n_rows)]))
        to_l = torch.from_numpy(np.concatenate([buf[r, lw:lw + wr[r] * o] for r in range(n_rows)]))
        fr_l, fr_r = torch.empty_like(to_r), torch.empty_like(to_l)

        def unpack():
            ol = orr = 0
            for r in range(n_rows):
                a, b = wl[r] * o, wr[r] * o
                buf[r, lw - a:lw] = fr_l.numpy()[ol:ol + a]
                buf[r, lw + nl * o:lw + nl * o + b] = fr_r.numpy()[orr:orr + b]
                ol += a
                orr += b

        seg = shard.SegmentIndex([n * o for n in part.counts()], "cpu")
        loc = torch.zeros(seg.max_width, dtype=torch.float64)
        loc[:nl * o] = torch.arange(c0 * o, (c0 + nl) * o, dtype=torch.float64)
        rho = torch.empty(nx * o, dtype=torch.float64)
        vec = torch.tensor([1.5 * rank, float(rank), 1.0], dtype=torch.float64)

        def gen():
            ev = yield ("halo", (to_r, to_l, fr_l, fr_r), unpack)
            assert ev is None                       # CPU tensors: synchronous
            yield ("allgather", loc, rho, seg)
            yield ("sum", vec)
            return "done"

        assert shard.Collectives(rank, world).run(gen()) == "done"
        result_q.put((rank, c0, nl, lw, buf, rho.numpy(), vec.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nx,o", [(2, 16, 3), (3, 24, 2), (2, 12, 4)])
def test_collectives_halo_allgather_sum(world, nx, o):
    rng = np.random.default_rng(world * 100 + nx)
    n_rows = 20
    f_glob = rng.standard_normal((n_rows, nx * o))
    wl, wr = _widths(rng, n_rows, nx // world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, f_glob, nx, o, wl, wr, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, c0, nl, lw, buf, rho, vec in res:
        for r in range(n_rows):   # margins hold the periodic neighbours' cells
            for k in range(wl[r]):
                gc = (c0 - wl[r] + k) % nx
                np.testing.assert_array_equal(buf[r, lw - (wl[r] - k) * o:lw - (wl[r] - k - 1) * o],
                                              f_glob[r, gc * o:(gc + 1) * o])
            for k in range(wr[r]):
                gc = (c0 + nl + k) % nx
                s0 = lw + (nl + k) * o
                np.testing.assert_array_equal(buf[r, s0:s0 + o], f_glob[r, gc * o:(gc + 1) * o])
        np.testing.assert_array_equal(rho, np.arange(nx * o, dtype=float))
        assert vec[0] == sum(1.5 * r for r in range(world)) and vec[2] == world


def test_partition_and_margins():
    p = shard.SlabPartition(10, 4)
    assert p.counts() == [3, 3, 2, 2] and p.start(2) == 6 and sum(p.counts()) == 10
    h = 4.0 * np.pi / 512
    hl, hr = shard.x_halo_cells(h, np.linspace(-6, 6, 145), 0.05)
    # cfg5 grid: max |v| dt/2 / h = 6*0.05/0.0245 = 12.2 cells
    assert hl == 13 and hr == 13
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
