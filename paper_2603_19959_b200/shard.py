"""x-slab sharding of the Strang step across the GPUs of one box.

The phase-space state f (N_v x N_x^DOF) is split along x into contiguous
slabs of cells, one per rank (one process per GPU).  The velocity mesh and
sweep plan are replicated.  Per Strang step the only data exchanged are:
  * the x-advection halo, per half step: each rank receives `hl` cells from
    its left neighbour and `hr` cells from its right neighbour (periodic ring),
    hl/hr = the upwind reach of the shifts (sources c-n and c-n-1 of cell c);
  * the all-gather of rho's local segment (N_x^DOF doubles in total) -- the
    1D Poisson solve is tiny and runs redundantly on every rank;
  * the per-rank diagnostics partials (3 doubles), summed in rank order.
The v-sweep is column-local.  Because the x kernels compute every output
from the same operands in the same order whether the row is periodic or a
slab with halos, and rho's row partition does not depend on the column
count, f and E are bitwise identical for any number of ranks.

The state carries its halo margins in place: each buffer is
  [ left margin | local cells | right margin ]
per row (margins rounded up to an even number of doubles so the local part
stays 16-byte aligned), so halos are written straight into the margins and
the slab kernel reads one strided buffer.  The communication layer uses
torch.distributed P2P (NCCL over NVLink on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .driver import Simulation
from .sldg1d import decompose_shift


@dataclass(frozen=True)
class SlabPartition:
    """Contiguous split of n_cells x-cells over `world` ranks (first ranks get the extra)."""

    n_cells: int
    world: int

    def counts(self):
        base, extra = divmod(self.n_cells, self.world)
        return [base + (1 if r < extra else 0) for r in range(self.world)]

    def start(self, rank):
        return int(sum(self.counts()[:rank]))

    def local(self, rank):
        return self.counts()[rank]


def x_halo_cells(h: float, speeds, dt: float):
    """(hl, hr): cells needed left/right of a slab for one half step.

    Output cell c reads cells c-n and c-n-1 (sldg1d.py:124-136 with the
    shift split of sldg1d.py:39-55), so the left reach is max(n+1) and the
    right reach max(-n) over the rows that actually move.
    """
    hl = hr = 0
    for u in np.unique(np.asarray(speeds, dtype=float)):
        d = decompose_shift(float(u), dt, h)
        if d.n_shift == 0 and d.frac == 0.0:
            continue
        hl = max(hl, d.n_shift + 1)
        hr = max(hr, -d.n_shift)
    return hl, hr


def margin_dofs(cells: int, o: int) -> int:
    """Margin width in doubles, rounded up to even (keeps the local part aligned)."""
    m = cells * o
    return m + (m & 1)


class HaloExchanger:
    """Fill the left/right margins of a slab buffer from the ring neighbours.

    buf: (n_rows, lw + n_local*o + rw) tensor, lw/rw = margin widths in doubles;
    the last hl cells of the left margin and the first hr cells of the right
    margin are written.  Works on any torch device / process group.
    """

    def __init__(self, rank, world, hl, hr, o, n_local, group=None):
        if hl > n_local or hr > n_local:
            raise ValueError(f"halo ({hl}, {hr}) wider than the slab ({n_local} cells)")
        self.rank, self.world = rank, world
        self.hl, self.hr, self.o, self.n_local = hl, hr, o, n_local
        self.lw, self.rw = margin_dofs(hl, o), margin_dofs(hr, o)
        self.group = group
        self._bufs = {}

    def _buf(self, name, like, cols):
        key = (name, like.device, like.shape[0], cols)
        b = self._bufs.get(key)
        if b is None:
            import torch
            b = torch.empty((like.shape[0], cols), dtype=like.dtype, device=like.device)
            self._bufs[key] = b
        return b

    def exchange(self, buf):
        import torch
        import torch.distributed as dist
        o, hl, hr, lw, nl = self.o, self.hl, self.hr, self.lw, self.n_local
        loc0 = lw                      # first local double
        loc1 = lw + nl * o             # one past the last local double
        # to the right neighbour: my last hl cells (its left halo)
        # to the left neighbour: my first hr cells (its right halo)
        send_r = buf[:, loc1 - hl * o:loc1] if hl else None
        send_l = buf[:, loc0:loc0 + hr * o] if hr else None
        left_dst = buf[:, lw - hl * o:lw] if hl else None
        right_dst = buf[:, loc1:loc1 + hr * o] if hr else None
        if self.world == 1:
            if hl:
                left_dst.copy_(send_r)
            if hr:
                right_dst.copy_(send_l)
            return buf
        left = (self.rank - 1) % self.world
        right = (self.rank + 1) % self.world
        ops = []
        if hl:
            sr = self._buf("sr", buf, hl * o)
            sr.copy_(send_r)
            rl = self._buf("rl", buf, hl * o)
            ops += [dist.P2POp(dist.isend, sr, right, self.group),
                    dist.P2POp(dist.irecv, rl, left, self.group)]
        if hr:
            sl = self._buf("sl", buf, hr * o)
            sl.copy_(send_l)
            rr = self._buf("rr", buf, hr * o)
            ops += [dist.P2POp(dist.isend, sl, left, self.group),
                    dist.P2POp(dist.irecv, rr, right, self.group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if hl:
            left_dst.copy_(rl)
        if hr:
            right_dst.copy_(rr)
        del torch
        return buf


def allgather_segments(local, counts, group=None):
    """Concatenate per-rank 1-D segments (rank order) on every rank."""
    import torch
    import torch.distributed as dist
    world = len(counts)
    if world == 1:
        return local
    width = max(counts)
    pad = torch.zeros(width, dtype=local.dtype, device=local.device)
    pad[:local.numel()] = local
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([out[r][:counts[r]] for r in range(world)])


def sum_in_rank_order(vec, group=None):
    """Deterministic cross-rank sum: all-gather the partials, add them in rank order."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return vec
    import torch
    world = dist.get_world_size(group)
    parts = [torch.empty_like(vec) for _ in range(world)]
    dist.all_gather(parts, vec.contiguous(), group=group)
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    return acc


class ShardedSimulation:
    """Strang step on an x-slab of the state, one rank per GPU.

    Same step as driver.Simulation: half-x (with halo exchange), rho of the
    local columns all-gathered -> Poisson on every rank -> E, v-sweep of the
    local columns, half-x (halo exchange), diagnostics (local partials summed
    in rank order).  f lives in [margin | local | margin] buffers.
    """

    def __init__(self, config, rank, world, group=None, mesh=None):
        import torch

        from ._device import device, to_device_f64
        from .basis import DGBasis
        from .driver import sample_initial_into, velocity_dof_coords, velocity_dof_weights
        from .pencil import classify_conforming, extract_pencils
        from .tensor import build_permutation
        from .vmesh import build_mesh
        from .vsweep import build_sweep_plan
        from .xfield import PoissonSolver, XGrid, precompute_x_matrices

        self.config = config.validate()
        c = self.config
        self.rank, self.world, self.group = rank, world, group
        self.basis = DGBasis(c.degree)
        self.mesh = mesh if mesh is not None else build_mesh(c.dim, c.n_base, c.levels, c.radius)
        self.perm = build_permutation(self.basis, c.dim)
        pset = classify_conforming(extract_pencils(self.mesh, 0, c.pencil_weights), self.mesh,
                                   c.bc)
        self.sweep_plan = build_sweep_plan(self.mesh, pset, self.perm, self.basis)
        self.xgrid = XGrid(c.n_x, c.degree_x, c.length)
        self.vcoords = velocity_dof_coords(self.mesh, self.basis, self.perm)
        self.vweights = velocity_dof_weights(self.mesh, self.basis, self.perm)
        self.part = SlabPartition(c.n_x, world)
        self.n_local = self.part.local(rank)
        self.cell0 = self.part.start(rank)
        o = self.xgrid.degree + 1
        self.o = o
        hl, hr = x_halo_cells(self.xgrid.h, self.vcoords[:, 0], 0.5 * c.dt)
        self.halo = HaloExchanger(rank, world, hl, hr, o, self.n_local, group)
        self.lw, self.rw = self.halo.lw, self.halo.rw
        self.width = self.lw + self.n_local * o + self.rw
        # x plan over the full periodic grid (shifts and matrices are per speed)
        self.x_plan = precompute_x_matrices(self.xgrid, self.vcoords[:, 0], 0.5 * c.dt)
        if c.dim == 3:
            self.x_plan.velocity_order = c.degree + 1   # enables the row-tile slab kernel
        self.poisson = PoissonSolver(self.xgrid)
        dev = device()
        self._vw = to_device_f64(self.vweights)
        self._v0 = to_device_f64(self.vcoords[:, 0])
        self._v2 = to_device_f64((self.vcoords ** 2).sum(axis=1))
        x0, x1 = self.cell0 * o, (self.cell0 + self.n_local) * o
        self._xw = to_device_f64(self.xgrid.dof_weights[x0:x1])
        n_v = len(self.vweights)
        self._F = torch.zeros((n_v, self.width), dtype=torch.float64, device=dev)
        self._G = torch.zeros_like(self._F)
        sample_initial_into(c, self.vcoords, self.xgrid.dof_coords[x0:x1], self.f)
        self._rho_loc = torch.empty(self.n_local * o, dtype=torch.float64, device=dev)
        self._phi = torch.empty(self.poisson.n_nodes, dtype=torch.float64, device=dev)
        self._e = torch.empty(self.xgrid.n_dofs, dtype=torch.float64, device=dev)
        self._rec = torch.empty(5, dtype=torch.float64, device=dev)
        self.t = 0.0

    def fused_step_supported(self) -> bool:
        return False   # the one-pass step needs whole rows; slabs use the separate passes

    # views ------------------------------------------------------------------
    def _local(self, buf):
        return buf[:, self.lw:self.lw + self.n_local * self.o]

    @property
    def f(self):
        """Local slab of the state (view into the margin buffer)."""
        return self._local(self._F)

    @property
    def _e_local(self):
        x0 = self.cell0 * self.o
        return self._e[x0:x0 + self.n_local * self.o]

    # operators --------------------------------------------------------------
    def _advect_x(self):
        from . import _capi
        from ._device import current_stream
        self.halo.exchange(self._F)
        hl, hr = self.halo.hl, self.halo.hr
        o = self.o
        src = self._F[:, self.lw - hl * o:]
        _capi.check(_capi.lib().sldg_advect_x_slab(
            self.x_plan.device_handle(), src.data_ptr(), self._F.stride(0), hl, hr,
            self.n_local, self._G[:, self.lw:].data_ptr(), self._G.stride(0),
            current_stream()), ValueError)
        self._F, self._G = self._G, self._F

    def _x_tiles(self, rho_out=None, mom_out3=None):
        """Half x-step of the slab with the row-tile kernel, rho of the result (local
        columns) or the moments of the result fused in; False if the kernel does not
        cover this slab (then nothing was done)."""
        import ctypes as C

        from . import _capi
        from ._device import SCRATCH, current_stream
        if getattr(self, "_tiles_ok", None) is False:
            return False
        o, hl = self.o, self.halo.hl
        lib = _capi.lib()
        if getattr(self, "_tiles_ok", None) is None:
            nb = C.c_size_t()
            self._tiles_ok = lib.sldg_advect_x_slab_tiles_scratch(
                self.x_plan.device_handle(), self.n_local, self._F.stride(0), C.byref(nb)) == 0 \
                and self._F.stride(0) % 2 == 0
            self._tiles_bytes = nb.value
            if not self._tiles_ok:
                return False
        self.halo.exchange(self._F)
        scratch = SCRATCH.get(("xslab", id(self)), self._tiles_bytes)
        _capi.check(lib.sldg_advect_x_slab_tiles(
            self.x_plan.device_handle(), self._F.data_ptr(), self._F.stride(0),
            self.lw - hl * o, hl, self.n_local, self._G.data_ptr(), self._G.stride(0), self.lw,
            self._vw.data_ptr(), self._v0.data_ptr(), self._v2.data_ptr(), self._xw.data_ptr(),
            None if mom_out3 is None else mom_out3.data_ptr(),
            None if rho_out is None else rho_out.data_ptr(), scratch.data_ptr(),
            current_stream()), ValueError)
        self._F, self._G = self._G, self._F
        return True

    def _solve_from_local_rho(self, e_out):
        rho = allgather_segments(self._rho_loc, [n * self.o for n in self.part.counts()],
                                 self.group)
        self.poisson.solve_into(rho.contiguous(), self._phi, e_out)

    def _field(self, e_out):
        from .xfield import rho_into
        rho_into(self.f, self._vw, self._rho_loc)
        self._solve_from_local_rho(e_out)

    def _advect_v(self, e):
        from .vsweep import advect_velocity_into
        c = self.config
        x0 = self.cell0 * self.o
        e_loc = e[x0:x0 + self.n_local * self.o]
        advect_velocity_into(self.f, self._local(self._G), e_loc, c.dt, self.sweep_plan, c.bc,
                             c.force_slow)
        self._F, self._G = self._G, self._F

    def _diag_into(self, e, rec5):
        from .driver import _moments_into
        from .xfield import field_diag_into
        field_diag_into(self.poisson, e, rec5[0:2])
        _moments_into(self.f, self._vw, self._v0, self._v2, self._xw, rec5[2:5])
        rec5[2:5] = sum_in_rank_order(rec5[2:5].clone(), self.group)

    def enqueue_step(self, e_buf, rec5, v_event=None):
        """One Strang step: 3 passes over the slab when the row-tile slab kernel covers
        it (x + rho, v, x + moments), else x, rho, v, x, moments."""
        import torch

        from .xfield import field_diag_into
        if self._x_tiles(rho_out=self._rho_loc):
            self._solve_from_local_rho(e_buf)
        else:
            self._advect_x()
            self._field(e_buf)
        if v_event is not None:
            v_event[0].record(torch.cuda.current_stream())
        self._advect_v(e_buf)
        if v_event is not None:
            v_event[1].record(torch.cuda.current_stream())
        if self._x_tiles(mom_out3=rec5[2:5]):
            rec5[2:5] = sum_in_rank_order(rec5[2:5].clone(), self.group)
            field_diag_into(self.poisson, e_buf, rec5[0:2])
        else:
            self._advect_x()
            self._diag_into(e_buf, rec5)

    def advance(self, n_steps, table=None, v_events=None):
        import torch
        if table is None:
            table = torch.empty((n_steps, 5), dtype=torch.float64, device=self._F.device)
        for k in range(n_steps):
            self.enqueue_step(self._e, table[k], None if v_events is None else v_events[k])
        return table

    def step(self):
        from .driver import DiagnosticsRecord
        self.enqueue_step(self._e, self._rec)
        self.t += self.config.dt
        r = self._rec.cpu().numpy()
        return DiagnosticsRecord(self.t, float(r[0]), float(r[2]), float(r[3]), float(r[4]),
                                 float(r[1]), 0.5 * float(r[4]) + float(r[1]))


def item_tile_range(n_tiles: int, cells_per_item: int, rank: int, world: int):
    """(first tile, tile count) of `rank`'s contiguous share of whole items: the
    v-sweep of a cell reads its pencil neighbours, which must be rows the same rank
    keeps current, so items are never split between ranks."""
    n_items = n_tiles // cells_per_item
    i0, i1 = rank * n_items // world, (rank + 1) * n_items // world
    return i0 * cells_per_item, (i1 - i0) * cells_per_item


class PencilShardedSimulation(Simulation):
    """Pencil sharding for the plans the fused step covers (uniform velocity meshes).

    For those plans a direction-0 pencil's cells are swept together and every
    x row belongs to exactly one (pencil, line group, cell) tile of k_step_fused,
    so the whole Strang step -- leading half-x, v-sweep, trailing half-x -- is
    local to a (pencil, line group) item.  Each rank holds the full state buffer but
    advances only its contiguous share of whole items (rows of other ranks are never
    read or written here); the only exchange per step is the rank's partial sums
    [rho (N_x^DOF) | m0 m1 m2], added in rank order on every rank
    (sum_in_rank_order) so all ranks solve the same Poisson problem.  Total work
    is fixed as ranks are added (strong scaling).

    `reducer(vec) -> vec` replaces the cross-rank sum (tests run ranks in lockstep
    on one device).
    """

    def __init__(self, config, rank, world, group=None, mesh=None, reducer=None):
        super().__init__(config, mesh=mesh)
        if not self.fused_step_supported():
            raise ValueError("pencil sharding needs a plan the fused step covers "
                             "(uniform velocity mesh)")
        import torch

        from . import _capi
        info = np.zeros(4, dtype=np.int64)
        _capi.check(_capi.lib().sldg_step_fused_tiles(
            self.sweep_plan.device_handle(), self.x_plan.device_handle(), self._f.shape[1],
            self._f.stride(0), _capi.i64ptr(info)), ValueError)
        self.n_tiles, self.rows_per_tile, self.line_groups, self.cells_per_pencil = \
            (int(v) for v in info)
        self._tile_range = item_tile_range(self.n_tiles, self.cells_per_pencil, rank, world)
        self.rank, self.world, self.group = rank, world, group
        self._reducer = reducer if reducer is not None else \
            (lambda v: sum_in_rank_order(v, group))
        self._part = torch.zeros(self._f.shape[1] + 3, dtype=torch.float64,
                                 device=self._f.device)

    def owned_rows(self) -> np.ndarray:
        """Rows of f this rank advances: the rows of its tiles (tile t = cell
        t % cells of item t // cells; item = pencil * line_groups + line group)."""
        a = self.sweep_plan._arrays
        t = np.arange(*((self._tile_range[0], self._tile_range[0] + self._tile_range[1])))
        cell = t % self.cells_per_pencil
        item = t // self.cells_per_pencil
        pencil, lgrp = item // self.line_groups, item % self.line_groups
        cid = a["cell_ids"][a["offsets"][pencil] + cell]
        base = cid * self.sweep_plan.n_dofs // self.sweep_plan.n_cells + lgrp * self.rows_per_tile
        return (base[:, None] + np.arange(self.rows_per_tile)[None, :]).ravel()

    # phases ----------------------------------------------------------------
    def _fold_partials(self, moments: bool):
        """This rank's [rho | m0 m1 m2] from the partials of its last deferred step."""
        from . import _capi
        from ._device import SCRATCH, current_stream
        n = self._f.shape[1]
        scratch = SCRATCH.get(("fused", id(self)), self._fused_bytes)
        if not moments:
            self._part[n:].zero_()
        _capi.check(_capi.lib().sldg_step_fused_fold(
            self.sweep_plan.device_handle(), self.x_plan.device_handle(), n, self._f.stride(0),
            self._part[:n].data_ptr(), self._part[n:].data_ptr() if moments else None,
            scratch.data_ptr(), current_stream()), ValueError)
        return self._part

    def _take_sums(self, tot, mom3=None):
        n = self._f.shape[1]
        self._rho.copy_(tot[:n])
        if mom3 is not None:
            mom3.copy_(tot[n:])

    def advance(self, n_steps: int, table=None, v_events=None):
        """n_steps pipelined Strang steps on this rank's tiles; row k of the returned
        table is step k's [max|E|, e_field, m0, m1, m2] (global, identical on all ranks)."""
        import torch
        if table is None:
            table = torch.empty((n_steps, 5), dtype=torch.float64, device=self._f.device)
        if n_steps == 0:
            return table
        e = self._e
        n = self._f.shape[1]
        # leading half x-step of step 0 on my tiles, rho summed over the ranks
        self._fused_step_deferred(e, mode=2)
        self._take_sums(self._reducer(self._fold_partials(False).clone()))
        for k in range(n_steps):
            self._field_chain(e, table[k, 0:2], None)   # Poisson, E, diagnostics, level mats
            if v_events is not None:
                v_events[k][0].record(torch.cuda.current_stream())
            last = k + 1 == n_steps
            if last:
                self._fused_step_deferred(e, final=True, mom_out3=self._part[n:])
                self._part[:n].zero_()
                table[k, 2:5].copy_(self._reducer(self._part.clone())[n:])
            else:
                self._fused_step_deferred(e)
                self._take_sums(self._reducer(self._fold_partials(True).clone()), table[k, 2:5])
            if v_events is not None:
                v_events[k][1].record(torch.cuda.current_stream())
        return table

    def step(self):
        """One Strang step (the pipelined path with n_steps = 1)."""
        table = self.advance(1)
        self.t += self.config.dt
        return self._record(self.t, table[0])

    def run(self):
        raise NotImplementedError("PencilShardedSimulation: use advance()/step(); run() "
                                  "needs the global t=0 diagnostics of all ranks' rows")

    # Simulation methods that act on the whole buffer: on a sharded rank the rows of the
    # other ranks are stale, so these would return plausible but wrong physics.
    def _whole_buffer_only(self, *_a, **_k):
        raise NotImplementedError("PencilShardedSimulation: only advance()/step() are valid on "
                                  "a sharded rank (rows of other ranks are not current); "
                                  "read this rank's rows with owned_rows()")

    enqueue_step = step_host = field_solve = diagnostics = advance_graph = _whole_buffer_only
    _lead_x_rho = _xx = _trail_x_mom = _advect_x = _advect_v = _field = _whole_buffer_only
