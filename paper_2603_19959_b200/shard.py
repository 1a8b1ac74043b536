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
The v-sweep is column-local.  The x kernels compute every output from the
same operands in the same order whether the row is periodic or a slab with
halos; the reductions (rho, moments) are deterministic for a given rank count
(fixed chunk and rank order) and agree with the single-device run to round-off.

The state carries its halo margins in place: each buffer is
  [ left margin | local cells | right margin ]
per row (margins rounded up to an even number of doubles so the local part
stays 16-byte aligned); halos are packed and unpacked by libsldg kernels
(per row, upwind side only) and exchanged with torch.distributed P2P (NCCL over
NVLink on GPUs; gloo for the CPU tests of the host logic).
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


class Collectives:
    """The exchanges of a sharded step over torch.distributed (NCCL between the GPUs of a
    box; gloo for CPU tensors in tests).  A sharded advance() is a generator that yields
    requests at its exchange points; `run` services them:

      ("sum", vec)          vec <- sum over ranks in rank order (all-gather + ordered add,
                            never an unordered all-reduce: every rank gets the same bits)
      ("allgather", loc, out, idx)   out <- the ranks' `loc` segments in rank order
      ("halo", bufs, after) P2P with the ring neighbours: bufs = (to_right, to_left,
                            from_left, from_right); `after()` (the unpack) runs on the
                            communication stream once the data is in; resumes with the
                            CUDA event the compute stream must wait on (None on CPU)

    `lockstep(gens)` services the same requests for ranks run one after another on one
    device (tests)."""

    def __init__(self, rank, world, group=None):
        self.rank, self.world, self.group = rank, world, group
        self._comm = None
        self._bufs = {}

    def _buf(self, key, n, like):
        import torch
        b = self._bufs.get(key)
        if b is None or b.numel() < n or b.device != like.device:
            b = torch.empty(n, dtype=like.dtype, device=like.device)
            self._bufs[key] = b
        return b[:n]

    def sum(self, vec):
        import torch.distributed as dist
        if self.world == 1:
            return vec
        parts = self._buf("sum", self.world * vec.numel(), vec)
        dist.all_gather_into_tensor(parts, vec.contiguous().view(-1), group=self.group)
        ordered_sum(parts.view(self.world, -1), vec.view(-1))
        return vec

    def allgather(self, loc, out, idx):
        """`loc` is this rank's segment padded to idx.max_width doubles."""
        import torch.distributed as dist
        if self.world == 1:
            gather_index(loc, idx.index, out)
            return out
        gat = self._buf("ag_out", self.world * idx.max_width, loc)
        dist.all_gather_into_tensor(gat, loc, group=self.group)
        gather_index(gat, idx.index, out)
        return out

    def halo(self, to_right, to_left, from_left, from_right):
        """Send to_right to the right neighbour and to_left to the left one; receive
        from_left from the left neighbour and from_right from the right one (periodic
        ring).  World 1: the slab is its own neighbour."""
        import torch.distributed as dist
        if self.world == 1:
            if to_right.numel():
                from_left.copy_(to_right)
            if to_left.numel():
                from_right.copy_(to_left)
            return
        left, right = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        ops = []
        if to_right.numel():
            ops += [dist.P2POp(dist.isend, to_right, right, self.group),
                    dist.P2POp(dist.irecv, from_left, left, self.group)]
        if to_left.numel():
            ops += [dist.P2POp(dist.isend, to_left, left, self.group),
                    dist.P2POp(dist.irecv, from_right, right, self.group)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def run(self, gen):
        """Drive one rank's advance() generator; returns its value."""
        import torch
        cuda = torch.cuda.is_available()
        try:
            req = next(gen)
            while True:
                kind = req[0]
                res = None
                if kind == "sum":
                    self.sum(req[1])
                elif kind == "allgather":
                    self.allgather(req[1], req[2], req[3])
                elif kind == "halo":
                    (to_r, to_l, fr_l, fr_r), after = req[1], req[2]
                    if cuda and to_r.is_cuda:
                        # the exchange and the unpack on the communication stream, after
                        # the packs; the compute stream waits only where it needs margins
                        if self._comm is None:
                            self._comm = torch.cuda.Stream()
                        packed = torch.cuda.Event()
                        packed.record()
                        with torch.cuda.stream(self._comm):
                            self._comm.wait_event(packed)
                            self.halo(to_r, to_l, fr_l, fr_r)
                            after()
                            res = torch.cuda.Event()
                            res.record()
                    else:
                        self.halo(to_r, to_l, fr_l, fr_r)
                        after()
                else:
                    raise ValueError(f"unknown exchange request {kind!r}")
                req = gen.send(res)
        except StopIteration as stop:
            return stop.value

    @staticmethod
    def lockstep(gens):
        """Drive the advance() generators of ranks 0..W-1 on one device in lockstep:
        every rank runs to its next exchange point, then the exchange is done for all of
        them (same arithmetic as `run` over NCCL).  Returns the ranks' values."""
        import torch
        world = len(gens)
        out = [None] * world
        reqs = []
        for r, g in enumerate(gens):
            try:
                reqs.append(next(g))
            except StopIteration as stop:
                out[r] = stop.value
                reqs.append(None)
        while any(q is not None for q in reqs):
            kinds = {q[0] for q in reqs if q is not None}
            if len(kinds) != 1 or any(q is None for q in reqs):
                raise RuntimeError(f"ranks out of step: {kinds}")
            kind = kinds.pop()
            if kind == "sum":
                parts = torch.stack([q[1].reshape(-1) for q in reqs])
                tot = torch.empty_like(parts[0])
                ordered_sum(parts, tot)
                for q in reqs:
                    q[1].view(-1).copy_(tot)
            elif kind == "allgather":
                cat = torch.cat([q[1] for q in reqs])
                for q in reqs:
                    gather_index(cat, q[3].index, q[2])
            elif kind == "halo":
                for r, q in enumerate(reqs):
                    fr_l, fr_r = q[1][2], q[1][3]
                    left, right = reqs[(r - 1) % world], reqs[(r + 1) % world]
                    if fr_l.numel():
                        fr_l.copy_(left[1][0])
                    if fr_r.numel():
                        fr_r.copy_(right[1][1])
                for q in reqs:
                    q[2]()
            else:
                raise ValueError(f"unknown exchange request {kind!r}")
            nxt = []
            for r, g in enumerate(gens):
                try:
                    nxt.append(g.send(None))
                except StopIteration as stop:
                    out[r] = stop.value
                    nxt.append(None)
            reqs = nxt
        return out


def ordered_sum(parts, out):
    """out[i] = parts[0][i] + parts[1][i] + ... in row order (libsldg, on the device)."""
    from . import _capi
    from ._device import current_stream
    _capi.check(_capi.lib().sldg_sum_parts(parts.data_ptr(), parts.shape[0], parts.shape[1],
                                           out.data_ptr(), current_stream()), ValueError)
    return out


def gather_index(src, idx, out):
    from . import _capi
    from ._device import current_stream
    _capi.check(_capi.lib().sldg_gather_index(src.data_ptr(), idx.data_ptr(), out.numel(),
                                              out.data_ptr(), current_stream()), ValueError)
    return out


class SegmentIndex:
    """Positions of the ranks' segments in an all-gathered buffer padded to the widest."""

    def __init__(self, counts, device):
        import torch
        self.max_width = max(counts)
        pos = np.concatenate([r * self.max_width + np.arange(c) for r, c in enumerate(counts)])
        self.index = torch.from_numpy(pos.astype(np.int64)).to(device)


class HaloPlan:
    """Per-row upwind halo layout of one x plan on a slab (libsldg sldg_halo)."""

    def __init__(self, x_plan, n_local, n_apply):
        import ctypes as C

        from . import _capi
        h = C.c_void_p()
        _capi.check(_capi.lib().sldg_halo_create(x_plan.device_handle(), n_local, n_apply,
                                                 C.byref(h)), ValueError)
        self.h = h.value
        r = np.zeros(2, dtype=np.int64)
        _capi.check(_capi.lib().sldg_halo_reach(self.h, _capi.i64ptr(r)))
        self.reach_l, self.reach_r = int(r[0]), int(r[1])
        self.n_apply = n_apply

    def extent(self, r0, r1):
        from . import _capi
        e = np.zeros(4, dtype=np.int64)
        _capi.check(_capi.lib().sldg_halo_extent(self.h, r0, r1, _capi.i64ptr(e)))
        return [int(v) for v in e]

    def __del__(self):
        try:
            from . import _capi
            _capi.lib().sldg_halo_destroy(self.h)
        except Exception:
            pass


class ShardedSimulation:
    """The Strang step on an x-slab of the state, one rank per GPU.

    The velocity mesh and plans are replicated; the state is split along x into
    contiguous slabs of cells, each row stored as [left margin | local | right margin].
    advance() is pipelined like Simulation.advance(): the trailing half x-step of step k
    and the leading one of step k + 1 run as ONE pass (k_xx_tiles, n_apply = 2) after one
    exchange of doubled upwind halos, so a step is  V (column-local) -> halo exchange ->
    X.X (+ moments of the intermediate, + rho of the result) -> all-gather of rho ->
    Poisson (every rank, the whole x grid) -> E.  The exchange is per row and upwind only
    (sldg_halo_pack/unpack: a row with shift n >= 0 needs 2n + 2 cells from the left, n < 0
    2|n| from the right), split into row chunks: the chunks' NCCL send/recv and unpack run
    on a communication stream while the compute stream runs the X.X of the chunks whose
    margins are in (fewer exchanges, overlapped with the x update).
    The reductions are deterministic for a given rank count (chunk order, rank order).
    """

    def __init__(self, config, rank, world, group=None, mesh=None, n_chunks=4):
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
        if c.dim != 3:
            raise ValueError("x-slab sharding needs the 3V velocity layout")
        self.rank, self.world, self.group = rank, world, group
        self.comm = Collectives(rank, world, group)
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
        self.x_plan = precompute_x_matrices(self.xgrid, self.vcoords[:, 0], 0.5 * c.dt)
        self.x_plan.velocity_order = c.degree + 1   # the row-tile kernel's layout
        self.halo1 = HaloPlan(self.x_plan, self.n_local, 1)
        self.halo2 = HaloPlan(self.x_plan, self.n_local, 2)
        # margins: the doubled reach (X.X), at least 2 cells left / 1 right (the X.X
        # intermediate's halo cells), rounded to an even number of doubles
        self.hl = max(2, self.halo2.reach_l)
        self.hr = max(1, self.halo2.reach_r)
        self.lw, self.rw = margin_dofs(self.hl, o), margin_dofs(self.hr, o)
        width = self.lw + self.n_local * o + self.rw
        self.width = width + (width & 1)
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
        self._segs = SegmentIndex([n * o for n in self.part.counts()], dev)
        # this slab's rho, padded to the widest slab (the all-gather's send buffer)
        self._rho_loc = torch.zeros(self._segs.max_width, dtype=torch.float64, device=dev)
        self._rho = torch.empty(self.xgrid.n_dofs, dtype=torch.float64, device=dev)
        self._phi = torch.empty(self.poisson.n_nodes, dtype=torch.float64, device=dev)
        self._e = torch.empty(self.xgrid.n_dofs, dtype=torch.float64, device=dev)
        self._rec = torch.empty(5, dtype=torch.float64, device=dev)
        # row chunks (whole velocity cells) of the overlapped exchange
        nloc = (c.degree + 1) ** 3
        n_cells = n_v // nloc
        k = max(1, min(int(n_chunks), n_cells))
        bounds = [(i * n_cells // k) * nloc for i in range(k + 1)]
        self.chunks = [(bounds[i], bounds[i + 1]) for i in range(k) if bounds[i + 1] > bounds[i]]
        self._hbuf = {}
        for hp in (self.halo1, self.halo2):
            tot = hp.extent(0, n_v)
            n_r, n_l = tot[1], tot[3]
            self._hbuf[hp.n_apply] = [torch.empty(max(n, 1), dtype=torch.float64, device=dev)
                                      for n in (n_r, n_l, n_r, n_l)]
        import ctypes as C

        from . import _capi
        nb = C.c_size_t()
        _capi.check(_capi.lib().sldg_advect_x_slab_tiles_scratch(
            self.x_plan.device_handle(), self.n_local, self.width, C.byref(nb)), ValueError)
        self._xscratch = torch.empty(nb.value, dtype=torch.uint8, device=dev)
        from ._device import SCRATCH
        SCRATCH.release_with(self.sweep_plan)
        self.t = 0.0

    def fused_step_supported(self) -> bool:
        return False   # the one-pass step needs whole rows; slabs run V and X.X passes

    # views ------------------------------------------------------------------
    def _local(self, buf):
        return buf[:, self.lw:self.lw + self.n_local * self.o]

    @property
    def f(self):
        """Local slab of the state (view into the margin buffer)."""
        return self._local(self._F)

    def _swap(self):
        self._F, self._G = self._G, self._F

    # building blocks --------------------------------------------------------
    def _exchange(self, hp):
        """Generator: pack every chunk, then one "halo" request per chunk; returns the
        per-chunk events the X pass waits on."""
        from . import _capi
        from ._device import current_stream
        lib = _capi.lib()
        to_r, to_l, fr_l, fr_r = self._hbuf[hp.n_apply]
        ext = [hp.extent(r0, r1) for r0, r1 in self.chunks]
        for (r0, r1), e in zip(self.chunks, ext):
            _capi.check(lib.sldg_halo_pack(hp.h, self._F.data_ptr(), self.width, self.lw, r0, r1,
                                           to_r[e[0]:].data_ptr(), to_l[e[2]:].data_ptr(),
                                           current_stream()), ValueError)
        events = []
        for (r0, r1), e in zip(self.chunks, ext):
            bufs = (to_r[e[0]:e[0] + e[1]], to_l[e[2]:e[2] + e[3]],
                    fr_l[e[0]:e[0] + e[1]], fr_r[e[2]:e[2] + e[3]])

            def unpack(r0=r0, r1=r1, e=e):
                _capi.check(lib.sldg_halo_unpack(hp.h, self._F.data_ptr(), self.width, self.lw,
                                                 r0, r1, fr_l[e[0]:].data_ptr(),
                                                 fr_r[e[2]:].data_ptr(), current_stream()),
                            ValueError)
            events.append((yield ("halo", bufs, unpack)))
        return events

    def _x_pass(self, n_apply, events, rho_out=None, mom_out3=None):
        """X (n_apply 1) or X.X (2) of every chunk F -> G, each after its halo event."""
        import torch

        from . import _capi
        from ._device import current_stream
        lib = _capi.lib()
        src_off = self.lw - self.hl * self.o
        for i, (r0, r1) in enumerate(self.chunks):
            if events[i] is not None:
                torch.cuda.current_stream().wait_event(events[i])
            _capi.check(lib.sldg_advect_x_slab_tiles(
                self.x_plan.device_handle(), self._F.data_ptr(), self.width, src_off, self.hl,
                self.hr, self.n_local, self._G.data_ptr(), self.width, self.lw, n_apply, r0,
                r1 - r0, 1 if i else 0, self._vw.data_ptr(), self._v0.data_ptr(),
                self._v2.data_ptr(), self._xw.data_ptr(),
                None if mom_out3 is None else mom_out3.data_ptr(),
                None if rho_out is None else rho_out.data_ptr(), self._xscratch.data_ptr(),
                current_stream()), ValueError)
        self._swap()

    def _v_pass(self, e):
        from .vsweep import advect_velocity_into
        c = self.config
        x0 = self.cell0 * self.o
        advect_velocity_into(self.f, self._local(self._G), e[x0:x0 + self.n_local * self.o],
                             c.dt, self.sweep_plan, c.bc, c.force_slow)
        self._swap()

    def _field(self, e_out, diag2):
        from .xfield import field_diag_into
        self.poisson.solve_into(self._rho, self._phi, e_out)
        if diag2 is not None:
            field_diag_into(self.poisson, e_out, diag2)

    # the pipelined Strang steps ------------------------------------------------
    def advance_steps(self, n_steps, table, v_events=None):
        """Generator form of advance() (exchange points yielded to a Collectives driver);
        v_events[k] = (start, end) CUDA events recorded around step k's v-sweep."""
        import torch
        if n_steps == 0:
            return table
        # leading half x-step of step 0 (+ rho of the slab), rho all-gathered
        ev = yield from self._exchange(self.halo1)
        self._x_pass(1, ev, rho_out=self._rho_loc)
        yield ("allgather", self._rho_loc, self._rho, self._segs)
        for k in range(n_steps):
            self._field(self._e, table[k, 0:2])
            if v_events is not None:
                v_events[k][0].record(torch.cuda.current_stream())
            self._v_pass(self._e)
            if v_events is not None:
                v_events[k][1].record(torch.cuda.current_stream())
            last = k + 1 == n_steps
            hp = self.halo1 if last else self.halo2
            ev = yield from self._exchange(hp)
            mom = table[k, 2:5]
            if last:   # trailing half step (+ moments): the state of the step
                self._x_pass(1, ev, mom_out3=mom)
            else:      # trailing + next leading half steps (+ moments, + rho)
                self._x_pass(2, ev, rho_out=self._rho_loc, mom_out3=mom)
            yield ("sum", mom)
            if not last:
                yield ("allgather", self._rho_loc, self._rho, self._segs)
        return table

    def advance(self, n_steps, table=None, v_events=None):
        """n_steps Strang steps of the slab; row k of the returned (n_steps, 5) table is
        step k's [max|E|, e_field, m0, m1, m2] (global, the same on every rank)."""
        import torch
        if table is None:
            table = torch.empty((n_steps, 5), dtype=torch.float64, device=self._F.device)
        return self.comm.run(self.advance_steps(n_steps, table, v_events))

    def step(self):
        from .driver import DiagnosticsRecord
        table = self.advance(1)
        self.t += self.config.dt
        r = table[0].cpu().numpy()
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
    (Collectives.sum) so all ranks solve the same Poisson problem.  Total work
    is fixed as ranks are added (strong scaling).

    advance() is a generator at heart (advance_steps): its one exchange per step is a
    ("sum", partials) request serviced by a Collectives driver (NCCL across processes,
    or Collectives.lockstep for ranks run on one device in tests).
    """

    def __init__(self, config, rank, world, group=None, mesh=None):
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
        self.comm = Collectives(rank, world, group)
        n = self._f.shape[1]
        self._part = torch.zeros(n + 3, dtype=torch.float64, device=self._f.device)
        self._rho_idx = torch.arange(n, dtype=torch.int64, device=self._f.device)
        self._mom_idx = torch.arange(n, n + 3, dtype=torch.int64, device=self._f.device)

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

    def advance_steps(self, n_steps: int, table, v_events=None):
        """Generator form of advance(): the rank's partial sums [rho | m0 m1 m2] are
        yielded for the rank-order sum, which lands in place; v_events[k] = (start, end)
        events around step k's fused kernel."""
        import torch

        from . import _capi
        from ._device import current_stream
        if n_steps == 0:
            return table
        e = self._e
        n = self._f.shape[1]
        lib = _capi.lib()

        def take_rho():   # the summed rho of all ranks -> this rank's Poisson input
            _capi.check(lib.sldg_gather_index(self._part.data_ptr(), self._rho_idx.data_ptr(),
                                              n, self._rho.data_ptr(), current_stream()))

        # leading half x-step of step 0 on my tiles, rho summed over the ranks
        self._fused_step_deferred(e, mode=2)
        self._fold_partials(False)
        yield ("sum", self._part)
        take_rho()
        for k in range(n_steps):
            self._field_chain(e, table[k, 0:2], None)   # Poisson, E, diagnostics, level mats
            last = k + 1 == n_steps
            if v_events is not None:
                v_events[k][0].record(torch.cuda.current_stream())
            if last:
                self._fused_step_deferred(e, final=True, mom_out3=self._part[n:])
                if v_events is not None:
                    v_events[k][1].record(torch.cuda.current_stream())
                yield ("sum", self._part[n:])
            else:
                self._fused_step_deferred(e)
                if v_events is not None:
                    v_events[k][1].record(torch.cuda.current_stream())
                self._fold_partials(True)
                yield ("sum", self._part)
                take_rho()
            _capi.check(lib.sldg_gather_index(self._part.data_ptr(), self._mom_idx.data_ptr(),
                                              3, table[k, 2:5].data_ptr(), current_stream()))
        return table

    def advance(self, n_steps: int, table=None, v_events=None):
        """n_steps pipelined Strang steps on this rank's tiles; row k of the returned
        table is step k's [max|E|, e_field, m0, m1, m2] (global, identical on all ranks)."""
        import torch
        if table is None:
            table = torch.empty((n_steps, 5), dtype=torch.float64, device=self._f.device)
        return self.comm.run(self.advance_steps(n_steps, table, v_events))

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
