"""Hybrid fast/slow v-sweep: the drop-in for `sldg_vlasov.vsweep` (vsweep.py:1-441).

Host side: group congruent pencils exactly like build_sweep_plan
(vsweep.py:307-387) and upload the CSR pencil structure once per device
(sldg_vplan_create).  Every sweep runs on the GPU (csrc/vsweep.cu):
per-column level matrices, whole-pencil fast walk, per-cell fast / slow path
and the deterministic weighted write-back.  There is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .basis import DGBasis
from .pencil import PencilSet
from .sldg1d import (ABSORBING, PERIODIC, OverlapPair, ShiftDecomposition, check_bc,  # noqa: F401
                     decompose_shift, overlap_pairs_device)   # (module names as in vsweep.py)
from .tensor import TensorPermutation
from .vmesh import VelocityMesh


class SweepError(RuntimeError):
    pass


@dataclass(frozen=True)
class LevelMatrices:
    """Per-level shift decompositions and overlap pairs (vsweep.py:36-44)."""

    speed: float
    dt: float
    n_shift: tuple
    frac: tuple
    pairs: tuple


def precompute_level_matrices(basis: DGBasis, speed: float, dt: float, base_width: float,
                              n_levels: int) -> LevelMatrices:
    """Level l uses width base_width/2^l (vsweep.py:47-61); pairs built on the device."""
    ds = [decompose_shift(speed, dt, base_width / 2 ** lev) for lev in range(n_levels)]
    A, B = overlap_pairs_device(basis, [d.frac for d in ds])
    pairs = tuple(OverlapPair(A[k], B[k], ds[k].frac) for k in range(n_levels))
    return LevelMatrices(speed, dt, tuple(d.n_shift for d in ds), tuple(d.frac for d in ds),
                         pairs)


@dataclass
class _PencilGroup:
    """Congruent pencils (vsweep.py:275-291); gather arrays are built on demand."""

    lowers: np.ndarray
    widths: np.ndarray
    levels: np.ndarray
    conforming: np.ndarray
    n_lines: int
    n_cells: int
    pencils: np.ndarray                  # pencil ids in plan order
    cell_ids: np.ndarray                 # (n_pencils_in_group, n_cells)
    cell_weights: np.ndarray             # (n_pencils_in_group, n_cells)
    _lines: np.ndarray = field(repr=False, default=None)
    _n_local: int = 0

    @property
    def gather(self) -> np.ndarray:
        base = self.cell_ids[:, None, :, None] * self._n_local
        g = base + self._lines[None, :, None, :]
        return g.reshape(self.n_lines, self.n_cells * self._lines.shape[1]).astype(np.int64)

    @property
    def simple(self) -> bool:
        return bool((self.cell_weights == 1.0).all())

    # the reference's copy / accumulate partition of the flat positions (vsweep.py:285-291,
    # 366-383); the device plan carries the same information as its target CSR
    @property
    def flat_weights(self) -> np.ndarray:
        o = self._lines.shape[1]
        w = np.broadcast_to(self.cell_weights[:, None, :, None],
                            (self.cell_weights.shape[0], self._lines.shape[0],
                             self.n_cells, o))
        return np.ascontiguousarray(w).reshape(self.n_lines, self.n_cells * o)

    @property
    def copy_pos(self) -> np.ndarray:
        return np.nonzero(self.flat_weights.ravel() == 1.0)[0]

    @property
    def copy_targets(self) -> np.ndarray:
        return self.gather.ravel()[self.copy_pos]

    @property
    def acc_pos(self) -> np.ndarray:
        return np.nonzero(self.flat_weights.ravel() != 1.0)[0]

    @property
    def acc_targets(self) -> np.ndarray:
        return self.gather.ravel()[self.acc_pos]

    @property
    def acc_weights(self) -> np.ndarray:
        return self.flat_weights.ravel()[self.acc_pos]


class SweepPlan:
    """Static plan for one sweep direction (vsweep.py:294-304) + its device image."""

    def __init__(self, direction, basis, radius, base_width, n_levels, n_dofs, groups, dim,
                 n_cells, desc_arrays):
        self.direction = direction
        self.basis = basis
        self.radius = radius
        self.base_width = base_width
        self.n_levels = n_levels
        self.n_dofs = n_dofs
        self.groups = groups
        self.dim = dim
        self.n_cells = n_cells
        self._arrays = desc_arrays
        self._dev = {}

    # -- device image ------------------------------------------------------
    def device_handle(self):
        from ._device import device
        dev = device()
        key = dev.index
        h = self._dev.get(key)
        if h is None:
            a = self._arrays
            ba = _capi.BasisArrays(self.basis)
            desc = _capi.SldgVPlanDesc(
                ba.struct, self.dim, self.direction, self.n_levels, float(self.radius),
                float(self.base_width), self.n_cells, len(a["offsets"]) - 1,
                _capi.i64ptr(a["offsets"]), _capi.i64ptr(a["group"]),
                _capi.i64ptr(a["cell_ids"]), _capi.dptr(a["lowers"]), _capi.dptr(a["widths"]),
                _capi.i64ptr(a["levels"]), _capi.u8ptr(a["conforming"]),
                _capi.dptr(a["weights"]))
            out = C.c_void_p()
            _capi.check(_capi.lib().sldg_vplan_create(C.byref(desc), C.byref(out)), SweepError)
            h = out.value
            self._dev[key] = h
        return h

    def scratch_bytes(self, n_cols):
        n = C.c_size_t()
        _capi.check(_capi.lib().sldg_vplan_scratch_bytes(self.device_handle(), n_cols,
                                                         C.byref(n)))
        return n.value

    def info(self):
        out = np.zeros(5, dtype=np.int64)
        _capi.check(_capi.lib().sldg_vplan_info(self.device_handle(), _capi.i64ptr(out)))
        return dict(n_entries=int(out[0]), n_acc_slots=int(out[1]), n_targets=int(out[2]),
                    n_walk_pencils=int(out[3]), n_dofs=int(out[4]))

    def __del__(self):
        try:
            lib = _capi.lib()
            for h in self._dev.values():
                lib.sldg_vplan_destroy(h)
        except Exception:
            pass


def build_sweep_plan(mesh: VelocityMesh, pset: PencilSet, perm: TensorPermutation,
                     basis: DGBasis) -> SweepPlan:
    """Group congruent pencils in first-seen order (vsweep.py:307-387)."""
    o = basis.n_nodes
    n_local = perm.n_local
    lines = perm.lines[pset.direction]
    keyed = {}
    for q in range(pset.n_pencils):
        sl = pset.pencil_slice(q)
        k = (pset.levels[sl].tobytes(), pset.lowers[sl].tobytes(), pset.widths[sl].tobytes(),
             pset.conforming[sl].tobytes())
        keyed.setdefault(k, []).append(q)
    groups = []
    order = []
    for qs in keyed.values():
        qs = np.asarray(qs, dtype=np.int64)
        sl0 = pset.pencil_slice(int(qs[0]))
        n_cells = sl0.stop - sl0.start
        starts = pset.offsets[qs]
        idx = starts[:, None] + np.arange(n_cells)[None, :]
        groups.append(_PencilGroup(
            lowers=pset.lowers[sl0].copy(), widths=pset.widths[sl0].copy(),
            levels=pset.levels[sl0].copy(), conforming=pset.conforming[sl0].copy(),
            n_lines=len(qs) * len(lines), n_cells=n_cells, pencils=qs,
            cell_ids=pset.cell_ids[idx], cell_weights=pset.weights[idx],
            _lines=lines, _n_local=n_local))
        order.append(qs)
    n_dofs = mesh.n_cells * n_local
    counts = np.bincount(pset.cell_ids, minlength=mesh.n_cells)
    if (counts == 0).any():
        raise SweepError("sweep plan leaves velocity DOFs uncovered")
    # device CSR in plan order: groups in order, pencils of a group in order
    qorder = np.concatenate(order)
    gid = np.concatenate([np.full(len(q), k, dtype=np.int64) for k, q in enumerate(order)])
    lens = np.diff(pset.offsets)[qorder]
    offsets = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    ent = np.concatenate([np.arange(pset.offsets[q], pset.offsets[q + 1]) for q in qorder])
    arrays = dict(
        offsets=offsets, group=gid,
        cell_ids=np.ascontiguousarray(pset.cell_ids[ent], dtype=np.int64),
        lowers=np.ascontiguousarray(pset.lowers[ent], dtype=np.float64),
        widths=np.ascontiguousarray(pset.widths[ent], dtype=np.float64),
        levels=np.ascontiguousarray(pset.levels[ent], dtype=np.int64),
        conforming=np.ascontiguousarray(pset.conforming[ent], dtype=np.uint8),
        weights=np.ascontiguousarray(pset.weights[ent], dtype=np.float64))
    return SweepPlan(pset.direction, basis, mesh.radius, mesh.base_width,
                     int(mesh.levels.max()) + 1, n_dofs, groups, mesh.dim, mesh.n_cells, arrays)


@dataclass(frozen=True)
class GeneralizedOverlap:
    """Projection block of one source cell onto one destination cell (vsweep.py:64-74):
    `matrix` includes M^-1; [lo, hi] is the foot/source overlap in foot coordinates."""

    matrix: np.ndarray
    lo: float
    hi: float


def generalized_overlap(basis: DGBasis, dest_lo: float, dest_width: float, src_lo: float,
                        src_width: float, displacement: float) -> GeneralizedOverlap:
    """Cross-size projection block (vsweep.py:98-122), evaluated on the device by the slow
    path's own block routine (csrc/vsweep.cu general_block)."""
    import torch

    from ._device import current_stream, device
    if dest_width <= 0 or src_width <= 0:
        raise ValueError("cell widths must be positive")
    o = basis.n_nodes
    foot_lo = dest_lo - displacement
    vl = max(foot_lo, src_lo)
    vr = min(foot_lo + dest_width, src_lo + src_width)
    if vr <= vl:
        return GeneralizedOverlap(np.zeros((o, o)), vl, vl)
    m = torch.empty((o, o), dtype=torch.float64, device=device())
    ba = _capi.BasisArrays(basis)
    _capi.check(_capi.lib().sldg_generalized_overlap(
        ba.struct, float(vl), float(vr), float(dest_lo), float(dest_width), float(src_lo),
        float(src_width), float(displacement), m.data_ptr(), current_stream()), ValueError)
    return GeneralizedOverlap(m.cpu().numpy(), vl, vr)


def weighted_writeback(f_in, gather, weights, values):
    """f_out = f_in + sum over contributions of w (value - f_in), a copy where w == 1
    (vsweep.py:249-272), on the device with numpy's order: copies in flat order, then
    the weighted deltas summed per element in flat order."""
    import torch

    from ._device import current_stream, device
    f = np.ascontiguousarray(np.asarray(f_in, dtype=float))
    g = np.asarray(gather, dtype=np.int64).ravel()
    w = np.ascontiguousarray(np.asarray(weights, dtype=float).ravel())
    v = np.ascontiguousarray(np.asarray(values, dtype=float).ravel())
    if not (g.size == w.size == v.size):
        raise ValueError("gather, weights and values must be aligned")
    counts = np.bincount(g, minlength=f.size)
    if (counts == 0).any():
        missing = int(np.nonzero(counts == 0)[0][0])
        raise SweepError(f"element {missing} has zero total write-back weight")
    order = np.argsort(g, kind="stable").astype(np.int64)   # per element, flat order
    off = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    dev = device()
    fd = torch.from_numpy(f.ravel().copy()).to(dev)
    out = torch.empty_like(fd)
    args = [torch.from_numpy(a).to(dev) for a in (off, order, w, v)]
    _capi.check(_capi.lib().sldg_weighted_writeback(
        fd.data_ptr(), f.size, args[0].data_ptr(), args[1].data_ptr(), args[2].data_ptr(),
        args[3].data_ptr(), out.data_ptr(), current_stream()), SweepError)
    return out.cpu().numpy().reshape(f.shape)


def sweep_pencil(values, lowers, widths, levels, conforming, speed, dt, lm: LevelMatrices, bc,
                 radius, basis: DGBasis, force_slow: bool = False):
    """Hybrid SLDG update of one pencil batched over leading axes (vsweep.py:173-246).

    Runs the device sweep of a one-pencil plan (the same kernels as advect_velocity:
    whole-pencil fast path, per-cell fast path, slow path); the batch becomes the
    plan's columns.  The level matrices are rebuilt on the device from
    (speed, dt, base width), i.e. `lm` must be precompute_level_matrices(basis, speed,
    dt, ...) as in the reference; only its level count is read.
    """
    import torch

    from ._device import device
    check_bc(bc)
    values = np.asarray(values, dtype=float)
    lowers = np.ascontiguousarray(np.asarray(lowers, dtype=np.float64))
    widths = np.ascontiguousarray(np.asarray(widths, dtype=np.float64))
    levels = np.ascontiguousarray(np.asarray(levels, dtype=np.int64))
    conforming = np.asarray(conforming, dtype=bool)
    n, o = len(lowers), basis.n_nodes
    if values.shape[-2:] != (n, o):
        raise SweepError(f"pencil values shaped {values.shape[-2:]}, expected ({n}, {o})")
    lead = values.shape[:-2]
    nb = int(np.prod(lead)) if lead else 1
    if nb == 0 or n == 0:
        return np.zeros(values.shape)
    base_width = float(widths[0] * 2.0 ** int(levels[0]))
    arrays = dict(offsets=np.array([0, n], dtype=np.int64), group=np.zeros(1, dtype=np.int64),
                  cell_ids=np.arange(n, dtype=np.int64), lowers=lowers, widths=widths,
                  levels=levels, conforming=conforming.astype(np.uint8),
                  weights=np.ones(n, dtype=np.float64))
    n_levels = max(len(lm.n_shift), int(levels.max()) + 1)
    plan = SweepPlan(0, basis, float(radius), base_width, n_levels, n * o, [], 1, n, arrays)
    dev = device()
    # state layout (rows = cell*o + node, columns = batch)
    f = torch.from_numpy(np.ascontiguousarray(values.reshape(nb, n * o).T)).to(dev)
    out = torch.empty_like(f)
    sp = torch.full((nb,), float(speed), dtype=torch.float64, device=dev)
    scratch = torch.empty(max(plan.scratch_bytes(nb), 256), dtype=torch.uint8, device=dev)
    from ._device import current_stream
    _capi.check(_capi.lib().sldg_advect_v(
        plan.device_handle(), f.data_ptr(), out.data_ptr(), nb, nb, sp.data_ptr(), float(dt),
        _capi.BC_CODE[bc], int(bool(force_slow)), scratch.data_ptr(), current_stream()),
        SweepError)
    return out.cpu().numpy().T.reshape(values.shape)


def advect_velocity_into(f_in, f_out, speeds, dt, plan: SweepPlan, bc=ABSORBING,
                         force_slow=False):
    """Device-resident sweep f_out = V(f_in) (torch CUDA fp64 buffers, no host sync)."""
    from ._device import SCRATCH, current_stream
    n_cols = f_in.shape[1]
    scratch = SCRATCH.get(("vsweep", id(plan)), plan.scratch_bytes(n_cols))
    _capi.check(_capi.lib().sldg_advect_v(
        plan.device_handle(), f_in.data_ptr(), f_out.data_ptr(), f_in.stride(0), n_cols,
        speeds.data_ptr(), float(dt), _capi.BC_CODE[bc], int(bool(force_slow)),
        scratch.data_ptr(), current_stream()), SweepError)
    return f_out


def advect_velocity(f, speeds, dt, plan: SweepPlan, bc: str = ABSORBING, workers: int = 1,
                    force_slow: bool = False):
    """Advect every x column along the plan's direction, in place (vsweep.py:413-441).

    `f` is a (n_velocity_dofs, n_x_dofs) float64 array: a torch CUDA tensor
    (device-resident, updated in place) or a numpy array (copied to the GPU,
    swept, copied back into `f`).  Columns with exactly zero speed keep their
    bits.  `workers` is accepted for API compatibility (results never depend
    on scheduling).
    """
    import torch

    from ._device import SCRATCH, is_device_tensor, to_device_f64
    check_bc(bc)
    shape = tuple(f.shape)
    sp_np = None if is_device_tensor(speeds) else np.asarray(speeds, dtype=float).ravel()
    n_sp = speeds.numel() if sp_np is None else sp_np.size
    if shape != (plan.n_dofs, n_sp):
        raise SweepError(f"field shaped {shape}, expected ({plan.n_dofs}, {n_sp})")
    if sp_np is not None and not (sp_np != 0.0).any():
        return f
    if not dt > 0.0:
        raise ValueError(f"time step must be positive, got {dt}")
    sp_d = to_device_f64(speeds if sp_np is None else sp_np)
    if is_device_tensor(f):
        if f.dtype != torch.float64 or f.stride(1) != 1:
            raise SweepError("device field must be float64 with unit column stride")
        out = SCRATCH.like(("vsweep_out", id(plan)), f)
        advect_velocity_into(f, out, sp_d, dt, plan, bc, force_slow)
        f.copy_(out)
        return f
    fd = to_device_f64(f)
    out = torch.empty_like(fd)
    advect_velocity_into(fd, out, sp_d, dt, plan, bc, force_slow)
    np.copyto(f, out.cpu().numpy())
    return f
