"""Spatial side: x-advection, charge density, 1D Poisson (drop-in for xfield.py:1-195).

Host setup (grid, unique speeds, FE stiffness assembly and its inverse) runs
once; every per-step operation runs on the GPU (csrc/xfield.cu).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from .basis import DGBasis
from .sldg1d import OverlapPair, ShiftDecomposition, decompose_shift, overlap_pairs_device


class XGrid:
    """Uniform periodic DG x grid (xfield.py:22-45)."""

    def __init__(self, n_cells: int, degree: int, length: float):
        if n_cells < 4:
            raise ValueError(f"need at least 4 x-cells, got {n_cells}")
        if length <= 0:
            raise ValueError(f"domain length must be positive, got {length}")
        self.n_cells = int(n_cells)
        self.length = float(length)
        self.basis = DGBasis(degree)
        self.degree = self.basis.degree
        self.h = self.length / self.n_cells
        lowers = np.arange(self.n_cells) * self.h
        self.node_coords = lowers[:, None] + 0.5 * (self.basis.nodes + 1.0) * self.h
        self.dof_coords = self.node_coords.ravel()
        self.dof_weights = np.tile(0.5 * self.h * self.basis.weights, self.n_cells)

    @property
    def n_dofs(self) -> int:
        return self.n_cells * (self.degree + 1)


@dataclass(frozen=True)
class _SpeedGroup:
    rows: np.ndarray
    decomp: ShiftDecomposition
    pair: OverlapPair


class XAdvectionPlan:
    """Rows grouped by unique speed (xfield.py:54-79); matrices live on the device."""

    def __init__(self, xgrid: XGrid, uniq, inverse, dt):
        self.xgrid = xgrid
        self.n_cells = xgrid.n_cells
        self.uniq = np.ascontiguousarray(uniq, dtype=np.float64)
        self.inverse = np.ascontiguousarray(inverse, dtype=np.int32)
        self.dt = float(dt)
        self._groups = None
        self._dev = {}

    @property
    def groups(self):
        if self._groups is None:
            ds = [decompose_shift(u, self.dt, self.xgrid.h) for u in self.uniq]
            A, B = overlap_pairs_device(self.xgrid.basis, [d.frac for d in ds])
            self._groups = tuple(
                _SpeedGroup(np.nonzero(self.inverse == u)[0], ds[u],
                            OverlapPair(A[u], B[u], ds[u].frac)) for u in range(len(ds)))
        return self._groups

    def device_handle(self):
        from ._device import device
        key = device().index
        h = self._dev.get(key)
        if h is None:
            ba = _capi.BasisArrays(self.xgrid.basis)
            desc = _capi.SldgXPlanDesc(ba.struct, self.xgrid.n_cells, float(self.xgrid.h),
                                       self.dt, len(self.inverse), len(self.uniq),
                                       _capi.dptr(self.uniq), _capi.i32ptr(self.inverse))
            out = C.c_void_p()
            _capi.check(_capi.lib().sldg_xplan_create(C.byref(desc), C.byref(out)), ValueError)
            h = out.value
            if getattr(self, "velocity_order", None):
                # rows are velocity cells x o^3 with one speed per (cell, v_x node):
                # enables the same-speed row-tile kernel (verified by the library)
                _capi.lib().sldg_xplan_set_vlayout(h, int(self.velocity_order))
            self._dev[key] = h
        return h

    def halo(self):
        lr = np.zeros(2, dtype=np.int64)
        _capi.check(_capi.lib().sldg_xplan_halo(self.device_handle(), _capi.i64ptr(lr)))
        return int(lr[0]), int(lr[1])

    def __del__(self):
        try:
            lib = _capi.lib()
            for h in self._dev.values():
                lib.sldg_xplan_destroy(h)
        except Exception:
            pass


def precompute_x_matrices(xgrid: XGrid, speeds, dt: float) -> XAdvectionPlan:
    """One shift/pair per distinct speed (xfield.py:63-79)."""
    speeds = np.asarray(speeds, dtype=float)
    if not np.isfinite(speeds).all():
        raise ValueError("advection speeds must be finite")
    if not dt > 0.0:
        raise ValueError(f"time step must be positive, got {dt}")
    uniq, inverse = np.unique(speeds, return_inverse=True)
    return XAdvectionPlan(xgrid, uniq, inverse.ravel(), dt)


def advect_x_into(f_in, f_out, plan: XAdvectionPlan):
    """Device-resident periodic x update f_out = X(f_in) (no host sync)."""
    from ._device import current_stream
    _capi.check(_capi.lib().sldg_advect_x(plan.device_handle(), f_in.data_ptr(),
                                          f_out.data_ptr(), f_in.stride(0), current_stream()),
                ValueError)
    return f_out


def advect_x_fused_into(f_in, f_out, plan: XAdvectionPlan, n_apply=1, mom=None, rho=None):
    """f_out = X^n_apply(f_in) with fused epilogues (csrc/xx_tiles.cuh k_xx_tiles).

    mom = (w, v0, v2, xw, out3): moments of the state after the first
    application; rho = (w, out): charge density of the final state.  All
    device tensors; enqueue only.
    """
    from ._device import SCRATCH, current_stream
    lib = _capi.lib()
    h = plan.device_handle()
    nb = C.c_size_t()
    _capi.check(lib.sldg_xadv_scratch_bytes(h, C.byref(nb)))
    scratch = SCRATCH.get(("xadv", id(plan)), nb.value) if (mom or rho) else None
    w = (mom[0] if mom else rho[0]) if (mom or rho) else None
    _capi.check(lib.sldg_advect_x_fused(
        h, f_in.data_ptr(), f_out.data_ptr(), f_in.stride(0), int(n_apply),
        w.data_ptr() if w is not None else None,
        mom[1].data_ptr() if mom else None, mom[2].data_ptr() if mom else None,
        mom[3].data_ptr() if mom else None, mom[4].data_ptr() if mom else None,
        rho[1].data_ptr() if rho else None,
        scratch.data_ptr() if scratch is not None else None, current_stream()), ValueError)
    return f_out


def advect_x(f, plan: XAdvectionPlan, workers: int = 1):
    """Periodic SLDG x update of every velocity row, in place (xfield.py:91-104)."""
    import torch

    from ._device import SCRATCH, is_device_tensor, to_device_f64
    if tuple(f.shape) != (len(plan.inverse), plan.xgrid.n_dofs):
        raise ValueError(f"field shaped {tuple(f.shape)}, expected "
                         f"({len(plan.inverse)}, {plan.xgrid.n_dofs})")
    if is_device_tensor(f):
        if f.dtype != torch.float64 or f.stride(1) != 1:
            raise ValueError("device field must be float64 with unit column stride")
        out = SCRATCH.like(("xadv_out", id(plan)), f)
        advect_x_into(f, out, plan)
        f.copy_(out)
        return f
    fd = to_device_f64(f)
    out = torch.empty_like(fd)
    advect_x_into(fd, out, plan)
    np.copyto(f, out.cpu().numpy())
    return f


def rho_into(f, w_dev, rho_out):
    """Device charge density rho_out = w . f (deterministic two-stage reduction)."""
    from ._device import SCRATCH, current_stream
    n_rows, n_cols = f.shape
    nb = C.c_size_t()
    _capi.check(_capi.lib().sldg_rho_scratch_bytes(n_rows, n_cols, C.byref(nb)))
    scratch = SCRATCH.get("rho", nb.value)
    _capi.check(_capi.lib().sldg_rho(f.data_ptr(), f.stride(0), n_rows, n_cols, w_dev.data_ptr(),
                                     rho_out.data_ptr(), scratch.data_ptr(), current_stream()),
                ValueError)
    return rho_out


def compute_rho(f, velocity_weights):
    """rho at the x DOFs = velocity quadrature of f (xfield.py:107-109)."""
    import torch

    from ._device import is_device_tensor, to_device_f64
    host = not is_device_tensor(f)
    fd = to_device_f64(f)
    w = to_device_f64(velocity_weights)
    if w.numel() != fd.shape[0]:
        raise ValueError("velocity weights / field shape mismatch")
    rho = torch.empty(fd.shape[1], dtype=torch.float64, device=fd.device)
    rho_into(fd, w, rho)
    return rho.cpu().numpy() if host else rho


class PoissonSolver:
    """Periodic -phi'' = rho - mean(rho) on continuous FE, zero-mean (xfield.py:112-179).

    The augmented system [[K, m], [m^T, 0]] is assembled and inverted once on
    the host (setup, like the reference's one-time LU); each solve runs on the
    GPU: rhs assembly, G b (warp-per-row GEMV, G = leading block of the
    inverse), E = -phi' at the DG nodes.
    """

    def __init__(self, xgrid: XGrid):
        self.xgrid = xgrid
        basis = xgrid.basis
        p = xgrid.degree
        n_nodes = xgrid.n_cells * p
        self.n_nodes = n_nodes
        cells = np.arange(xgrid.n_cells)
        self.conn = (cells[:, None] * p + np.arange(p + 1)[None, :]) % n_nodes
        local = (2.0 / xgrid.h) * basis.diff.T @ (basis.weights[:, None] * basis.diff)
        k = np.zeros((n_nodes, n_nodes))
        for c in range(xgrid.n_cells):
            k[np.ix_(self.conn[c], self.conn[c])] += local
        lumped = np.zeros(n_nodes)
        np.add.at(lumped, self.conn.ravel(), np.tile(0.5 * xgrid.h * basis.weights, xgrid.n_cells))
        aug = np.zeros((n_nodes + 1, n_nodes + 1))
        aug[:n_nodes, :n_nodes] = k
        aug[:n_nodes, n_nodes] = lumped
        aug[n_nodes, :n_nodes] = lumped
        self._stiffness = k
        self._lumped = lumped
        self._green = np.ascontiguousarray(np.linalg.inv(aug)[:n_nodes, :n_nodes])
        self._dev = {}

    def device_handle(self):
        from ._device import device
        key = device().index
        h = self._dev.get(key)
        if h is None:
            xg = self.xgrid
            xw = np.ascontiguousarray(xg.dof_weights, dtype=np.float64)
            D = np.ascontiguousarray(xg.basis.diff, dtype=np.float64)
            desc = _capi.SldgPoissonDesc(xg.degree, xg.n_cells, float(xg.h), float(xg.length),
                                         _capi.dptr(xw), _capi.dptr(D), _capi.dptr(self._green))
            out = C.c_void_p()
            _capi.check(_capi.lib().sldg_poisson_create(C.byref(desc), C.byref(out)), ValueError)
            h = out.value
            self._dev[key] = h
        return h

    def __del__(self):
        try:
            lib = _capi.lib()
            for h in self._dev.values():
                lib.sldg_poisson_destroy(h)
        except Exception:
            pass

    # device path -----------------------------------------------------------
    def solve_into(self, rho_dev, phi_dev, e_dev):
        from ._device import current_stream
        _capi.check(_capi.lib().sldg_poisson_solve(
            self.device_handle(), rho_dev.data_ptr(),
            phi_dev.data_ptr() if phi_dev is not None else None,
            e_dev.data_ptr() if e_dev is not None else None, current_stream()), ValueError)

    def solve(self, rho):
        """Mean-zero potential at the FE nodes (xfield.py:157-164)."""
        import torch

        from ._device import is_device_tensor, to_device_f64
        host = not is_device_tensor(rho)
        r = to_device_f64(rho)
        if r.numel() != self.xgrid.n_dofs:
            raise ValueError("rho has the wrong length")
        phi = torch.empty(self.n_nodes, dtype=torch.float64, device=r.device)
        self.solve_into(r, phi, None)
        return phi.cpu().numpy() if host else phi

    def electric_field(self, phi):
        """E = -phi' at the DG GLL nodes, per-element derivative (xfield.py:170-179)."""
        import torch

        from ._device import current_stream, is_device_tensor, to_device_f64
        host = not is_device_tensor(phi)
        ph = to_device_f64(phi)
        e = torch.empty(self.xgrid.n_dofs, dtype=torch.float64, device=ph.device)
        _capi.check(_capi.lib().sldg_poisson_efield(self.device_handle(), ph.data_ptr(),
                                                    e.data_ptr(), current_stream()), ValueError)
        return e.cpu().numpy() if host else e

    # host diagnostics (test helpers of the reference, not on the transport path)
    def rhs(self, rho):
        rho = np.asarray(rho, dtype=float)
        rho_bar = (self.xgrid.dof_weights @ rho) / self.xgrid.length
        b = np.zeros(self.n_nodes)
        np.add.at(b, self.conn.ravel(), self.xgrid.dof_weights * (rho - rho_bar))
        return b

    def residual(self, phi, rho):
        return self._stiffness @ np.asarray(phi, dtype=float) - self.rhs(rho)


def solve_poisson(rho, xgrid: XGrid):
    return PoissonSolver(xgrid).solve(rho)


def compute_E(phi, xgrid: XGrid):
    return PoissonSolver(xgrid).electric_field(phi)


_DIAG_SOLVERS = {}


def field_diag_into(solver: PoissonSolver, e_dev, out2_dev):
    """[max|E|, 0.5 w.E^2] on the device (driver.py:220-229, xfield.py:192-195)."""
    from ._device import current_stream
    _capi.check(_capi.lib().sldg_field_diag(solver.device_handle(), e_dev.data_ptr(),
                                            out2_dev.data_ptr(), current_stream()), ValueError)


def field_energy(e_field, xgrid: XGrid) -> float:
    """One half the GLL quadrature of E^2 (xfield.py:192-195), on the device."""
    import torch

    from ._device import to_device_f64
    key = (xgrid.n_cells, xgrid.degree, xgrid.length)
    solver = _DIAG_SOLVERS.get(key)
    if solver is None:
        solver = _DIAG_SOLVERS[key] = PoissonSolver(xgrid)
    e = to_device_f64(e_field)
    out = torch.empty(2, dtype=torch.float64, device=e.device)
    field_diag_into(solver, e, out)
    return float(out[1].item())
