"""1D SLDG pieces of the public API (sldg_vlasov.sldg1d, sldg1d.py:18-100).

`decompose_shift` is the scalar split every kernel restates on the device
(bit-identical, csrc/sldg_common.cuh split_shift); `overlap_pair` evaluates
the A/B projection blocks ON THE DEVICE through sldg_overlap_pairs -- the same
code the sweep kernels run per column and level.  `apply_update` and
`projection_oracle` (sldg1d.py:124-178) run as kernels too (csrc/pencil_ops.cu).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PERIODIC = "periodic"
ABSORBING = "absorbing"

_ONE_MINUS_ULP = float(np.nextafter(1.0, 0.0))


def check_bc(bc: str) -> str:
    if bc not in (PERIODIC, ABSORBING):
        raise ValueError(f"boundary mode must be {PERIODIC!r} or {ABSORBING!r}, got {bc!r}")
    return bc


def shifted_source(values: np.ndarray, k: int, bc: str) -> np.ndarray:
    """out[..., i, :] = values[..., i - k, :] (sldg1d.py:103-121): a wrap (periodic) or a
    zero-filled shift (absorbing) of the cell axis -- index bookkeeping of the
    reference's apply_update, which itself runs on the device here."""
    values = np.asarray(values)
    n = values.shape[-2]
    if bc == PERIODIC:
        return np.roll(values, k, axis=-2)
    if k == 0:
        return values
    out = np.zeros_like(values)
    if 0 < k < n:
        out[..., k:, :] = values[..., :n - k, :]
    elif 0 < -k < n:
        out[..., :n + k, :] = values[..., -k:, :]
    return out


@dataclass(frozen=True)
class ShiftDecomposition:
    n_shift: int
    frac: float


def decompose_shift(speed: float, dt: float, width: float) -> ShiftDecomposition:
    """speed*dt/width = n + frac, frac in [0, 1), 1-ulp fold (sldg1d.py:39-55)."""
    if width <= 0.0:
        raise ValueError(f"cell width must be positive, got {width}")
    if dt <= 0.0:
        raise ValueError(f"time step must be positive, got {dt}")
    r = speed * dt / width
    n = math.floor(r)
    frac = r - n
    if frac >= _ONE_MINUS_ULP:
        return ShiftDecomposition(n + 1, 0.0)
    return ShiftDecomposition(n, frac)


@dataclass(frozen=True)
class OverlapPair:
    same: np.ndarray
    neighbor: np.ndarray
    frac: float


def overlap_pairs_device(basis, fracs):
    """A/B blocks for many fractional shifts, computed by the CUDA kernel."""
    import torch

    from . import _capi
    from ._device import current_stream, device

    fr = np.ascontiguousarray(np.asarray(fracs, dtype=np.float64).ravel())
    if fr.size and (fr.min() < 0.0 or fr.max() >= 1.0):
        raise ValueError("fractional shift must lie in [0, 1)")
    o = basis.degree + 1
    dev = device()
    f_d = torch.from_numpy(fr).to(dev)
    A = torch.empty((fr.size, o, o), dtype=torch.float64, device=dev)
    B = torch.empty_like(A)
    ba = _capi.BasisArrays(basis)
    _capi.check(_capi.lib().sldg_overlap_pairs(ba.struct, f_d.data_ptr(), fr.size, A.data_ptr(),
                                               B.data_ptr(), current_stream()), ValueError)
    return A.cpu().numpy(), B.cpu().numpy()


def overlap_pair(basis, frac: float) -> OverlapPair:
    """Same/neighbour blocks for one fractional shift (sldg1d.py:82-100), on device."""
    if not 0.0 <= frac < 1.0:
        raise ValueError(f"fractional shift must lie in [0, 1), got {frac}")
    A, B = overlap_pairs_device(basis, [frac])
    return OverlapPair(A[0], B[0], float(frac))


def apply_update(values, decomp: ShiftDecomposition, pair: OverlapPair, bc: str = PERIODIC):
    """One SLDG step on a uniform pencil, on the device (apply_update, sldg1d.py:124-136).

    `values` has shape (..., n_cells, p+1) (numpy, or a CUDA float64 tensor, which
    is then also what is returned); destination cell i draws from source cells
    i - n_shift and i - n_shift - 1 (periodic wrap, absorbing zero fill).
    """
    import torch

    from . import _capi
    from ._device import current_stream, device, is_device_tensor
    check_bc(bc)
    on_dev = is_device_tensor(values)
    v = values if on_dev else np.asarray(values, dtype=float)
    if v.ndim < 2:
        raise ValueError("expected pencil values of shape (..., n_cells, p+1)")
    n, o = int(v.shape[-2]), int(v.shape[-1])
    A = np.ascontiguousarray(pair.same, dtype=np.float64)
    B = np.ascontiguousarray(pair.neighbor, dtype=np.float64)
    if A.shape != (o, o) or B.shape != (o, o):
        raise ValueError(f"overlap pair shaped {A.shape}, values have {o} nodes per cell")
    dev = device()
    vd = (v.to(torch.float64).contiguous() if on_dev
          else torch.from_numpy(np.ascontiguousarray(v)).to(dev))
    out = torch.empty_like(vd)
    Ad, Bd = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
    n_batch = vd.numel() // (n * o) if n * o else 0
    _capi.check(_capi.lib().sldg_apply_update(vd.data_ptr(), n_batch, n, o, int(decomp.n_shift),
                                              Ad.data_ptr(), Bd.data_ptr(), _capi.BC_CODE[bc],
                                              out.data_ptr(), current_stream()), ValueError)
    return out if on_dev else out.cpu().numpy()


def projection_oracle(values, displacement: float, width: float, basis, bc: str = PERIODIC):
    """Brute-force projection of the exactly translated pencil (sldg1d.py:139-178), on
    the device: 50-point Gauss quadrature over every overlap of the foot of cell
    i = [i w, (i+1) w) - displacement with a source cell (and its periodic images)."""
    import torch

    from . import _capi
    from ._device import current_stream, device
    check_bc(bc)
    v = np.ascontiguousarray(np.asarray(values, dtype=float))
    if v.ndim != 2 or v.shape[1] != basis.n_nodes:
        raise ValueError(f"expected values of shape (n_cells, {basis.n_nodes})")
    gq, gw = np.polynomial.legendre.leggauss(50)
    dev = device()
    vd = torch.from_numpy(v).to(dev)
    gqd, gwd = torch.from_numpy(gq).to(dev), torch.from_numpy(gw).to(dev)
    out = torch.empty_like(vd)
    ba = _capi.BasisArrays(basis)
    _capi.check(_capi.lib().sldg_projection_oracle(
        ba.struct, vd.data_ptr(), v.shape[0], float(displacement), float(width),
        _capi.BC_CODE[bc], gqd.data_ptr(), gwd.data_ptr(), gq.size, out.data_ptr(),
        current_stream()), ValueError)
    return out.cpu().numpy()
