"""Device-buffer plumbing: torch CUDA tensors are only buffer carriers.

No torch compute kernel is ever used on the transport path: tensors provide
device memory (and pinned host staging), `current_stream()` provides the
cudaStream_t every libsldg entry point enqueues on.
"""
from __future__ import annotations

import numpy as np
import torch


def device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_19959_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def current_stream():
    return torch.cuda.current_stream().cuda_stream


def is_device_tensor(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


def to_device_f64(a, contiguous=True):
    """numpy / torch -> contiguous float64 CUDA tensor (no copy when already one)."""
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            a = a.to(device())
        if a.dtype != torch.float64:
            a = a.to(torch.float64)
        return a.contiguous() if contiguous else a
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return torch.from_numpy(arr).to(device(), non_blocking=False)


class Scratch:
    """Grow-only device byte buffer cache keyed by name.

    Once a CUDA graph has captured launches that use these buffers (`pin()`, called by
    Simulation.advance_graph), a buffer that has to grow is retired instead of freed, so
    a replayed graph never writes into memory the allocator handed to another tensor.
    Entries keyed by an object's id are dropped when the object is collected
    (`release_with`)."""

    def __init__(self):
        self._bufs = {}
        self._retired = []
        self._pinned = False

    def pin(self):
        self._pinned = True

    def _replace(self, name, buf):
        old = self._bufs.get(name)
        if old is not None and self._pinned:
            self._retired.append(old)
        self._bufs[name] = buf

    def get(self, name, nbytes):
        nbytes = max(int(nbytes), 256)
        buf = self._bufs.get(name)
        if buf is None or buf.numel() < nbytes or buf.device != device():
            buf = torch.empty(nbytes, dtype=torch.uint8, device=device())
            self._replace(name, buf)
        return buf

    def like(self, name, t: torch.Tensor):
        """float64 tensor with t's shape (cached, contents undefined)."""
        buf = self._bufs.get(name)
        if buf is None or buf.shape != t.shape or buf.device != t.device:
            buf = torch.empty_like(t)
            self._replace(name, buf)
        return buf

    def drop(self, key):
        """Forget the entries of `key` (a name, or the id-tagged names (tag, key))."""
        for name in [n for n in self._bufs if n == key or (isinstance(n, tuple) and n[1:] == (key,))]:
            if not self._pinned:
                del self._bufs[name]

    def release_with(self, obj):
        """Drop the entries keyed by id(obj) when obj is garbage collected."""
        import weakref
        weakref.finalize(obj, self.drop, id(obj))


SCRATCH = Scratch()
