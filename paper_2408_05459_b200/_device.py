"""Device-memory plumbing: CSR factors resident in HBM and reusable workspaces.

PyTorch only allocates and owns the buffers here; every computation on them
goes through libancka_b200.so.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib


def dev():
    return torch.device("cuda", torch.cuda.current_device())


_PIN = {}          # device -> (two pinned staging buffers, their reuse events)
_PIN_CHUNK = 64 << 20
_POOL = None


def to_device(a: np.ndarray) -> torch.Tensor:
    """Host array -> new device tensor on the current stream, through two
    pinned 64 MiB staging buffers: host threads fill one chunk while the
    other one's copy runs (a pageable copy stages serially through one
    driver buffer).  Small arrays take the plain copy."""
    global _POOL
    a = np.ascontiguousarray(a)
    d = dev()
    if a.nbytes < 4 * _PIN_CHUNK:
        return torch.from_numpy(a).to(d)
    from concurrent.futures import ThreadPoolExecutor
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=4)
    if d not in _PIN:
        bufs = [torch.empty(_PIN_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        _PIN[d] = (bufs, [torch.cuda.Event(), torch.cuda.Event()])
    bufs, evs = _PIN[d]
    out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=d)
    src = a.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(torch.uint8)
    stream = torch.cuda.current_stream()
    quarter = _PIN_CHUNK // 4
    for k, o in enumerate(range(0, src.size, _PIN_CHUNK)):
        b = k & 1
        evs[b].synchronize()                       # the buffer's previous copy is done
        m = min(_PIN_CHUNK, src.size - o)
        hb = bufs[b].numpy()
        list(_POOL.map(lambda q: np.copyto(hb[q:min(q + quarter, m)], src[o + q:o + min(q + quarter, m)]),
                       range(0, m, quarter)))
        dst[o:o + m].copy_(bufs[b][:m], non_blocking=True)
        evs[b].record(stream)
    return out


class DeviceCSR:
    """Row-sorted CSR on the device with f64 and f32 value copies."""

    def __init__(self, rows, cols, rowptr, colidx, val64=None, val32=None):
        self.rows, self.cols = int(rows), int(cols)
        self.rowptr, self.colidx = rowptr, colidx
        self.val64, self.val32 = val64, val32

    @property
    def nnz(self) -> int:
        return int(self.colidx.numel())

    @classmethod
    def from_scipy(cls, m: sp.csr_matrix) -> "DeviceCSR":
        m = sp.csr_matrix(m)
        if not m.has_sorted_indices:
            m = m.copy()
            m.sort_indices()
        d = dev()
        rp = torch.from_numpy(np.ascontiguousarray(m.indptr, dtype=np.int64)).to(d)
        ci = torch.from_numpy(np.ascontiguousarray(m.indices, dtype=np.int32)).to(d)
        v64 = torch.from_numpy(np.ascontiguousarray(m.data, dtype=np.float64)).to(d)
        return cls(m.shape[0], m.shape[1], rp, ci, v64, v64.to(torch.float32))

    def struct(self, dtype: int) -> _lib.CSR:
        vals = self.val64 if dtype == _lib.F64 else self.val32
        return _lib.CSR(self.rows, self.cols, self.nnz, self.rowptr.data_ptr(),
                        self.colidx.data_ptr(), None if vals is None else vals.data_ptr())

    def to_scipy(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.val64.cpu().numpy(), self.colidx.cpu().numpy().astype(np.int32),
                              self.rowptr.cpu().numpy()), shape=(self.rows, self.cols))


_EMPTY = _lib.CSR(0, 0, 0, None, None, None)


def csr_struct(m: DeviceCSR | None, dtype: int) -> _lib.CSR:
    return _EMPTY if m is None else m.struct(dtype)


class Workspace:
    """Grow-only byte buffers keyed by purpose (stable addresses for graph capture)."""

    def __init__(self):
        self._bufs: dict[str, torch.Tensor] = {}

    def release(self, *keys: str) -> None:
        """Drop phase-specific buffers (the caching allocator keeps the
        memory for the next phase's tensors)."""
        for k in keys:
            self._bufs.pop(k, None)

    def get(self, key: str, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        b = self._bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.empty(nbytes, dtype=torch.uint8, device=dev())
            self._bufs[key] = b
        return b


WORKSPACE = Workspace()


def ld_for(c: int, dtype: torch.dtype) -> int:
    w = 4 if dtype == torch.float32 else 2
    return (c + w - 1) // w * w


def padded(m, dtype: torch.dtype) -> torch.Tensor:
    """Host or device n x c block -> device, row-major with padded leading dim."""
    t = torch.as_tensor(m)
    if t.ndim == 1:
        t = t[:, None]
    n, c = t.shape
    out = torch.zeros((n, ld_for(c, dtype)), dtype=dtype, device=dev())
    out[:, :c] = t.to(device=out.device, dtype=dtype)
    return out
