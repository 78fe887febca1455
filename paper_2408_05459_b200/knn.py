"""Subsystem 1: exact KNN graph on the B200 (reference: ancka/knn.py).

`knn_search_exact` runs `ancka_knn_exact` (tcgen05 integer-exact path for
integer-valued attributes such as bag-of-words; tcgen05 split-bf16
candidates + exact f64 re-rank with an error certificate for real-valued
attributes, uncertified rows recomputed by the f64 CUDA-core scan) and `build_knn_adjacency` / `knn_transition` run
`ancka_knn_graph`.  Results stay in HBM; the numpy/scipy views the reference
API exposes (`NeighborLists.ids`, `KnnGraph.adjacency`, ...) are materialised
lazily on first access.  `knn_search_approx` is the reference's inverted-file
search (knn.py:143-280) on the device (csrc/knn_ivf.cu); `search_knn` and the
engine dispatch AUTO as the reference does (approximate at n >= 100k).
"""
from __future__ import annotations

import hashlib
import struct
import warnings

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from ._device import WORKSPACE, DeviceCSR, dev, to_device
from .network import APPROX_KNN_THRESHOLD, KnnMode, NetworkError

_PAD = -1
#: route attributes to the tcgen05 kernels (knn_tc.cu, knn_tc_real.cu); when
#: False every row takes the f64 CUDA-core scan (level -1)
TENSOR_CORE_KNN = True
#: list-length limits of the tensor-core kernels (integer / real-valued)
TC_MAX_K_INTEGER, TC_MAX_K_REAL = 32, 24


class NeighborLists:
    """Per-node top-K neighbour ids and cosine scores, padded with -1
    (knn.py:30-44).  Device-resident; `.ids`/`.scores` are host views."""

    def __init__(self, ids_dev=None, scores_dev=None, K=None, ids=None, scores=None):
        self._ids_dev, self._scores_dev = ids_dev, scores_dev
        self._ids, self._scores = ids, scores
        self.K = int(K if K is not None else (ids.shape[1] if ids is not None else ids_dev.shape[1]))

    @classmethod
    def from_host(cls, ids, scores):
        ids = np.asarray(ids, dtype=np.int64)
        return cls(ids=ids, scores=np.asarray(scores, dtype=np.float64), K=ids.shape[1])

    @property
    def ids(self) -> np.ndarray:
        if self._ids is None:
            self._ids = self._ids_dev.cpu().numpy().astype(np.int64)
        return self._ids

    @property
    def scores(self) -> np.ndarray:
        if self._scores is None:
            self._scores = self._scores_dev.cpu().numpy()
        return self._scores

    def device(self):
        if self._ids_dev is None:
            self._ids_dev = torch.from_numpy(self._ids.astype(np.int32)).to(dev())
            self._scores_dev = torch.from_numpy(np.ascontiguousarray(self._scores)).to(dev())
        return self._ids_dev, self._scores_dev

    @property
    def n(self) -> int:
        return self._ids_dev.shape[0] if self._ids_dev is not None else self._ids.shape[0]

    def row(self, i: int):
        ok = self.ids[i] != _PAD
        return self.ids[i][ok], self.scores[i][ok]


class KnnGraph:
    """Symmetric weighted KNN adjacency A_K plus the lists (knn.py:47-51)."""

    def __init__(self, a_k: DeviceCSR, p_k: DeviceCSR, zero_rows, neighbors, mode_used):
        self.a_k_dev, self.p_k_dev, self.zero_rows_dev = a_k, p_k, zero_rows
        self.neighbors = neighbors
        self.mode_used = mode_used
        self._adj = None

    @property
    def adjacency(self) -> sp.csr_matrix:
        if self._adj is None:
            self._adj = self.a_k_dev.to_scipy()
        return self._adj


def _normalize_host(x):
    """knn.py:54-65, used only by the small host helper `cosine_sim`."""
    x = np.asarray(x, dtype=np.float64)
    nrm = np.linalg.norm(x)
    return x / nrm if nrm > 0 else x


def cosine_sim(xi, xj) -> float:
    """Cosine of two rows; 0 if either is all-zero (knn.py:68-80)."""
    if sp.issparse(xi):
        xi = xi.toarray()
    if sp.issparse(xj):
        xj = xj.toarray()
    xi = np.asarray(xi, dtype=np.float64).ravel()
    xj = np.asarray(xj, dtype=np.float64).ravel()
    ni, nj = np.linalg.norm(xi), np.linalg.norm(xj)
    if ni == 0.0 or nj == 0.0:
        return 0.0
    return float(xi @ xj) / (ni * nj)


def integer_exact(X) -> int:
    """Tensor-core eligibility of X: 2 = integers with |x| <= 16 (exact in
    e4m3 fp8), 1 = integers with |x| <= 256 (exact in bf16), 0 = otherwise.
    Every row's sum of squares must stay < 2^24 so the f32 accumulation of
    the dot products is exact."""
    vals = X.data if sp.issparse(X) else np.asarray(X)
    if vals.size == 0 or not np.all(vals == np.rint(vals)):
        return 0
    vmax = float(np.abs(vals).max())
    if vmax > 256:
        return 0
    sq = np.asarray(X.multiply(X).sum(axis=1)).ravel() if sp.issparse(X) else (vals * vals).sum(axis=1)
    if sq.max() >= 2 ** 24:
        return 0
    return 2 if vmax <= 16 else 1


def _level_from_checks(nonint: float, vmax: float, sqmax: float) -> int:
    """integer_exact's rule applied to the device-side checks."""
    if nonint or vmax > 256 or sqmax >= 2 ** 24:
        return 0
    return 2 if vmax <= 16 else 1


class DeviceAttributes:
    """Attributes resident in HBM: CSR (sparse input on an integer-exact
    path, fed to the tensor-core kernel as is) or dense f64.  With
    `level=None` the integer-exact level is decided on the device after the
    upload (ancka_attr_check), so the host never scans X."""

    def __init__(self, X, level: int | None):
        self.shape = X.shape
        d = dev()
        self.dense = None
        if sp.issparse(X):
            x = sp.csr_matrix(X)
            self.indptr = torch.from_numpy(x.indptr.astype(np.int64)).to(d)
            self.indices = torch.from_numpy(x.indices.astype(np.int32)).to(d)
            self.data = torch.from_numpy(x.data.astype(np.float64)).to(d)
            if level is None:
                level = self._check(self.indptr.data_ptr(), self.data.data_ptr(), 0, 0)
            if level <= 0:
                t = torch.sparse_csr_tensor(self.indptr, self.indices.long(), self.data,
                                            size=x.shape)
                self.dense = t.to_dense().contiguous()
                self.indptr = self.indices = self.data = None
        else:
            self.dense = to_device(np.asarray(X, dtype=np.float64))
            if level is None:
                level = self._check(None, self.dense.data_ptr(), self.dense.stride(0),
                                    self.dense.shape[1])
        self.level = int(level)

    @classmethod
    def from_device_csr(cls, indptr, indices, data, shape) -> "DeviceAttributes":
        """CSR already in HBM (e.g. a shard received over the KNN ring)."""
        self = cls.__new__(cls)
        self.shape, self.dense = tuple(shape), None
        self.indptr, self.indices, self.data = indptr, indices, data
        level = self._check(indptr.data_ptr(), data.data_ptr(), 0, 0)
        if level <= 0:
            t = torch.sparse_csr_tensor(indptr, indices.long(), data, size=self.shape)
            self.dense = t.to_dense().contiguous()
            self.indptr = self.indices = self.data = None
        self.level = int(level)
        return self

    @classmethod
    def from_device_dense(cls, x) -> "DeviceAttributes":
        self = cls.__new__(cls)
        self.shape, self.dense = tuple(x.shape), x.contiguous()
        self.indptr = self.indices = self.data = None
        self.level = int(self._check(None, self.dense.data_ptr(), self.dense.stride(0),
                                     self.dense.shape[1]))
        return self

    def _check(self, rowptr, values, ld, ncols) -> int:
        out = torch.empty(3, dtype=torch.float64, device=dev())
        _lib.call("ancka_attr_check", rowptr, values, self.shape[0], ld, ncols, out.data_ptr(),
                  _lib.stream())
        nonint, vmax, sqmax = out.cpu().tolist()
        return _level_from_checks(nonint, vmax, sqmax)


def attributes_to_device(X, level: int | None = None) -> DeviceAttributes:
    return DeviceAttributes(X, level)


def knn_search_exact_device(X, K: int, integer: int | None = None, rows=None):
    """Device exact KNN: returns (ids int32 (nq,K), scores f64 (nq,K)) tensors
    for query rows `rows` = (q_begin, q_end) (default: all n) against all keys.
    X: numpy/scipy host matrix, DeviceAttributes, or a dense f64 CUDA tensor."""
    _lib.require_device()
    n, d = X.shape
    if K >= n:
        raise NetworkError(f"K={K} must be smaller than n={n}")
    if integer is None:
        integer = (X.level if isinstance(X, DeviceAttributes) else
                   0 if isinstance(X, torch.Tensor) else integer_exact(X))
    if (not TENSOR_CORE_KNN or (integer > 0 and K > TC_MAX_K_INTEGER)
            or (integer == 0 and K > TC_MAX_K_REAL)):
        integer = -1
    if isinstance(X, torch.Tensor):
        xa = None
        xd = X
    else:
        xa = X if isinstance(X, DeviceAttributes) else DeviceAttributes(X, integer)
        xd = xa.dense
        if xd is None and integer <= 0:  # CSR held for the integer path, real path requested
            xd = torch.sparse_csr_tensor(xa.indptr, xa.indices.long(), xa.data,
                                         size=xa.shape).to_dense()
    dv = dev()
    q0, q1 = rows if rows is not None else (0, n)
    ids = torch.empty((q1 - q0, K), dtype=torch.int32, device=dv)
    scores = torch.empty((q1 - q0, K), dtype=torch.float64, device=dv)
    wsb = _lib.load().ancka_knn_workspace_size(n, d, K, int(integer))
    ws = WORKSPACE.get("knn", wsb)
    if xd is None:
        _lib.call("ancka_knn_exact_csr", xa.indptr.data_ptr(), xa.indices.data_ptr(),
                  xa.data.data_ptr(), n, d, K, int(integer), q0, q1, ids.data_ptr(),
                  scores.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    else:
        _lib.call("ancka_knn_exact", xd.data_ptr(), n, d, xd.stride(0), K, int(integer), q0, q1,
                  ids.data_ptr(), scores.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    LAST_STATS.pop("fallback_rows", None)
    if integer == 0:   # the count stays on the device until someone reads it
        cnt = torch.zeros(1, dtype=torch.int32, device=dv)
        _lib.call("ancka_knn_fallback_rows_async", ws.data_ptr(), ws.numel(), n, d, K, q0, q1,
                  cnt.data_ptr(), _lib.stream())
        LAST_STATS["fallback_rows"] = lambda: int(cnt.item())
    LAST_STATS["level"] = int(integer)
    return ids, scores


class _LazyStats(dict):
    """Values may be zero-argument callables, evaluated (and cached) on first
    read: a device count read back only when asked for, so the search itself
    never waits for the GPU."""

    def __getitem__(self, key):
        v = super().__getitem__(key)
        if callable(v):
            v = v()
            super().__setitem__(key, v)
        return v

    def get(self, key, default=None):
        return self[key] if key in self else default


#: diagnostics of the last device search: path level and, for real-valued
#: attributes, how many rows the tensor-core certificate sent to the f64 scan
LAST_STATS: dict = _LazyStats()


def knn_search_exact(X, K: int, block_rows: int | None = None) -> NeighborLists:
    """Exact top-K cosine neighbours (knn.py:112-140).  `block_rows` is
    accepted for signature compatibility; tiling is fixed by the kernel."""
    ids, scores = knn_search_exact_device(X, K)
    return NeighborLists(ids_dev=ids, scores_dev=scores, K=K)


# --------------------------------------------------------------------------
# Approximate search: inverted-file index (knn.py:143-280; csrc/knn_ivf.cu)
# --------------------------------------------------------------------------

#: per-chunk device bytes for the probe scores and partial lists (at most;
#: also at most a quarter of the free device memory)
IVF_CHUNK_BYTES = 32 << 30
#: extra slots per (query, list) partial list and in the merged list; the
#: f64 re-rank certifies the top-K against the K2-th f32 score
IVF_MARGIN = 8
#: score the scan on the tensor cores (fp16 single product, certified; 32
#: list slots) when d <= 256; False: the f32 SIMT scan
IVF_TENSOR_CORES = True


def ivf_defaults(n: int, nlist: int | None, nprobe: int | None):
    """knn.py:181-187."""
    if nlist is None:
        nlist = int(min(4096, max(8, round(np.sqrt(n)))))
    nlist = min(nlist, n)
    if nprobe is None:
        nprobe = max(4, nlist // 32)
    return nlist, min(nprobe, nlist)


def _ivf_xn(X):
    """Row-normalised f32 attributes on the device (knn.py:172-174): n x dp."""
    n, d = X.shape
    dp = max(4, (d + 3) // 4 * 4)
    xn = torch.empty((n, dp), dtype=torch.float32, device=dev())
    if isinstance(X, torch.Tensor):
        _lib.call("ancka_ivf_normalize", X.data_ptr(), X.stride(0), None, None, None, n, d,
                  xn.data_ptr(), dp, _lib.stream())
        return xn
    xa = X if isinstance(X, DeviceAttributes) else DeviceAttributes(X, 0)
    if xa.dense is not None:
        _lib.call("ancka_ivf_normalize", xa.dense.data_ptr(), xa.dense.stride(0), None, None, None,
                  n, d, xn.data_ptr(), dp, _lib.stream())
    else:
        _lib.call("ancka_ivf_normalize", None, 0, xa.indptr.data_ptr(), xa.indices.data_ptr(),
                  xa.data.data_ptr(), n, d, xn.data_ptr(), dp, _lib.stream())
    return xn


def _bucket(keys, count: int, nbuckets: int, tile: int = 0):
    dv = keys.device
    ptr = torch.empty(nbuckets + 1, dtype=torch.int64, device=dv)
    tiles = torch.empty(nbuckets + 1, dtype=torch.int64, device=dv) if tile else None
    ent = torch.empty(max(count, 1), dtype=torch.int32, device=dv)
    wsb = _lib.load().ancka_ivf_bucket_workspace_size(nbuckets)
    ws = WORKSPACE.get("ivf_bucket", wsb)
    _lib.call("ancka_ivf_bucket", keys.data_ptr(), count, nbuckets, ptr.data_ptr(),
              tiles.data_ptr() if tile else None, tile, ent.data_ptr(), ws.data_ptr(), ws.numel(),
              _lib.stream())
    return ptr, tiles, ent


def _argmax_rows(xn, rows, m, C, bias, labels, changed=None):
    keys = torch.zeros(m, dtype=torch.int64, device=xn.device)
    _lib.call("ancka_ivf_gemm", xn.data_ptr(), xn.stride(0),
              rows.data_ptr() if rows is not None else None, m, C.data_ptr(), C.stride(0),
              C.shape[0], xn.shape[1], bias.data_ptr() if bias is not None else None, None, 0,
              keys.data_ptr(), _lib.stream())
    _lib.call("ancka_ivf_argmax_finish", keys.data_ptr(), m, labels.data_ptr(),
              changed.data_ptr() if changed is not None else None, _lib.stream())


def train_ivf_device(xn, nlist: int, seed: int, max_iter: int = 25):
    """Centroids for the index (knn.py:143-153) by Lloyd iterations on the
    device, on the reference's training sample (the same `rng.choice` rows).
    The reference runs sklearn's KMeans (k-means++ seeding); here the first
    centres are `nlist` sample rows drawn from a second seeded generator, and
    the iterations stop when no assignment changes or after `max_iter`
    (sklearn's strict-convergence rule and cap).  Parity with the reference
    is pinned by passing its centroids (`knn_search_approx(centroids=...)`)."""
    n, dp = xn.shape
    dv = xn.device
    max_train = 50 * nlist
    if n > max_train:
        rng = np.random.default_rng(seed)
        rows_h = rng.choice(n, size=max_train, replace=False)
    else:
        rows_h = np.arange(n)
    ms = rows_h.size
    rows = torch.from_numpy(rows_h.astype(np.int32)).to(dv)
    init = np.random.default_rng([seed, 1]).choice(ms, size=nlist, replace=False)
    C = xn[torch.from_numpy(rows_h[init].astype(np.int64)).to(dv)].contiguous()
    bias = torch.empty(nlist, dtype=torch.float32, device=dv)
    sums = torch.zeros((nlist, dp), dtype=torch.int64, device=dv)
    counts = torch.zeros(nlist, dtype=torch.int32, device=dv)
    _lib.call("ancka_ivf_kmeans_update", None, 0, None, 0, None, nlist, dp, None, None,
              C.data_ptr(), C.stride(0), bias.data_ptr(), _lib.stream())
    labels = torch.full((ms,), -1, dtype=torch.int32, device=dv)
    changed = torch.zeros(1, dtype=torch.int32, device=dv)
    iters = 0
    for it in range(max_iter):
        changed.zero_()
        _argmax_rows(xn, rows, ms, C, bias, labels, changed)
        iters = it + 1
        if it > 0 and int(changed.item()) == 0:
            break
        _lib.call("ancka_ivf_kmeans_update", xn.data_ptr(), xn.stride(0), rows.data_ptr(), ms,
                  labels.data_ptr(), nlist, dp, sums.data_ptr(), counts.data_ptr(), C.data_ptr(),
                  C.stride(0), bias.data_ptr(), _lib.stream())
    return C, iters


class IvfIndex:
    """Device inverted-file index: f32 normalised rows, centroids, and the
    lists as (list_ptr, perm) -- rows of list c are perm[list_ptr[c]:
    list_ptr[c+1]] (knn.py:198-203).  `half()` adds the fp16 copy and the
    per-row residual norms the tensor-core scan certifies with."""

    def __init__(self, xn, C, labels, list_ptr, perm, train_iters):
        self.xn, self.C, self.labels = xn, C, labels
        self.list_ptr, self.perm = list_ptr, perm
        self.nlist = C.shape[0]
        self.train_iters = train_iters
        self._half = None

    def half(self):
        if self._half is None:
            n, dp = self.xn.shape
            dh = (dp + 15) // 16 * 16
            h = torch.empty((n, dh), dtype=torch.float16, device=self.xn.device)
            lres = torch.empty(n, dtype=torch.float32, device=self.xn.device)
            lmax = torch.zeros(1, dtype=torch.int32, device=self.xn.device)
            _lib.call("ancka_ivf_half_prep", self.xn.data_ptr(), n, dp, h.data_ptr(), dh,
                      lres.data_ptr(), lmax.data_ptr(), _lib.stream())
            self._half = (h, dh, lres, lmax)
        return self._half


def build_ivf_index(X, nlist: int, seed: int = 0, centroids=None) -> IvfIndex:
    xn = X if (isinstance(X, torch.Tensor) and X.dtype == torch.float32) else _ivf_xn(X)
    n, dp = xn.shape
    iters = 0
    if centroids is None:
        C, iters = train_ivf_device(xn, nlist, seed)
    else:
        c = np.asarray(centroids, dtype=np.float32)
        C = torch.zeros((c.shape[0], dp), dtype=torch.float32, device=xn.device)
        C[:, :c.shape[1]] = torch.from_numpy(c).to(xn.device)
    labels = torch.empty(n, dtype=torch.int32, device=xn.device)
    _argmax_rows(xn, None, n, C, None, labels)                 # knn.py:197 (inner product)
    list_ptr, _, perm = _bucket(labels, n, C.shape[0])
    return IvfIndex(xn, C, labels, list_ptr, perm, iters)


def _ivf_err(dp: int) -> float:
    """Bound on |f32 dot - exact dot| for unit rows: (dp + 2) u (Cauchy-Schwarz)."""
    return float((dp + 2) * 2.0 ** -24 * 1.001)


def ivf_search_all_device(index: IvfIndex, K: int, nprobe: int, stats: dict | None = None):
    """_ivf_search_all (knn.py:236-262) for every row: (ids int32, scores f64)."""
    xn, nlist = index.xn, index.nlist
    n, dp = xn.shape
    dv = xn.device
    tc = IVF_TENSOR_CORES and (dp + 15) // 16 * 16 <= 256 and K + IVF_MARGIN <= 32
    K2 = 32 if tc else min(K + IVF_MARGIN, 256)
    err = _ivf_err(dp)
    if tc:
        h, dh, lres, lmax = index.half()
        err = float((dh + 2) * 2.0 ** -22)
    ids = torch.empty((n, K), dtype=torch.int32, device=dv)
    scores = torch.empty((n, K), dtype=torch.float64, device=dv)
    per_row = nlist * 4 + nprobe * 4 + nprobe * K2 * 8
    budget = min(IVF_CHUNK_BYTES, torch.cuda.mem_get_info(dv)[0] // 4)
    chunk = int(max(1, min(n, budget // per_row)))
    flagged = torch.empty(chunk, dtype=torch.int32, device=dv)
    nflag = torch.zeros(1, dtype=torch.int32, device=dv)
    counter = torch.zeros(1, dtype=torch.int32, device=dv)
    S = torch.empty((chunk, nlist), dtype=torch.float32, device=dv)
    probes = torch.empty((chunk, nprobe), dtype=torch.int32, device=dv)
    part_s = torch.empty(chunk * nprobe * K2, dtype=torch.float32, device=dv)
    part_i = torch.empty(chunk * nprobe * K2, dtype=torch.int32, device=dv)
    qthr = torch.empty(chunk, dtype=torch.int32, device=dv)
    own = torch.empty((chunk, nprobe), dtype=torch.int32, device=dv) if tc else None
    rest = torch.empty((chunk, nprobe), dtype=torch.int32, device=dv) if tc else None
    st = _lib.stream()
    total_flag = 0
    for q0 in range(0, n, chunk):
        m = min(chunk, n - q0)
        _lib.call("ancka_ivf_gemm", xn[q0:].data_ptr(), dp, None, m, index.C.data_ptr(), dp, nlist,
                  dp, None, S.data_ptr(), nlist, None, st)
        _lib.call("ancka_ivf_topsel", S.data_ptr(), nlist, m, nlist, nprobe, probes.data_ptr(), st)
        qthr.zero_()
        if tc:
            # two phases: every query's own list first (a whole-list threshold
            # for each query), then its other probes with that threshold
            _lib.call("ancka_ivf_split_probes", probes.data_ptr(), index.labels.data_ptr(), q0, m,
                      nprobe, own.data_ptr(), rest.data_ptr(), st)
            for keys in (own, rest):
                pair_ptr, tile_ptr, pair_ent = _bucket(keys, m * nprobe, nlist, tile=64)
                _lib.call("ancka_ivf_search_tc", h.data_ptr(), dh, lres.data_ptr(),
                          lmax.data_ptr(), index.perm.data_ptr(), index.list_ptr.data_ptr(),
                          pair_ptr.data_ptr(), pair_ent.data_ptr(), tile_ptr.data_ptr(),
                          counter.data_ptr(), nlist, nprobe, q0, K2, err, part_s.data_ptr(),
                          part_i.data_ptr(), qthr.data_ptr(), st)
        else:
            pair_ptr, tile_ptr, pair_ent = _bucket(probes, m * nprobe, nlist, tile=64)
            _lib.call("ancka_ivf_search", xn.data_ptr(), dp, index.perm.data_ptr(),
                      index.list_ptr.data_ptr(), pair_ptr.data_ptr(), pair_ent.data_ptr(),
                      tile_ptr.data_ptr(), counter.data_ptr(), nlist, nprobe, q0, K2, err,
                      part_s.data_ptr(), part_i.data_ptr(), qthr.data_ptr(), st)
        nflag.zero_()
        _lib.call("ancka_ivf_merge", xn.data_ptr(), dp, q0, m, nprobe, K2, K, part_s.data_ptr(),
                  part_i.data_ptr(), err, ids[q0:].data_ptr(), scores[q0:].data_ptr(),
                  flagged.data_ptr(), nflag.data_ptr(), lres.data_ptr() if tc else None,
                  lmax.data_ptr() if tc else None, st)
        nf = int(nflag.item())
        if nf:
            _lib.call("ancka_ivf_rows_exact", xn.data_ptr(), dp, n, flagged.data_ptr(), nf,
                      probes.data_ptr(), nprobe, q0, index.perm.data_ptr(),
                      index.list_ptr.data_ptr(), K, ids[q0:].data_ptr(), scores[q0:].data_ptr(),
                      0, st)
        total_flag += nf
    if stats is not None:
        stats["uncertified_rows"] = stats.get("uncertified_rows", 0) + total_flag
        stats["chunks"] = (n + chunk - 1) // chunk
        stats["scan"] = "tensor-core fp16" if tc else "f32 SIMT"
    return ids, scores


def ivf_exact_rows_device(xn, rows: np.ndarray, K: int):
    """Exact top-K of the listed rows against all keys (the audit truth,
    _exact_rows_for, knn.py:225-233): (ids int32, scores f64), row b = rows[b]."""
    n, dp = xn.shape
    m = rows.size
    r = torch.from_numpy(rows.astype(np.int32)).to(xn.device)
    ids = torch.empty((max(m, 1), K), dtype=torch.int32, device=xn.device)
    scores = torch.empty((max(m, 1), K), dtype=torch.float64, device=xn.device)
    _lib.call("ancka_ivf_rows_exact", xn.data_ptr(), dp, n, r.data_ptr(), m, None, 0, 0, None, None,
              K, ids.data_ptr(), scores.data_ptr(), 1, _lib.stream())
    return ids[:m], scores[:m]


def _audit_recall(ids_h: np.ndarray, truth_h: np.ndarray) -> float:
    """knn.py:265-274 on the audit rows (host, m x K)."""
    hits = []
    for got, truth in zip(ids_h, truth_h):
        t = truth[truth >= 0]
        if t.size == 0:
            continue
        hits.append(np.isin(t, got[got >= 0]).mean())
    return float(np.mean(hits)) if hits else 1.0


def knn_search_approx(X, K: int, recall_target: float = 0.9, seed: int = 0,
                      nlist: int | None = None, nprobe: int | None = None,
                      audit_size: int = 1000, centroids=None) -> NeighborLists:
    """Approximate top-K cosine neighbours through an inverted-file index
    (knn.py:156-213): same defaults, the same audit sample and the same
    probe escalation (x2 until the audited recall reaches `recall_target`
    or every list is probed, warning as the reference does).  `centroids`
    (nlist x d) replaces the device training, e.g. with the reference's
    sklearn centroids for parity.  Diagnostics in LAST_STATS["approx"]."""
    _lib.require_device()
    n = X.shape[0]
    if K >= n:
        raise NetworkError(f"K={K} must be smaller than n={n}")
    if centroids is not None:
        nlist = np.asarray(centroids).shape[0]
    nlist, nprobe = ivf_defaults(n, nlist, nprobe)
    index = build_ivf_index(X, nlist, seed, centroids)
    rng = np.random.default_rng(seed)                               # knn.py:205-208
    m = min(n, max(audit_size, 1000))
    audit_idx = np.sort(rng.choice(n, size=m, replace=False))
    truth, _ = ivf_exact_rows_device(index.xn, audit_idx, K)
    truth_h = truth.cpu().numpy()
    audit_dev = torch.from_numpy(audit_idx.astype(np.int64)).to(index.xn.device)
    stats = {"nlist": nlist, "train_iters": index.train_iters, "escalations": 0}
    while True:
        if nprobe >= nlist:     # probing every list is the exact search (knn.py:244-245)
            ids, scores = knn_search_exact_device(X, K)
        else:
            ids, scores = ivf_search_all_device(index, K, nprobe, stats)
        recall = _audit_recall(ids[audit_dev].cpu().numpy(), truth_h)
        if recall >= recall_target or nprobe >= nlist:
            if recall < recall_target:
                warnings.warn(f"approximate KNN recall {recall:.3f} below target "
                              f"{recall_target:.3f} even at exhaustive probing")
            break
        old = nprobe
        nprobe = min(nlist, nprobe * 2)
        stats["escalations"] += 1
        warnings.warn(f"approximate KNN recall {recall:.3f} < {recall_target:.3f}; "
                      f"escalating probes {old} -> {nprobe}")
    stats.update(nprobe=nprobe, recall=recall)
    LAST_STATS["approx"] = stats
    return NeighborLists(ids_dev=ids, scores_dev=scores, K=K)


def resolve_knn_mode(mode: KnnMode, n: int) -> KnnMode:
    """AUTO: exact below APPROX_KNN_THRESHOLD nodes, approximate at or above
    (knn.py:286-287, network.py:36)."""
    if mode is KnnMode.AUTO:
        return KnnMode.EXACT if n < APPROX_KNN_THRESHOLD else KnnMode.APPROX
    return mode


def search_knn(X, K: int, mode: KnnMode = KnnMode.AUTO, seed: int = 0,
               recall_target: float = 0.9):
    """Mode dispatch (knn.py:283-291)."""
    mode = resolve_knn_mode(mode, X.shape[0])
    if mode is KnnMode.EXACT:
        return knn_search_exact(X, K), KnnMode.EXACT
    return knn_search_approx(X, K, recall_target=recall_target, seed=seed), KnnMode.APPROX


def build_knn_graph_device(ids, scores, n: int):
    """A_K and P_K on the device from (ids, scores) device tensors."""
    K = ids.shape[1]
    d = ids.device
    cap = 2 * n * K
    rowptr = torch.empty(n + 1, dtype=torch.int64, device=d)
    colidx = torch.empty(cap, dtype=torch.int32, device=d)
    a_k = torch.empty(cap, dtype=torch.float64, device=d)
    p64 = torch.empty(cap, dtype=torch.float64, device=d)
    p32 = torch.empty(cap, dtype=torch.float32, device=d)
    zero = torch.empty(n, dtype=torch.uint8, device=d)
    nnz = torch.zeros(1, dtype=torch.int64, device=d)
    wsb = _lib.load().ancka_knn_graph_workspace_size(n, K)
    ws = WORKSPACE.get("knn_graph", wsb)
    _lib.call("ancka_knn_graph", ids.data_ptr(), scores.data_ptr(), n, K, rowptr.data_ptr(),
              colidx.data_ptr(), a_k.data_ptr(), p64.data_ptr(), p32.data_ptr(), zero.data_ptr(),
              nnz.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    m = int(nnz.item())
    A = DeviceCSR(n, n, rowptr, colidx[:m], a_k[:m], None)
    P = DeviceCSR(n, n, rowptr, colidx[:m], p64[:m], p32[:m])
    return A, P, zero


def build_knn_adjacency(neighbors: NeighborLists, X=None, mode_used: KnnMode = KnnMode.EXACT) -> KnnGraph:
    """A_K = M + M^T (knn.py:294-309), built on the device."""
    _lib.require_device()
    ids, scores = neighbors.device()
    A, P, zero = build_knn_graph_device(ids, scores, neighbors.n)
    return KnnGraph(A, P, zero, neighbors, mode_used)


def knn_transition(g: KnnGraph):
    """P_K = D_K^-1 A_K and the zero-row flags (knn.py:312-324), host views."""
    return g.p_k_dev.to_scipy(), g.zero_rows_dev.cpu().numpy().astype(bool)


# ---------------------------------------------------------------- cache ---
# knn.py:327-382: b"AKNC", version u8, mode u8, reserved u16, n u64, K u32,
# then n*K (id u32, score f32), absent = 0xFFFFFFFF.
_MAGIC, _VERSION, _SENTINEL = b"AKNC", 1, 0xFFFFFFFF
_HEADER = struct.Struct("<4sBBHQI")


def cache_key(X, K: int, mode: KnnMode) -> str:
    h = hashlib.sha256()
    if sp.issparse(X):
        x = X.tocsr()
        h.update(np.asarray(x.indptr, dtype=np.int64).tobytes())
        h.update(np.asarray(x.indices, dtype=np.int64).tobytes())
        h.update(np.asarray(x.data, dtype=np.float64).tobytes())
    else:
        h.update(np.ascontiguousarray(X, dtype=np.float64).tobytes())
    h.update(struct.pack("<Iq", K, X.shape[1]))
    h.update(mode.value.encode())
    return h.hexdigest()[:32]


def save_neighbor_cache(path, neighbors: NeighborLists, mode: KnnMode) -> None:
    ids = neighbors.ids.copy()
    n, k = ids.shape
    ids[ids == _PAD] = _SENTINEL
    rec = np.empty((n, k), dtype=[("id", "<u4"), ("score", "<f4")])
    rec["id"] = ids.astype(np.uint64).astype("<u4")
    rec["score"] = neighbors.scores.astype("<f4")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(_MAGIC, _VERSION, 0 if mode is KnnMode.EXACT else 1, 0, n, k))
        fh.write(rec.tobytes())


def load_neighbor_cache(path):
    with open(path, "rb") as fh:
        magic, version, mode_code, _, n, k = _HEADER.unpack(fh.read(_HEADER.size))
        if magic != _MAGIC or version != _VERSION:
            raise NetworkError(f"{path}: not a neighbor cache file")
        rec = np.frombuffer(fh.read(), dtype=[("id", "<u4"), ("score", "<f4")])
    if rec.size != n * k:
        raise NetworkError(f"{path}: truncated neighbor cache")
    rec = rec.reshape(n, k)
    ids = rec["id"].astype(np.int64)
    ids[ids == _SENTINEL] = _PAD
    scores = rec["score"].astype(np.float64)
    scores[ids == _PAD] = 0.0
    return NeighborLists.from_host(ids, scores), (KnnMode.EXACT if mode_code == 0 else KnnMode.APPROX)
