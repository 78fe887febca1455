"""ANCKA clustering engine on the B200 (reference: ancka/engine.py).

`run_ancka` keeps the whole loop device-resident:

* greedy init          -> ancka_init_bcm (f64, engine.py:87-127)
* t = 1 (rank-deficient by construction) -> f64 apply +
  f64 CGS2 QR with the reference's rank test and its exact numpy noise
  draw (engine.py:139-149), so Q^(1) matches the reference to rounding
* t >= 2               -> c <= 8: ancka_orth_block_f32 (one cooperative
  kernel per tau-block); wider blocks: ancka_orth_step_f32 per step.  CUDA
  graphs per tau-block are available (use_graphs=True) but off by default:
  a capture costs 17 ms (DBLP) to 110 ms (Amazon2M) of host time per run
  and saves ~0.1 ms per replayed block, which a single run never recovers
* every tau            -> ancka_discretize (one cooperative kernel) and
  ancka_mhc; one small device->host read of (phi, ||dQ||, flags) drives the
  reference's stop rules on the host (engine.py:402-418).

A suspect Cholesky pivot anywhere in a tau-block rolls the block back and
replays it with the exact f64 step.
"""
from __future__ import annotations

import time
import os
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import WORKSPACE, dev, ld_for, padded
from .knn import (KnnGraph, NeighborLists, attributes_to_device, build_knn_graph_device,
                  cache_key, integer_exact, knn_search_approx, knn_search_exact_device,
                  load_neighbor_cache, resolve_knn_mode, save_neighbor_cache)
from .network import (AttributedNetwork, BcmMatrix, ClusterParams, KnnMode, NetworkError,
                      default_knn_k, validate_network, NetworkKind)
from .walk import StructureFactors, WalkOperator, build_walk_operator

DISCRETIZE_MAX_ITER = 100
DISCRETIZE_TOL = 1e-10
#: reuse the previous tau sample's MHC when the new labels are the same
#: partition relabelled (ancka_same_partition); ANCKA_MHC_REUSE=0 disables
MHC_REUSE = os.environ.get("ANCKA_MHC_REUSE", "1") != "0"
_TIMING_KEYS = ("knn_ms", "init_ms", "ortho_ms", "discretize_ms", "mhc_ms")


class EngineState:
    """Loop state (engine.py:41-49); `q` is materialised from HBM on access."""

    def __init__(self, q_dev, best_y, best_mhc, mhc_history=None, iteration=0, c=None):
        self.q_dev = q_dev
        self._c = c
        self.best_y = best_y
        self.best_mhc = best_mhc
        self.mhc_history = mhc_history if mhc_history is not None else []
        self.iteration = iteration

    @property
    def q(self) -> np.ndarray:
        t = self.q_dev if self._c is None else self.q_dev[:, : self._c]
        return t.double().cpu().numpy()


@dataclass
class ClusterResult:
    y: BcmMatrix
    mhc: float
    iterations: int
    timings_ms: dict
    state: EngineState
    knn: KnnGraph
    operator: WalkOperator
    converged: bool
    stop_reason: str
    warnings: list = field(default_factory=list)
    error: str | None = None


@dataclass
class DiscretizeResult:
    y: BcmMatrix
    scores: np.ndarray
    objectives: list
    iterations: int
    converged: bool
    runs: tuple = ()


class _PhaseTimer:
    """CUDA-event phase timing (engine.py:67-72 semantics, device clock)."""

    def __init__(self):
        self.totals = {k: 0.0 for k in _TIMING_KEYS}
        self._open = []

    def span(self, key):
        timer = self

        class _Span:
            def __enter__(self_):
                self_.a = torch.cuda.Event(enable_timing=True)
                self_.a.record()

            def __exit__(self_, *exc):
                b = torch.cuda.Event(enable_timing=True)
                b.record()
                timer._open.append((key, self_.a, b))

        return _Span()

    def add_host(self, key, t0):
        self.totals[key] += (time.perf_counter() - t0) * 1e3

    def flush(self):
        for key, a, b in self._open:
            b.synchronize()
            self.totals[key] += a.elapsed_time(b)
        self._open.clear()


class _LazyTimings(dict):
    """ClusterResult.timings_ms: a plain dict once read.  The CUDA-event spans
    are resolved on first access instead of at the end of the run, so the
    ~2 event reads per span stay out of the clustering's own wall time."""

    def __init__(self, timer: "_PhaseTimer"):
        super().__init__()
        self._timer = timer

    def _resolve(self):
        if self._timer is not None:
            t, self._timer = self._timer, None
            t.flush()
            for k2, v in t.totals.items():
                super().__setitem__(k2, super().get(k2, 0.0) + v)

    def __getitem__(self, key):
        self._resolve()
        return super().__getitem__(key)

    def __setitem__(self, key, value):
        self._resolve()
        super().__setitem__(key, value)

    def __iter__(self):
        self._resolve()
        return super().__iter__()

    def __len__(self):
        self._resolve()
        return super().__len__()

    def __contains__(self, key):
        self._resolve()
        return super().__contains__(key)

    def __repr__(self):
        self._resolve()
        return super().__repr__()

    def get(self, key, default=None):
        self._resolve()
        return super().get(key, default)

    def items(self):
        self._resolve()
        return super().items()

    def keys(self):
        self._resolve()
        return super().keys()

    def values(self):
        self._resolve()
        return super().values()

    def copy(self):
        self._resolve()
        return dict(self)


# ----------------------------------------------------------------------------
def normalize_bcm(y: BcmMatrix) -> np.ndarray:
    """Column-orthonormal membership (engine.py:75-84)."""
    sizes = y.cluster_sizes()
    if (sizes == 0).any():
        raise NetworkError(f"empty cluster(s) {y.empty_clusters().tolist()}: normalization undefined")
    out = np.zeros((y.n, y.k))
    out[np.arange(y.n), y.assignment] = 1.0 / np.sqrt(sizes[y.assignment])
    return out


def _centers(deg: np.ndarray, k: int) -> np.ndarray:
    """Top-k degree nodes, ties to the smaller index, sorted (engine.py:97-110)."""
    n = deg.size
    nonzero = int((deg > 0).sum())
    if k > nonzero:
        warnings.warn(f"only {nonzero} nodes have nonzero degree; "
                      f"filling {k - nonzero} center(s) in index order")
        chosen = np.lexsort((np.arange(n), -deg))[:nonzero]
        mask = np.zeros(n, dtype=bool)
        mask[chosen] = True
        rest = np.flatnonzero(~mask)[: k - nonzero]
        return np.sort(np.concatenate([chosen, rest]).astype(np.int64))
    if k == n:
        return np.arange(n, dtype=np.int64)
    kth = np.partition(-deg, k - 1)[k - 1]        # -(k-th largest degree)
    above = np.flatnonzero(-deg < kth)
    ties = np.flatnonzero(-deg == kth)[: k - above.size]
    return np.sort(np.concatenate([above, ties]).astype(np.int64))


def _init_labels_device(op: WalkOperator, k: int, t_i: int, alpha: float):
    labels, centers, _, _ = _init_labels_sizes(op, k, t_i, alpha)
    return labels, centers


def _init_labels_sizes(op: WalkOperator, k: int, t_i: int, alpha: float):
    """init_bcm on the device: (labels, centers, device sizes, host sizes)."""
    n = op.n
    if k > n:
        raise NetworkError(f"k={k} exceeds node count n={n}")
    cache = op._fac.__dict__.setdefault("_centers_cache", {})   # degrees are per network
    if k not in cache:
        with warnings.catch_warnings(record=True) as wr:
            warnings.simplefilter("always")
            c_host = _centers(op.degrees, k)
        cache[k] = (c_host, torch.from_numpy(c_host).to(dev()), [str(w.message) for w in wr])
    centers, cdev, msgs = cache[k]
    for m in msgs:
        warnings.warn(m)
    labels = torch.empty(n, dtype=torch.int32, device=dev())
    s64 = op.struct(_lib.F64)
    wsb = _lib.load().ancka_init_workspace_size(s64, k)
    ws = WORKSPACE.get("init", wsb)
    _lib.call("ancka_init_bcm", s64, cdev.data_ptr(), k, t_i, float(alpha), labels.data_ptr(),
              ws.data_ptr(), ws.numel(), _lib.stream())
    sizes_dev = _cluster_sizes_dev(labels, k)
    sizes = sizes_dev.cpu().numpy()
    if (sizes == 0).any():
        warnings.warn("greedy init left empty cluster(s); pinning centers")
        labels[cdev] = torch.arange(k, dtype=torch.int32, device=dev())
        sizes_dev = _cluster_sizes_dev(labels, k)
        sizes = sizes_dev.cpu().numpy()
    return labels, centers, sizes_dev, sizes


def _cluster_sizes_dev(labels: torch.Tensor, k: int) -> torch.Tensor:
    sizes = torch.empty(k, dtype=torch.int64, device=labels.device)
    _lib.call("ancka_cluster_sizes", labels.data_ptr(), labels.numel(), k, sizes.data_ptr(),
              _lib.stream())
    return sizes



def init_bcm(op: WalkOperator, k: int, t_i: int, alpha: float) -> BcmMatrix:
    """Greedy membership seeding (engine.py:87-127), on the device."""
    _lib.require_device()
    labels, _ = _init_labels_device(op, k, t_i, alpha)
    return BcmMatrix(assignment=labels.cpu().numpy().astype(np.int64), k=k)


# --------------------------------------------------------------- QR ---------
def _qr_f64_inplace(z: torch.Tensor, c: int) -> np.ndarray:
    n = z.shape[0]
    rdiag = torch.empty(c, dtype=torch.float64, device=z.device)
    wsb = _lib.load().ancka_qr_f64_workspace_size(n, c)
    ws = WORKSPACE.get("qr64", wsb)
    _lib.call("ancka_qr_f64", z.data_ptr(), n, z.stride(0), c, rdiag.data_ptr(), ws.data_ptr(),
              ws.numel(), _lib.stream())
    return rdiag.cpu().numpy()


class _NoisePrefetch:
    """The first draw of the reference's rank-deficiency noise
    (default_rng(seed).standard_normal((n, 1)), engine.py:141-146) computed on
    a host thread while the device runs the KNN phase: step 1 always flags one
    column.  The generator state after the draw is kept so the
    caller's rng continues exactly as if it had drawn itself."""

    def __init__(self, seed: int, n: int):
        import threading
        self.seed, self.n, self.noise, self.state = seed, n, None, None
        self.fresh = np.random.default_rng(seed).bit_generator.state
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        g = np.random.default_rng(self.seed)
        self.noise = g.standard_normal((self.n, 1))
        self.state = g.bit_generator.state

    def take(self, rng: np.random.Generator, n: int, cols: int):
        if cols != 1 or n != self.n or rng.bit_generator.state != self.fresh:
            return None
        self._t.join()
        rng.bit_generator.state = self.state
        return self.noise


def _exact_step(op: WalkOperator, q64: torch.Tensor, c: int, rng: np.random.Generator,
                prefetch: "_NoisePrefetch | None" = None):
    """orthogonal_step (engine.py:130-149) in f64: apply, QR, the reference's
    rank test on |R_jj|, seeded noise on bad columns, re-QR.  Returns the new
    f64 block (diag R > 0 by construction) and Z."""
    n = op.n
    z = torch.empty_like(q64)
    scr = op.scratch(c, torch.float64)
    _lib.call("ancka_op_apply", op.struct(_lib.F64), q64.data_ptr(), q64.stride(0), c,
              z.data_ptr(), z.stride(0), scr.data_ptr(), _lib.stream())
    q = z.clone()
    d = _qr_f64_inplace(q, c)
    bad = d < 1e-12 * max(1.0, d.max() if d.size else 1.0)
    if bad.any():
        warnings.warn(f"rank-deficient iterate; perturbing {int(bad.sum())} column(s)")
        noise = prefetch.take(rng, n, int(bad.sum())) if prefetch is not None else None
        if noise is None:
            noise = rng.standard_normal((n, int(bad.sum())))
        cols = torch.from_numpy(np.flatnonzero(bad)).to(z.device)
        z[:, cols] += 1e-8 * torch.from_numpy(noise).to(z.device)
        q = z.clone()
        _qr_f64_inplace(q, c)
    return q, z


def orthogonal_step(op: WalkOperator, q_prev, rng: np.random.Generator):
    """One multiply-then-QR step with the reference's rank handling and sign
    convention (engine.py:130-149).  numpy in, numpy (q, r) out."""
    _lib.require_device()
    q_prev = np.asarray(q_prev, dtype=np.float64)
    c = q_prev.shape[1]
    q, z = _exact_step(op, padded(q_prev, torch.float64), c, rng)
    qc, zc = q[:, :c], z[:, :c]
    r = torch.triu(qc.T @ zc)
    return qc.cpu().numpy(), r.cpu().numpy()


# --------------------------------------------------------- discretize -------
#: blocks up to this width run on the device (discretize.cu for k <= 64,
#: disc_wide_dev.cu's device-driven rounds above); wider ones the
#: host-driven path (per-round n-sized work on the device, the k x k SVD on
#: the host as np.linalg.svd)
WIDE_DISCRETIZE_K = 192


class _WideDiscretizer:
    """_alternate_rounding / _prototype_rotation (engine.py:183-218) for k > 192.
    Buffers are per (n, k) and reused across calls."""

    def __init__(self, n: int, k: int):
        d = dev()
        self.n, self.k = n, k
        self.ldt = ld_for(k, torch.float32)
        self.qt = torch.empty((n, self.ldt), dtype=torch.float32, device=d)
        self.zero = torch.zeros(1, dtype=torch.int32, device=d)
        self.lab = [torch.empty(n, dtype=torch.int32, device=d) for _ in range(2)]
        self.margin = torch.empty(n, dtype=torch.float32, device=d)
        self.R = torch.zeros((k, self.ldt), dtype=torch.float32, device=d)
        self.S = torch.empty(k * k, dtype=torch.int64, device=d)
        self.cnt = torch.empty(k, dtype=torch.int64, device=d)
        self.acc = torch.empty(n, dtype=torch.float64, device=d)
        self.rcol = torch.empty(k, dtype=torch.float64, device=d)
        bits = int(np.ceil(np.log2(n + 1)))
        self.shift = 61 - bits                  # |sum| <= n: no int64 overflow
        self.scale = float(2.0 ** self.shift)

    def _reseed(self, lab, sizes):
        """_reseed_empty_columns (engine.py:162-180) with device tensor ops."""
        k = self.k
        empties = np.flatnonzero(sizes == 0)
        if not empties.size or k < 2:
            return
        for c in empties:
            sz = torch.bincount(lab.long(), minlength=k)
            movable = sz[lab.long()] >= 2
            if not bool(movable.any()):
                break
            cand = torch.where(movable, self.margin, torch.full_like(self.margin, -np.inf))
            lab[int(torch.argmax(cand))] = int(c)

    def run(self, R0: np.ndarray, lab, max_iter: int, tol: float):
        n, k = self.n, self.k
        objs, conv, R = [], False, R0
        Rh = torch.empty((k, self.ldt), dtype=torch.float32, pin_memory=True)
        out = torch.empty(k * k + k, dtype=torch.int64, pin_memory=True)
        SC = torch.empty(k * k + k, dtype=torch.int64, device=self.S.device)

        def accumulate():
            # one read-back per round: the k x k fixed-point sums and the sizes
            _lib.call("ancka_disc_accumulate", self.qt.data_ptr(), self.ldt, n, k, lab.data_ptr(),
                      self.scale, SC.data_ptr(), SC[k * k:].data_ptr(), _lib.stream())
            out.copy_(SC)
            return out.numpy()

        for _ in range(max_iter):
            R_used = R                            # rotation behind this round's scores
            Rh[:, :k] = torch.from_numpy(R.astype(np.float32))
            self.R.copy_(Rh, non_blocking=True)
            _lib.call("ancka_disc_score", self.qt.data_ptr(), self.ldt, n, k, self.R.data_ptr(),
                      self.ldt, lab.data_ptr(), self.margin.data_ptr(), _lib.stream())
            h = accumulate()
            if (h[k * k:] == 0).any() and k >= 2:  # reseed empties, then recount
                self._reseed(lab, h[k * k:].copy())
                h = accumulate()
            S = h[:k * k].reshape(k, k).astype(np.float64) / self.scale
            sizes = h[k * k:].astype(np.float64)
            M = np.divide(S, sizes[:, None], out=np.zeros_like(S), where=sizes[:, None] > 0)
            try:
                u, omega, vh = np.linalg.svd(M)     # Y~^T Q~ (engine.py:199-200)
            except np.linalg.LinAlgError:       # gesdd non-convergence: QR-iteration SVD
                import scipy.linalg
                u, omega, vh = scipy.linalg.svd(M, lapack_driver="gesvd")
            objs.append(n - 2.0 * float(omega.sum()))
            if len(objs) >= 2 and abs(objs[-1] - objs[-2]) < tol:
                conv = True
                break
            R = vh.T @ u.T
        return objs, conv, R_used, int((sizes == 0).sum())

    def prototype(self) -> np.ndarray:
        """_prototype_rotation (engine.py:209-218): k - 1 greedy passes."""
        n, k = self.n, self.k
        R = np.zeros((k, k))
        R[:, 0] = self.qt[0, :k].double().cpu().numpy()
        self.acc.zero_()
        for j in range(1, k):
            self.rcol.copy_(torch.from_numpy(R[:, j - 1]))
            _lib.call("ancka_disc_proto_pass", self.qt.data_ptr(), self.ldt, n, k,
                      self.rcol.data_ptr(), self.acc.data_ptr(), _lib.stream())
            i = int(torch.argmin(self.acc))      # first minimum, as np.argmin
            R[:, j] = self.qt[i, :k].double().cpu().numpy()
        return R

    def __call__(self, q32, col0, max_iter, tol, labels_out, info):
        n, k = self.n, self.k
        _lib.call("ancka_disc_normalize", q32.data_ptr(), q32.stride(0), col0, n, k,
                  self.qt.data_ptr(), self.ldt, self.zero.data_ptr(), _lib.stream())
        results = []
        for r, R0 in enumerate((np.eye(k), None)):
            if R0 is None:
                R0 = self.prototype()
            results.append(self.run(R0, self.lab[r], max_iter, tol))
        # identity wins unless the prototype run is lower by more than 1e-15
        win = 1 if results[1][0][-1] < results[0][0][-1] - 1e-15 else 0
        objs, conv, R, empties = results[win]
        labels_out.copy_(self.lab[win])
        head = [objs[-1], len(objs), 1.0 if conv else 0.0, win, empties,
                float(self.zero.item()), len(results[0][0]), len(results[1][0])]
        host = np.zeros(info.numel())
        host[:8] = head
        for r in range(2):
            o = results[r][0]
            host[8 + r * max_iter: 8 + r * max_iter + len(o)] = o
            host[8 + 2 * max_iter + r * k * k: 8 + 2 * max_iter + (r + 1) * k * k] = \
                results[r][2].ravel()
        info.copy_(torch.from_numpy(host))


_WIDE = {}

#: ANCKA_DISC_TIMING=1: the discretize kernel's per-phase timers (ns / clocks,
#: slots as tools/disc_timing.py names them) summed over the calls of a run
DISC_PROFILE = {} if os.environ.get("ANCKA_DISC_TIMING") else None


def _disc_profile_add(info, k):
    t = info[8 + 2 * DISCRETIZE_MAX_ITER + 2 * k * k:].cpu().numpy().view(np.uint64)
    h = info[:8].cpu().numpy()
    DISC_PROFILE["calls"] = DISC_PROFILE.get("calls", 0) + 1
    DISC_PROFILE["rounds"] = DISC_PROFILE.get("rounds", 0) + int(h[6] + h[7])
    for i, v in enumerate(t):
        DISC_PROFILE[i] = DISC_PROFILE.get(i, 0) + int(v)


def _discretize_device(q32: torch.Tensor, col0: int, k: int, max_iter: int, tol: float,
                       labels_out: torch.Tensor, info: torch.Tensor):
    n = q32.shape[0]
    if k > WIDE_DISCRETIZE_K:
        w = _WIDE.get((n, k))
        if w is None:
            w = _WIDE[(n, k)] = _WideDiscretizer(n, k)
        w(q32, col0, max_iter, tol, labels_out, info)
        return
    wsb = _lib.load().ancka_discretize_workspace_size(n, k, max_iter)
    ws = WORKSPACE.get("disc", wsb)
    _lib.call("ancka_discretize", q32.data_ptr(), q32.stride(0), col0, n, k, max_iter, float(tol),
              labels_out.data_ptr(), info.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())


def discretize(q, max_iter: int = DISCRETIZE_MAX_ITER, tol: float = DISCRETIZE_TOL) -> DiscretizeResult:
    """Alternating argmax rounding / Procrustes rotation from the identity and
    the prototype start (engine.py:221-263), one cooperative kernel."""
    _lib.require_device()
    qh = np.asarray(q, dtype=np.float64) if not isinstance(q, torch.Tensor) else q
    if qh.ndim != 2 or qh.shape[1] < 1:
        raise NetworkError("discretize expects an n x k block with k >= 1")
    n, k = qh.shape
    q32 = padded(torch.as_tensor(qh), torch.float32)
    labels = torch.empty(n, dtype=torch.int32, device=dev())
    info = torch.zeros(8 + 2 * max_iter + 2 * k * k, dtype=torch.float64, device=dev())
    _discretize_device(q32, 0, k, max_iter, tol, labels, info)
    inf = info.cpu().numpy()
    if inf[5] > 0:
        warnings.warn(f"{int(inf[5])} all-zero row(s); assigning to cluster 0")
    win = int(inf[3])
    runs = tuple((name, list(inf[8 + r * max_iter: 8 + r * max_iter + int(inf[6 + r])]))
                 for r, name in enumerate(("identity", "prototype")))
    rot = inf[8 + 2 * max_iter + win * k * k: 8 + 2 * max_iter + (win + 1) * k * k].reshape(k, k)
    qd = torch.as_tensor(qh, dtype=torch.float64, device=dev())
    nrm = torch.linalg.vector_norm(qd, dim=1, keepdim=True)
    qt = torch.where(nrm > 0, qd / torch.where(nrm > 0, nrm, torch.ones_like(nrm)), torch.zeros_like(qd))
    scores = (qt @ torch.from_numpy(rot).to(qd.device)).cpu().numpy()
    lab = labels.cpu().numpy().astype(np.int64)
    return DiscretizeResult(y=BcmMatrix(assignment=lab, k=k), scores=scores,
                            objectives=runs[win][1], iterations=int(inf[1]),
                            converged=bool(inf[2]), runs=runs)


def repair_empty_clusters(y: BcmMatrix, scores: np.ndarray) -> BcmMatrix:
    """Margin-based re-seeding of empty clusters (engine.py:266-288).  Host
    API helper; inside run_ancka the discretisation kernel performs it."""
    empties = y.empty_clusters()
    if not empties.size:
        return y
    warnings.warn(f"re-seeding {empties.size} empty cluster(s) after discretization")
    a = y.assignment.copy()
    margin = np.partition(scores, -2, axis=1)[:, -2] if scores.shape[1] >= 2 else scores[:, 0]
    for c in empties:
        movable = np.bincount(a, minlength=y.k)[a] >= 2
        if not movable.any():
            raise NetworkError("cannot repair empty clusters: no movable nodes")
        a[int(np.argmax(np.where(movable, margin, -np.inf)))] = c
    return BcmMatrix(assignment=a, k=y.k)


def _repair_missing_columns(q32: torch.Tensor, kd: int, k: int, labels: torch.Tensor,
                            info: torch.Tensor) -> None:
    """k == n: the discretised block has kd = n - 1 < k columns, so clusters
    kd..k-1 are empty and repair_empty_clusters (engine.py:266-288) fills them
    from the winning run's final scores.  Degenerate (tiny n) case: the scores
    are rebuilt on the host from the winning rotation the kernel reports."""
    inf = info.cpu().numpy()
    win = int(inf[3])
    base = 8 + 2 * DISCRETIZE_MAX_ITER + win * kd * kd
    rot = inf[base: base + kd * kd].reshape(kd, kd)
    q = q32[:, 1:1 + kd].double().cpu().numpy()
    nrm = np.linalg.norm(q, axis=1)
    qt = np.divide(q, nrm[:, None], out=np.zeros_like(q), where=nrm[:, None] > 0)
    y = BcmMatrix(assignment=labels.cpu().numpy().astype(np.int64), k=k)
    y = repair_empty_clusters(y, qt @ rot)
    labels.copy_(torch.from_numpy(y.assignment.astype(np.int32)))


# ---------------------------------------------------------------- MHC -------
class _MhcRunner:
    def __init__(self, op: WalkOperator, k: int, dtype: int):
        self.op, self.k, self.dtype = op, k, dtype
        self.s = op.struct(dtype)
        self.ws = WORKSPACE.get(f"mhc{dtype}", _lib.load().ancka_mhc_workspace_size(self.s, k))
        self.phi = torch.zeros(1, dtype=torch.float64, device=dev())
        self.sizes = torch.zeros(k, dtype=torch.int64, device=dev())

    def __call__(self, labels: torch.Tensor, phi_out: torch.Tensor | None = None):
        out = self.phi if phi_out is None else phi_out
        _lib.call("ancka_mhc", self.s, labels.data_ptr(), self.k, self.op.alpha, self.op.gamma,
                  out.data_ptr(), self.sizes.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                  _lib.stream())
        return out


def calc_mhc(op: WalkOperator, y: BcmMatrix) -> float:
    """Multi-hop conductance (engine.py:291-299), f64 on the device."""
    _lib.require_device()
    normalize_bcm(y)  # raises on empty clusters, as the reference
    lab = torch.from_numpy(y.assignment.astype(np.int32)).to(dev())
    return float(_MhcRunner(op, y.k, _lib.F64)(lab).item())


# ------------------------------------------------------------ pipeline ------
@dataclass
class PreparedNetwork:
    """A validated network whose attributes and structural factors are
    resident in HBM: the input of the device pipeline (build_pipeline_device)."""

    net: AttributedNetwork
    K: int
    x_dev: object           # knn.DeviceAttributes
    x_level: int            # 2 fp8-exact, 1 bf16-exact, 0 general (knn.integer_exact)
    factors: StructureFactors | None   # None: structure not validated / uploaded yet
    cache_path: object = None

    def finish_structure(self) -> None:
        """Host validation of the structure (network.py:266-313) and the
        structural uploads on a side stream.  run_ancka calls it after the
        KNN launch, so this host work overlaps the KNN on the device (the
        attributes -- all the KNN reads -- are not changed by validation)."""
        if self.factors is not None:
            return
        main = torch.cuda.current_stream()
        side = _structure_stream()
        with torch.cuda.stream(side):
            self.net, report = validate_network(self.net)
            self.factors = StructureFactors(self.net, report.degrees)
        main.wait_stream(side)

    def h2d_bytes(self, x) -> int:
        import scipy.sparse as sp
        xb = (x.indptr.nbytes + x.indices.nbytes + x.data.nbytes) if sp.issparse(x) else x.nbytes
        return int(xb + self.factors.h2d_bytes())


_SIDE_STREAMS: dict = {}


def _structure_stream() -> torch.cuda.Stream:
    """One persistent side stream per device (the caching allocator keeps
    per-stream pools: a fresh stream per run would miss them every time)."""
    d = torch.cuda.current_device()
    if d not in _SIDE_STREAMS:
        _SIDE_STREAMS[d] = torch.cuda.Stream(device=d)
    return _SIDE_STREAMS[d]


def prepare_network(net: AttributedNetwork, params: ClusterParams, knn_cache_dir=None, *,
                    defer_structure: bool = False) -> PreparedNetwork:
    """Host validation (network.py:266-313) and the one-time uploads.
    defer_structure: upload the attributes only; the structure is validated
    and uploaded by PreparedNetwork.finish_structure (after the KNN launch)."""
    from pathlib import Path

    _lib.require_device()
    report = None
    if not defer_structure:
        net, report = validate_network(net)
    params.validate_for(net.n)
    K = params.knn_k if params.knn_k is not None else default_knn_k(net.kind, net.n)
    if K >= net.n:
        warnings.warn(f"clamping KNN K={K} to n-1={net.n - 1}")
        K = net.n - 1
    cache_path = None
    if knn_cache_dir is not None:
        cache_path = Path(knn_cache_dir) / f"{cache_key(net.attributes, K, params.knn_mode)}.aknn"
    xd = attributes_to_device(net.attributes, None if K <= 32 else 0)
    factors = None if report is None else StructureFactors(net, report.degrees)
    return PreparedNetwork(net, K, xd, xd.level, factors, cache_path)


def build_pipeline_device(prep: PreparedNetwork, params: ClusterParams):
    """Exact KNN, KNN graph and walk operator on the device (engine.py:314-339)."""
    K, n = prep.K, prep.net.n
    neighbors, mode_used = None, None
    if prep.cache_path is not None and prep.cache_path.exists():
        neighbors, mode_used = load_neighbor_cache(prep.cache_path)
    if neighbors is None:
        if resolve_knn_mode(params.knn_mode, n) is KnnMode.APPROX:      # knn.py:286-291
            neighbors = knn_search_approx(prep.x_dev, K, seed=params.seed)
            mode_used = KnnMode.APPROX
        else:
            ids, scores = knn_search_exact_device(prep.x_dev, K, integer=prep.x_level)
            neighbors, mode_used = NeighborLists(ids_dev=ids, scores_dev=scores, K=K), KnnMode.EXACT
        if prep.cache_path is not None:
            prep.cache_path.parent.mkdir(parents=True, exist_ok=True)
            save_neighbor_cache(prep.cache_path, neighbors, mode_used)
    prep.finish_structure()          # host work overlapping the KNN kernel
    ids, scores = neighbors.device()
    A, P, zero = build_knn_graph_device(ids, scores, n)
    g = KnnGraph(A, P, zero, neighbors, mode_used)
    op = build_walk_operator(prep.net, P, zero, params.alpha, params.beta, params.gamma,
                             factors=prep.factors)
    return op, g


def build_pipeline(net: AttributedNetwork, params: ClusterParams, knn_cache_dir=None):
    """Validate (host), exact KNN + KNN graph + walk operator (device)
    (engine.py:302-340).  Returns (operator, KnnGraph, timings)."""
    t0 = time.perf_counter()
    prep = prepare_network(net, params, knn_cache_dir)
    op, g = build_pipeline_device(prep, params)
    torch.cuda.current_stream().synchronize()
    return op, g, {"knn_ms": (time.perf_counter() - t0) * 1e3}


class _Loop:
    """Device buffers and captured tau-block graphs of the f32 iteration."""

    def __init__(self, op: WalkOperator, c: int, k: int, tau: int, use_graphs: bool,
                 fused: bool = True):
        self.op, self.c, self.k, self.tau = op, c, k, tau
        n = op.n
        # narrow blocks use the fused cooperative kernel, which wants ld == 8
        self.fused = (fused and c <= 8 and op.kind is not NetworkKind.MULTIPLEX
                      and not os.environ.get("ANCKA_ORTH_UNFUSED"))
        self.ld = 8 if self.fused else ld_for(c, torch.float32)
        d = dev()
        self.Q = [torch.zeros((n, self.ld), dtype=torch.float32, device=d) for _ in range(2)]
        self.Z = torch.zeros((n, self.ld), dtype=torch.float32, device=d)
        self.Qsave = torch.zeros((n, self.ld), dtype=torch.float32, device=d)
        self.stats = torch.zeros(16, dtype=torch.float64, device=d)   # [4:12] debug timers
        self._flag_init = torch.tensor([1.0, 0.0], dtype=torch.float64, device=d)
        self.s32 = op.struct(_lib.F32)
        self.ws = WORKSPACE.get("orth", _lib.load().ancka_orth_workspace_size(self.s32, c))
        if self.fused:
            self.ws_fused = WORKSPACE.get("orth_block", _lib.load().ancka_orth_block_workspace_size(self.s32))
        self.cur = 0
        self.use_graphs = use_graphs
        self.graphs = {}
        self.captured = 0   # kernel launches recorded into graphs (not executed)
        self.replayed = 0   # kernel launches executed by graph replays

    def reset_flags(self):
        self.stats[1:3].copy_(self._flag_init)   # device->device: capturable

    def _step(self, src: int):
        _lib.call("ancka_orth_step_f32", self.s32, self.Q[src].data_ptr(), self.Q[1 - src].data_ptr(),
                  self.Z.data_ptr(), self.ld, self.c, self.stats.data_ptr(), self.ws.data_ptr(),
                  self.ws.numel(), _lib.stream())

    def _block(self, start: int, steps: int):
        self.Qsave.copy_(self.Q[start])
        self.reset_flags()
        src = start
        for _ in range(steps):
            self._step(src)
            src = 1 - src

    def replay_exact(self, rng):
        """Redo the last block from its saved start with exact f64 steps."""
        start, steps = self.last
        self.Q[start].copy_(self.Qsave)
        src = start
        for _ in range(steps):
            q64 = self.Q[src][:, : self.c].double()
            q, _ = _exact_step(self.op, padded(q64, torch.float64), self.c, rng)
            self.Q[1 - src][:, : self.c] = q[:, : self.c].to(torch.float32)
            src = 1 - src
        self.stats[0] = torch.sum((self.Q[src][:, : self.c].double()
                                   - self.Q[1 - src][:, : self.c].double()) ** 2)
        self.stats[2] = 0.0
        self.cur = src

    def run(self, steps: int):
        """Advance `steps` f32 orthogonal steps from Q[cur]."""
        start = self.cur
        self.last = (start, steps)
        if self.fused:
            self.Qsave.copy_(self.Q[start])
            self.reset_flags()
            _lib.call("ancka_orth_block_f32", self.s32, self.Q[start].data_ptr(),
                      self.Q[1 - start].data_ptr(), self.Z.data_ptr(), self.ld, self.c, steps,
                      self.stats.data_ptr(), self.ws_fused.data_ptr(), self.ws_fused.numel(),
                      _lib.stream())
        elif self.use_graphs and steps == self.tau:
            g = self.graphs.get(start)
            if g is None:
                self._block(start, steps)          # warm-up
                torch.cuda.current_stream().synchronize()
                self.Q[start].copy_(self.Qsave)    # undo the warm-up
                # manual capture on a side stream: torch.cuda.graph() would run
                # gc.collect() + empty_cache() on every capture
                g = torch.cuda.CUDAGraph()
                c0 = _lib.load().ancka_launch_count()
                cur = torch.cuda.current_stream()
                side = torch.cuda.Stream()
                side.wait_stream(cur)
                with torch.cuda.stream(side):
                    g.capture_begin()
                    self._block(start, steps)
                    g.capture_end()
                cur.wait_stream(side)
                nodes = _lib.load().ancka_launch_count() - c0
                self.graphs[start] = (g, nodes)
                self.captured += nodes             # captured, not executed
            g, nodes = self.graphs[start]
            g.replay()
            self.replayed += nodes
        else:
            self._block(start, steps)
        self.cur = (start + steps) % 2

    @property
    def q(self) -> torch.Tensor:
        return self.Q[self.cur]


def run_ancka(net: AttributedNetwork, params: ClusterParams, knn_cache_dir=None,
              early_stop: bool = True, *, use_graphs: bool = False, fused: bool = True) -> ClusterResult:
    """Full clustering pipeline (engine.py:343-437): host validation and
    uploads, then the device-resident pipeline (`run_prepared`)."""
    _lib.require_device()
    with warnings.catch_warnings(record=True) as wrec:
        warnings.simplefilter("always")
        t0 = time.perf_counter()
        prep = prepare_network(net, params, knn_cache_dir, defer_structure=True)
        prep_ms = (time.perf_counter() - t0) * 1e3
    res = run_prepared(prep, params, early_stop, use_graphs=use_graphs, fused=fused)
    res.timings_ms["knn_ms"] += prep_ms
    res.warnings = [str(w.message) for w in wrec] + res.warnings
    return res


def run_prepared(prep: PreparedNetwork, params: ClusterParams, early_stop: bool = True, *,
                 use_graphs: bool = False, fused: bool = True) -> ClusterResult:
    """The device pipeline on HBM-resident inputs: KNN -> KNN graph ->
    operator -> init -> orthogonal iterations / discretisation / MHC."""
    _lib.require_device()
    timer = _PhaseTimer()
    launches0 = _lib.load().ancka_launch_count()
    prefetch = _NoisePrefetch(params.seed, prep.net.n)
    with warnings.catch_warnings(record=True) as wrec:
        warnings.simplefilter("always")
        with timer.span("knn_ms"):
            op, g = build_pipeline_device(prep, params)
        n, k = op.n, params.k
        # KNN / graph-assembly buffers are dead from here on (tens of GB at
        # 1e7+ nodes); the allocator reuses the memory for the loop's blocks
        WORKSPACE.release("knn", "knn_graph", "csr_transpose", "row_split")
        with timer.span("init_ms"):
            labels0, _, sizes0_dev, sizes0 = _init_labels_sizes(op, k, params.t_i, params.alpha)
        WORKSPACE.release("init")
        op.set_locality(labels0, k)       # row order of the f32 graph applies (L2 reuse)
        rng = np.random.default_rng(params.seed)
        c = min(k + 1, n)
        # Q0 = [1/sqrt(n) | Yhat0] (engine.py:368-371), f64 for the exact first step
        ld64 = ld_for(c, torch.float64)
        q0 = torch.empty((n, ld64), dtype=torch.float64, device=dev())
        _lib.call("ancka_bcm_block", labels0.data_ptr(), n, c, sizes0_dev.data_ptr(),
                  1.0 / np.sqrt(n), q0.data_ptr(), ld64, _lib.stream())
        with timer.span("mhc_ms"):
            if (sizes0 == 0).any():
                raise NetworkError(f"empty cluster(s) {np.flatnonzero(sizes0 == 0).tolist()}: "
                                   "normalization undefined")
            # phi(Y0) stays on the device; it rides along with the first sample's
            # read-back (no synchronisation here)
            mhc0_dev = _MhcRunner(op, k, _lib.F64)(labels0)
        WORKSPACE.release(f"mhc{_lib.F64}")          # 2 n k f64: re-acquired at the end
        best_mhc = None
        best_labels = labels0.clone()
        history = [(0, None)]
        loop = _Loop(op, c, k, params.tau, use_graphs, fused)
        mhc = _MhcRunner(op, k, _lib.F32)
        lab_t = torch.empty(n, dtype=torch.int32, device=dev())
        # (+16: per-phase timers when ANCKA_DISC_TIMING is set)
        info = torch.zeros(8 + 2 * DISCRETIZE_MAX_ITER + 2 * k * k + 16, dtype=torch.float64,
                           device=dev())
        error, stop_reason, converged, t = None, "max_iterations", False, 0
        host_info = torch.empty(8, dtype=torch.float64, pin_memory=True)
        host_rb = torch.empty(4, dtype=torch.float64, pin_memory=True)
        host_rb0 = torch.empty(1, dtype=torch.float64, pin_memory=True)
        rb_ready = torch.cuda.Event()
        # MHC reuse: a sample whose labels are the previous evaluated sample's
        # partition relabelled repeats its phi exactly (calc_mhc depends on
        # the partition only) -- the check is one small kernel and a flag read
        mhc_reuse = MHC_REUSE
        lab_mhc = torch.empty(n, dtype=torch.int32, device=dev()) if mhc_reuse else None
        same_ws = torch.empty(2 * k, dtype=torch.int32, device=dev()) if mhc_reuse else None
        same_dev = torch.zeros(1, dtype=torch.int32, device=dev())
        host_same = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        same_ready = torch.cuda.Event()
        phi_last = torch.zeros(1, dtype=torch.float64, device=dev())
        have_mhc = False
        mhc_reused = 0

        # discretize(state.q[:, 1:]) sees c - 1 columns: fewer than k only in
        # the degenerate k == n case (engine.py:370-371, 392-394)
        kd = c - 1

        def sample_issue(t_now, dq_first):
            # loop.stats = [dq^2, min pivot ratio, suspect pivots, phi]: one
            # read-back per sample next to the discretisation info
            if kd < 1:
                raise NetworkError("discretize expects an n x k block with k >= 1")
            qt = loop.q
            with timer.span("discretize_ms"):
                _discretize_device(qt, 1, kd, DISCRETIZE_MAX_ITER, DISCRETIZE_TOL, lab_t, info)
                if DISC_PROFILE is not None:
                    _disc_profile_add(info, kd)
                if kd < k:
                    _repair_missing_columns(qt, kd, k, lab_t, info)
            nonlocal have_mhc, mhc_reused
            with timer.span("mhc_ms"):
                same = False
                if mhc_reuse and have_mhc:
                    _lib.call("ancka_same_partition", lab_mhc.data_ptr(), lab_t.data_ptr(), n, k,
                              same_ws.data_ptr(), same_dev.data_ptr(), _lib.stream())
                    host_same.copy_(same_dev, non_blocking=True)
                    same_ready.record()
                    same_ready.synchronize()
                    same = bool(host_same[0])
                if same:
                    loop.stats[3:4].copy_(phi_last)
                    mhc_reused += 1
                else:
                    mhc(lab_t, loop.stats[3:4])
                    if mhc_reuse:
                        phi_last.copy_(loop.stats[3:4])
                        lab_mhc.copy_(lab_t)
                        have_mhc = True
            op.set_locality(lab_t, k)     # regroup the apply's rows by the current clusters
            if dq_first is not None:
                loop.stats[0] = dq_first * dq_first
                loop.stats[2] = 0.0
            if best_mhc is None:
                host_rb0.copy_(mhc0_dev, non_blocking=True)
            host_info.copy_(info[:8], non_blocking=True)
            host_rb.copy_(loop.stats[:4], non_blocking=True)
            rb_ready.record()

        def sample_collect():
            nonlocal best_mhc
            rb_ready.synchronize()
            if best_mhc is None:                    # phi(Y0) (engine.py:373)
                best_mhc = float(host_rb0[0])
                history[0] = (0, best_mhc)
            rb = host_rb.numpy()
            return host_info.numpy().copy(), (float(rb[3]), float(rb[0]), float(rb[2]))

        def sample(t_now, dq_first):
            sample_issue(t_now, dq_first)
            return sample_collect()

        Qsave_prev = torch.empty_like(loop.Qsave)
        disc_rounds = []            # rounds (both starts) of every discretisation
        best_sampled = False        # best labels from a sample (phi in f32) or Y0 (f64)

        spec = None
        try:
            # ---- t = 1: exact f64 step on the rank-deficient block
            t = 1
            with timer.span("ortho_ms"):
                q1, _ = _exact_step(op, q0, c, rng, prefetch)
                loop.Q[0][:, :c] = q1[:, :c].to(torch.float32)
                loop.cur = 0
                dq1 = torch.linalg.vector_norm(q1[:, :c] - q0[:, :c])
                del q1, q0
            t_done = 1
            sample_needed = params.tau == 1
            # spec: a tau-block enqueued while the sample is read back

            # the fused path holds no captured pointer to loop.Qsave, so the
            # save of the previous block start is a buffer swap, not a copy
            swap_saves = loop.fused or not loop.use_graphs

            def save_prev():
                nonlocal Qsave_prev
                if swap_saves:
                    Qsave_prev, loop.Qsave = loop.Qsave, Qsave_prev
                else:
                    Qsave_prev.copy_(loop.Qsave)

            def undo_spec():
                # return to the iterate at t_done: the speculative block saved it
                nonlocal Qsave_prev
                start, prev_last = spec[1], spec[2]
                loop.Q[start].copy_(loop.Qsave)
                loop.cur = start
                if swap_saves:
                    Qsave_prev, loop.Qsave = loop.Qsave, Qsave_prev
                else:
                    loop.Qsave.copy_(Qsave_prev)
                loop.last = prev_last

            while True:
                if sample_needed:
                    t = t_done
                    sample_issue(t_done, dq1 if t_done == 1 else None)
                    if t_done < params.t_a:
                        # overlap the host decision with the next block (discarded on stop)
                        nxt_s = min(params.t_a, (t_done // params.tau + 1) * params.tau)
                        save_prev()
                        spec = (nxt_s, loop.cur, getattr(loop, "last", None))
                        with timer.span("ortho_ms"):
                            loop.run(nxt_s - t_done)
                    inf, (phi, dq2, nbad) = sample_collect()
                    if nbad > 0:
                        # a suspect Cholesky pivot: replay the block with exact f64 steps
                        if spec is not None:
                            undo_spec()
                            spec = None
                        warnings.warn("ill-conditioned iterate; replaying tau-block in f64")
                        with timer.span("ortho_ms"):
                            loop.replay_exact(rng)
                        inf, (phi, dq2, nbad) = sample(t_done, None)
                    disc_rounds.append(int(inf[6]) + int(inf[7]))
                    if inf[5] > 0:
                        warnings.warn(f"{int(inf[5])} all-zero row(s); assigning to cluster 0")
                    if inf[4] > 0:
                        warnings.warn(f"re-seeding {int(inf[4])} empty cluster(s) after discretization")
                        raise NetworkError("cannot repair empty clusters: no movable nodes")
                    history.append((t, float(phi)))
                    if phi < best_mhc:
                        best_mhc = float(phi)
                        best_labels.copy_(lab_t)
                        best_sampled = True
                    if float(np.sqrt(dq2)) < params.eps_q:
                        stop_reason, converged = "subspace_converged", True
                        if spec is not None:
                            undo_spec()
                        break
                    if early_stop and len(history) >= 3:
                        p = [v for _, v in history[-3:]]
                        if p[0] < p[1] < p[2]:
                            stop_reason, converged = "mhc_rising", True
                            if spec is not None:
                                undo_spec()
                            break
                    # (span events are resolved once at the end: resolving them here
                    # would wait for the speculative block and idle the device)
                if t_done >= params.t_a:
                    t = t_done
                    break
                if spec is not None:            # the next block already ran
                    nxt, spec = spec[0], None
                else:
                    nxt = min(params.t_a, (t_done // params.tau + 1) * params.tau)
                    with timer.span("ortho_ms"):
                        loop.run(nxt - t_done)
                t_done = nxt
                t = t_done
                sample_needed = t_done % params.tau == 0
        except NetworkError as exc:
            error, stop_reason = str(exc), "error"
            if spec is not None:
                undo_spec()
        if best_mhc is None:                        # no sample was taken
            best_mhc = float(mhc0_dev.item())
            history[0] = (0, best_mhc)
        if best_sampled:
            # the loop compares f32 phi values (engine.py:403); the returned
            # phi of the best labels is the f64 calc_mhc, as the reference's
            with timer.span("mhc_ms"):
                best_mhc = float(_MhcRunner(op, k, _lib.F64)(best_labels).item())
        caught = [str(w.message) for w in wrec]
    best_y = BcmMatrix(assignment=best_labels.cpu().numpy().astype(np.int64), k=k)
    state = EngineState(loop.q, best_y, best_mhc, history, t, c=c)
    res = ClusterResult(y=best_y, mhc=best_mhc, iterations=t, timings_ms=_LazyTimings(timer),
                        state=state, knn=g, operator=op, converged=converged,
                        stop_reason=stop_reason, warnings=caught, error=error)
    # kernels of this library executed by the run (graph captures excluded,
    # graph replays included)
    res.disc_rounds = disc_rounds
    res.gpu_launches = int(_lib.load().ancka_launch_count() - launches0 - loop.captured
                           + loop.replayed)
    return res

