"""Row-partitioned multi-GPU ANCKA.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank r
owns a contiguous block of node rows [r0, r1) (balanced by operator
nonzeros) and, for hypergraphs, a block of hyperedges [e0, e1):

* KNN       query-stationary ring: rank r keeps its rows [r0, r1) as queries
            and as its first key block; the other key shards travel around
            the ring (P2P send/recv, overlapped with the kernel).  Each step
            ranks (own rows + visiting shard) and merges the lists exactly
            (score desc, index asc), so every rank ends with its rows' global
            top-K holding only 2 shards of X at a time; the lists are then
            all-gathered and A_K / P_K are assembled on every rank.
* operator  per apply: all-gather Q (n x c); hypergraphs compute their share
            of T = P_E Q and all-gather T; each rank produces its rows of
            Z = (I-B) P_struct Q + B P_K Q.
* QR        local Gram Z_r^T Z_r -> all-reduce (c x c) -> every rank factors
            the same R and applies R^-1 to its rows; ||dQ||^2 is all-reduced.
* step 1    (rank deficient) Z^(1) is all-gathered in f64 and
            the exact f64 QR with the reference's rank test and noise draw is
            replicated, so every rank holds the reference's Q^(1).
* init/MHC  the transposed / joint applies are row-partitioned the same way;
            the MHC trace is all-reduced.
* discretisation is replicated on the gathered Q (identical on every rank).

The orchestration is backend-generic: `CudaBackend` drives libancka_b200
kernels and NCCL; the CPU tests drive the same code with a numpy backend over
gloo (tests/test_dist.py), which is how the N>1 logic is verified without
several GPUs.
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .network import (AttributedNetwork, BcmMatrix, ClusterParams, NetworkError, NetworkKind,
                      default_knn_k, node_degrees, symmetrize_union, validate_network)


# ----------------------------------------------------------------------------
def partition_rows(cost: np.ndarray, world: int) -> np.ndarray:
    """Contiguous row blocks with ~equal total cost: boundaries[world + 1]."""
    n = cost.size
    c = np.concatenate([[0.0], np.cumsum(cost, dtype=np.float64)])
    targets = c[-1] * np.arange(1, world) / world
    cuts = np.searchsorted(c, targets, side="left")
    b = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    return np.maximum.accumulate(np.clip(b, 0, n))


def _row_normalize(a: sp.csr_matrix) -> sp.csr_matrix:
    rs = np.asarray(a.sum(axis=1)).ravel()
    inv = np.divide(1.0, rs, out=np.zeros_like(rs), where=rs > 0)
    p = (sp.diags(inv) @ a).tocsr()
    p.sort_indices()
    return p


@dataclass
class Plan:
    """Ownership of rows / hyperedges for one rank."""
    rank: int
    world: int
    n: int
    m: int
    rows: np.ndarray      # world + 1 node-row boundaries
    edges: np.ndarray     # world + 1 hyperedge boundaries (hypergraph)

    @property
    def r0(self):
        return int(self.rows[self.rank])

    @property
    def r1(self):
        return int(self.rows[self.rank + 1])

    @property
    def e0(self):
        return int(self.edges[self.rank])

    @property
    def e1(self):
        return int(self.edges[self.rank + 1])

    def row_counts(self):
        return np.diff(self.rows)

    def edge_counts(self):
        return np.diff(self.edges)


class HostFactors:
    """Structural factors of the validated network, normalised on the host
    exactly as the reference (walk.py:38-79); sliced per rank."""

    def __init__(self, net: AttributedNetwork):
        self.kind = net.kind
        self.n = net.n
        self.degrees = node_degrees(net)
        if net.kind is NetworkKind.HYPERGRAPH:
            h = net.incidence
            self.p_v = _row_normalize(h.T.tocsr())
            self.p_e = _row_normalize(h)
            self.t_a = self.p_v.T.tocsr()      # P_V^T  (m x n)
            self.t_b = self.p_e.T.tocsr()      # P_E^T  (n x m)
            for mtx in (self.t_a, self.t_b):
                mtx.sort_indices()
            self.m = h.shape[0]
        else:
            a = symmetrize_union(net.adjacency) if net.directed else net.adjacency
            self.p_n = _row_normalize(a)
            self.t_a = self.p_n.T.tocsr()
            self.t_a.sort_indices()
            self.m = 0

    def row_cost(self, K: int) -> np.ndarray:
        s = self.p_v if self.kind is NetworkKind.HYPERGRAPH else self.p_n
        return np.diff(s.indptr).astype(np.float64) + 2 * K + 1


def make_plan(fac: HostFactors, K: int, rank: int, world: int) -> Plan:
    rows = partition_rows(fac.row_cost(K), world)
    if fac.kind is NetworkKind.HYPERGRAPH:
        edges = partition_rows(np.diff(fac.p_e.indptr).astype(np.float64) + 1, world)
    else:
        edges = np.zeros(world + 1, dtype=np.int64)
    return Plan(rank, world, fac.n, fac.m, rows, edges)


# ----------------------------------------------------------------------------
class DistOperator:
    """A rank's share of the joint-walk operator (row slices, backend handles)."""

    def __init__(self, B, fac: HostFactors, plan: Plan, p_k_rows, beta_full: np.ndarray,
                 selfloop_full: np.ndarray, alpha: float, gamma: int):
        self.B, self.plan, self.kind = B, plan, fac.kind
        self.alpha, self.gamma = alpha, gamma
        r0, r1 = plan.r0, plan.r1
        if fac.kind is NetworkKind.HYPERGRAPH:
            self.S = B.csr(fac.p_v[r0:r1])             # n_loc x m, gathers T
            self.E = B.csr(fac.p_e[plan.e0:plan.e1])   # m_loc x n, gathers Q
            self.TA = B.csr(fac.t_a[plan.e0:plan.e1])  # P_V^T rows: m_loc x n
            self.TB = B.csr(fac.t_b[r0:r1])            # P_E^T rows: n_loc x m
        else:
            self.S = B.csr(fac.p_n[r0:r1])
            self.TA = B.csr(fac.t_a[r0:r1])
        self.K = p_k_rows
        self.beta = B.vec(beta_full[r0:r1])
        self.selfloop = B.mask(selfloop_full[r0:r1])

    # -- joint apply (walk.py:177-190) on the local rows; Q_full gathered
    def apply(self, Q_full, c, dtype, tag=None, tagval=None, scale=1.0):
        B, pl = self.B, self.plan
        if self.kind is NetworkKind.HYPERGRAPH:
            T_loc = B.spmm(self.E, Q_full, None, None, None, None, None, 0, None, None, 1.0, c, dtype)
            T_full = B.all_gather_rows(T_loc, pl.edge_counts())
            src = T_full
        else:
            src = Q_full
        return B.spmm(self.S, src, self.K, Q_full, self.beta, self.selfloop, Q_full, pl.r0,
                      tag, tagval, scale, c, dtype)

    # -- transposed structure apply (walk.py:153-174) with the init epilogue
    def apply_t(self, P_full, c, tag, tagval, scale):
        B, pl = self.B, self.plan
        if self.kind is NetworkKind.HYPERGRAPH:
            U_loc = B.spmm(self.TA, P_full, None, None, None, None, None, 0, None, None, 1.0, c, "f64")
            U_full = B.all_gather_rows(U_loc, pl.edge_counts())
            return B.spmm(self.TB, U_full, None, None, None, self.selfloop, P_full, pl.r0,
                          tag, tagval, scale, c, "f64")
        return B.spmm(self.TA, P_full, None, None, None, self.selfloop, P_full, pl.r0,
                      tag, tagval, scale, c, "f64")


def knn_ring(B, X, K: int, plan: Plan):
    """Exact top-K of rows [r0, r1) against all n keys, with only the own shard
    and one visiting shard of X resident (SURVEY.md §8(e) KNN ring).

    Step 0 ranks the own rows; step s ranks (own rows + the shard of rank
    r - s).  Every key of shard b that belongs to a row's global top-K is in
    that row's top-K over (own rows + shard b) -- its rank there cannot exceed
    its global rank -- so merging the step lists by (score desc, index asc)
    and keeping K gives the global lists exactly."""
    rank, world = plan.rank, plan.world
    r0, r1 = plan.r0, plan.r1
    mine = B.x_shard(X, r0, r1)
    ids, sc = B.knn_local(mine, None, K, r0, 0)
    block, src = mine, rank
    pending = B.ring_start(block) if world > 1 else None
    for _step in range(1, world):
        block, src = B.ring_finish(pending), (src - 1) % world
        pending = B.ring_start(block) if _step < world - 1 else None   # overlaps the kernel
        i2, s2 = B.knn_local(mine, block, K, r0, int(plan.rows[src]))
        ids, sc = B.merge_lists(ids, sc, i2, s2, K)
    return ids, sc


def discretize_dist(B, Q_loc, k: int, plan: Plan, max_iter: int = 100, tol: float = 1e-10):
    """discretize (engine.py:183-263) row-partitioned:
    argmax and the cluster sums are local; per round the k x k sums and the
    k counts are all-reduced and every rank runs the same k x k SVD.  The
    empty-cluster reseed and the prototype start use global (value, index)
    reductions.  Returns (local labels as numpy, global empties count)."""
    n = plan.n
    qt = B.disc_prepare(Q_loc, 1, k)

    def gather_best(v, gidx, extra=0.0, want_max=True):
        rows = B.all_gather_small(np.array([v, float(gidx), float(extra)]))
        ok = [r for r in rows if r[1] >= 0]
        if not ok:
            return None
        key = (lambda r: (-r[0], r[1])) if want_max else (lambda r: (r[0], r[1]))
        return min(ok, key=key)

    def run(R0):
        objs, conv, R = [], False, R0
        lab = None
        empties_left = 0
        for _ in range(max_iter):
            R_used = R
            lab, margin = B.disc_score(qt, R)
            sizes = B.all_reduce(B.disc_counts(lab, k).astype(np.float64)).astype(np.int64)
            for c in np.flatnonzero(sizes == 0):            # _reseed_empty_columns
                if k < 2:
                    break
                v, li, old = B.disc_best_movable(lab, margin, sizes)
                best = gather_best(v, plan.r0 + li if li >= 0 else -1, old)
                if best is None:
                    break
                g, old = int(best[1]), int(best[2])
                if plan.r0 <= g < plan.r1:
                    B.disc_set_label(lab, g - plan.r0, int(c))
                sizes[old] -= 1
                sizes[c] += 1
            S, cnt = B.disc_cluster_sums(qt, lab, k)
            M = np.divide(S, cnt[:, None], out=np.zeros_like(S), where=cnt[:, None] > 0)
            try:
                u, omega, vh = np.linalg.svd(M)
            except np.linalg.LinAlgError:
                import scipy.linalg
                u, omega, vh = scipy.linalg.svd(M, lapack_driver="gesvd")
            objs.append(n - 2.0 * float(omega.sum()))
            empties_left = int((cnt == 0).sum())
            if len(objs) >= 2 and abs(objs[-1] - objs[-2]) < tol:
                conv = True
                break
            R = vh.T @ u.T
        return objs, conv, R_used, lab, empties_left

    def prototype():
        R = np.zeros((k, k))
        R[:, 0] = B.all_reduce(B.disc_row(qt, 0) if plan.r0 == 0 < plan.r1 else np.zeros(k))
        B.disc_proto_reset(qt)
        for j in range(1, k):
            v, li = B.disc_proto_pass(qt, R[:, j - 1])
            best = gather_best(v, plan.r0 + li if li >= 0 else -1, want_max=False)
            g = int(best[1])
            R[:, j] = B.all_reduce(B.disc_row(qt, g - plan.r0) if plan.r0 <= g < plan.r1
                                   else np.zeros(k))
        return R

    r0_res = run(np.eye(k))
    r1_res = run(prototype())
    win = 1 if r1_res[0][-1] < r0_res[0][-1] - 1e-15 else 0
    res = (r0_res, r1_res)[win]
    return B.disc_labels_host(res[3]), res[4]


def _centers(deg: np.ndarray, k: int) -> np.ndarray:
    n = deg.size
    nz = int((deg > 0).sum())
    order = np.lexsort((np.arange(n), -deg))
    if k > nz:
        warnings.warn(f"only {nz} nodes have nonzero degree; filling {k - nz} center(s) in index order")
        chosen = order[:nz]
        mask = np.zeros(n, dtype=bool)
        mask[chosen] = True
        rest = np.flatnonzero(~mask)[: k - nz]
        return np.sort(np.concatenate([chosen, rest]).astype(np.int64))
    return np.sort(order[:k]).astype(np.int64)


@dataclass
class DistResult:
    labels: np.ndarray
    mhc: float
    iterations: int
    stop_reason: str
    history: list
    converged: bool
    error: str | None = None


def run_ancka_dist(net: AttributedNetwork, params: ClusterParams, B, early_stop: bool = True) -> DistResult:
    """run_ancka (engine.py:343-437) row-partitioned over the backend's ranks."""
    rank, world = B.rank, B.world
    net, _ = validate_network(net)
    if net.kind is NetworkKind.MULTIPLEX:
        raise NetworkError("the row-partitioned path covers graphs and hypergraphs")
    params.validate_for(net.n)
    n, k = net.n, params.k
    K = params.knn_k if params.knn_k is not None else default_knn_k(net.kind, n)
    K = min(K, n - 1)
    fac = HostFactors(net)
    plan = make_plan(fac, K, rank, world)

    # ---- KNN: query-stationary key ring, all-gather of the lists, replicated P_K
    ids_loc, sc_loc = knn_ring(B, net.attributes, K, plan)
    ids = B.all_gather_rows(ids_loc, plan.row_counts())
    scores = B.all_gather_rows(sc_loc, plan.row_counts())
    pk_rows, zero_rows = B.knn_graph_rows(ids, scores, n, plan.r0, plan.r1)

    # beta_vector / self-loops (walk.py:47-57, 121-123)
    deg = fac.degrees
    beta = np.full(n, float(params.beta))
    beta[deg == 0] = 1.0
    beta[zero_rows] = 0.0
    selfloop = (deg == 0) & (beta == 0.0)
    op = DistOperator(B, fac, plan, pk_rows, beta, selfloop, params.alpha, params.gamma)

    # ---- greedy init (engine.py:87-127): T_i transposed restart walks
    centers = _centers(deg, k)
    center_of = np.full(n, -1, dtype=np.int32)
    center_of[centers] = np.arange(k, dtype=np.int32)
    tag_loc = B.ivec(center_of[plan.r0:plan.r1])
    tagval = B.vec(np.full(k, params.alpha))
    P_loc = B.tagged(tag_loc, tagval, k, "f64")
    for _ in range(params.t_i):
        P_full = B.all_gather_rows(P_loc, plan.row_counts())
        P_loc = op.apply_t(P_full, k, tag_loc, tagval, 1.0 - params.alpha)
    lab0 = B.to_host_i(B.all_gather_rows(B.argmax_rows(P_loc, k), plan.row_counts()))
    if (np.bincount(lab0, minlength=k) == 0).any():
        warnings.warn("greedy init left empty cluster(s); pinning centers")
        lab0 = lab0.copy()
        lab0[centers] = np.arange(k)

    def mhc(labels: np.ndarray, dtype: str) -> float:
        """calc_mhc (engine.py:291-299), row-partitioned."""
        sizes = np.bincount(labels, minlength=k)
        if (sizes == 0).any():
            raise NetworkError("empty cluster: normalization undefined")
        yhat = 1.0 / np.sqrt(sizes.astype(np.float64))
        tag = B.ivec(labels[plan.r0:plan.r1].astype(np.int32))
        tv = B.vec(params.alpha * yhat)
        F_loc = B.tagged(tag, tv, k, dtype)
        for _ in range(params.gamma):
            F_full = B.all_gather_rows(F_loc, plan.row_counts())
            F_loc = op.apply(F_full, k, dtype, tag, tv, 1.0 - params.alpha)
        tr = B.all_reduce(np.array([B.trace_labels(F_loc, labels[plan.r0:plan.r1], yhat)]))[0]
        return 1.0 - tr / k

    rng = np.random.default_rng(params.seed)
    c = min(k + 1, n)
    sizes0 = np.bincount(lab0, minlength=k)
    q0 = np.zeros((n, c))
    q0[:, 0] = 1.0 / np.sqrt(n)
    keep = lab0 + 1 < c
    q0[np.flatnonzero(keep), lab0[keep] + 1] = 1.0 / np.sqrt(sizes0[lab0[keep]])
    best_phi = mhc(lab0, "f64")
    best = lab0.copy()
    hist = [(0, best_phi)]

    # ---- t = 1: exact f64 step, replicated on the gathered Z^(1)
    Z1 = op.apply(B.rows_from_host(q0, "f64"), c, "f64")
    Z1_full = B.to_host(B.all_gather_rows(Z1, plan.row_counts()))[:, :c]
    q1 = B.exact_qr_step(Z1_full, rng)
    Q_loc = B.rows_from_host(q1[plan.r0:plan.r1], "f32")
    dq = float(np.linalg.norm(q1 - q0))
    stop, converged, t, err = "max_iterations", False, 1, None
    try:
        t = 1
        while True:
            if t % params.tau == 0:
                lab_loc, empties = discretize_dist(B, Q_loc, k, plan)
                if empties > 0:
                    raise NetworkError("cannot repair empty clusters: no movable nodes")
                labels = B.all_gather_labels(lab_loc, plan.row_counts())
                phi = mhc(labels, "f32")
                hist.append((t, phi))
                if phi < best_phi:
                    best_phi, best = phi, labels.copy()
                if dq < params.eps_q:
                    stop, converged = "subspace_converged", True
                    break
                if early_stop and len(hist) >= 3 and hist[-3][1] < hist[-2][1] < hist[-1][1]:
                    stop, converged = "mhc_rising", True
                    break
            if t >= params.t_a:
                break
            # one f32 orthogonal step (engine.py:130-149), row-partitioned
            Q_full = B.all_gather_rows(Q_loc, plan.row_counts())
            Z_loc = op.apply(Q_full, c, "f32")
            G = B.all_reduce(B.gram(Z_loc, c))
            Q_loc, dq2_loc = B.cholqr_apply(Z_loc, Q_loc, G, c)
            dq = float(np.sqrt(B.all_reduce(np.array([dq2_loc]))[0]))
            t += 1
    except NetworkError as exc:
        err, stop = str(exc), "error"
    return DistResult(best, best_phi, t, stop, hist, converged, err)


# ----------------------------------------------------------------------------
class CudaBackend:
    """libancka_b200 kernels + NCCL collectives (one rank per GPU)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib
        self.torch, self.dist, self._lib, self.group = torch, dist, _lib, group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        _lib.require_device()

    # --- data
    def _t(self, a, dtype):
        return self.torch.as_tensor(a, dtype=dtype).to("cuda")

    def vec(self, a):
        return self._t(np.asarray(a, dtype=np.float64), self.torch.float64)

    def ivec(self, a):
        return self._t(np.asarray(a, dtype=np.int32), self.torch.int32)

    def mask(self, a):
        return self._t(np.asarray(a, dtype=np.uint8), self.torch.uint8)

    def csr(self, m):
        from ._device import DeviceCSR
        return DeviceCSR.from_scipy(sp.csr_matrix(m))

    def _ld(self, c, dtype):
        from ._device import ld_for
        return ld_for(c, self.torch.float32 if dtype == "f32" else self.torch.float64)

    def rows_from_host(self, a, dtype):
        from ._device import padded
        return padded(self.torch.from_numpy(np.ascontiguousarray(a)),
                      self.torch.float32 if dtype == "f32" else self.torch.float64)

    def to_host(self, a):
        return a.double().cpu().numpy()

    def to_host_i(self, a):
        return a.cpu().numpy().astype(np.int64)

    def tagged(self, tag, tagval, c, dtype):
        torch = self.torch
        dt = torch.float32 if dtype == "f32" else torch.float64
        out = torch.zeros((tag.numel(), self._ld(c, dtype)), dtype=dt, device="cuda")
        rows = torch.nonzero(tag >= 0).flatten()
        out[rows, tag[rows].long()] = tagval[tag[rows].long()].to(dt)
        return out

    # --- collectives
    def all_gather_rows(self, x, counts):
        torch = self.torch
        if self.world == 1:
            return x
        mx = int(np.max(counts))
        buf = torch.zeros((mx,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        buf[: x.shape[0]] = x
        if self.dist.get_backend(self.group) == "nccl":
            out = torch.empty((self.world * mx,) + tuple(x.shape[1:]), dtype=x.dtype,
                              device=x.device)
            self.dist.all_gather_into_tensor(out, buf, group=self.group)
            parts = [out[r * mx: r * mx + int(counts[r])] for r in range(self.world)]
        else:   # gloo (tests): list form
            lst = [torch.empty_like(buf) for _ in range(self.world)]
            self.dist.all_gather(lst, buf, group=self.group)
            parts = [lst[r][: int(counts[r])] for r in range(self.world)]
        return torch.cat(parts, dim=0)

    def all_reduce(self, a):
        torch = self.torch
        t = torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    # --- kernels
    # --- KNN key ring: shards are ("csr", indptr, indices, data, d) or ("dense", X)
    def x_shard(self, X, r0, r1):
        torch = self.torch
        if sp.issparse(X):
            x = sp.csr_matrix(X)[r0:r1]
            return ("csr", torch.from_numpy(x.indptr.astype(np.int64)).cuda(),
                    torch.from_numpy(x.indices.astype(np.int32)).cuda(),
                    torch.from_numpy(x.data.astype(np.float64)).cuda(), X.shape[1])
        return ("dense", torch.from_numpy(np.ascontiguousarray(X[r0:r1], dtype=np.float64)).cuda())

    def _concat(self, a, b):
        torch = self.torch
        if b is None:
            return a
        if a[0] == "csr":
            ip = torch.cat([a[1], b[1][1:] + a[1][-1]])
            return ("csr", ip, torch.cat([a[2], b[2]]), torch.cat([a[3], b[3]]), a[4])
        return ("dense", torch.cat([a[1], b[1]]))

    def knn_local(self, mine, block, K, r0, boff):
        """Top-K of the own rows over (own rows + block), global indices.  The
        two shards are concatenated in global row order, so the kernel's
        index tie-break is the global one."""
        from .knn import DeviceAttributes, knn_search_exact_device
        torch = self.torch
        rows_of = (lambda t: int(t[1].numel() - 1)) if mine[0] == "csr" else (lambda t: int(t[1].shape[0]))
        nq = rows_of(mine)
        first = block is not None and boff < r0
        x = self._concat(block, mine) if first else self._concat(mine, block)
        nb = rows_of(block) if first else 0
        if x[0] == "csr":
            xa = DeviceAttributes.from_device_csr(x[1], x[2], x[3], (int(x[1].numel() - 1), x[4]))
        else:
            xa = DeviceAttributes.from_device_dense(x[1])
        kk = min(K, xa.shape[0] - 1)
        ids, sc = knn_search_exact_device(xa, kk, rows=(nb, nb + nq))
        ids = ids.long()
        if first:
            g = torch.where(ids < nb, ids + boff, ids - nb + r0)
        else:
            g = torch.where(ids < nq, ids + r0, ids - nq + boff)
        g = torch.where(ids < 0, torch.full_like(ids, -1), g)
        if kk < K:
            pad = K - kk
            g = torch.cat([g, torch.full((nq, pad), -1, dtype=g.dtype, device=g.device)], 1)
            sc = torch.cat([sc, torch.zeros((nq, pad), dtype=sc.dtype, device=sc.device)], 1)
        return g, sc

    def merge_lists(self, ia, sa, ib, sb, K):
        """Per row: union, dedup, order (score desc, index asc), first K."""
        torch = self.torch
        ids = torch.cat([ia, ib], 1)
        sc = torch.cat([sa, sb], 1)
        big = torch.iinfo(torch.int64).max
        key_i = torch.where(ids < 0, torch.full_like(ids, big), ids)
        o = torch.argsort(key_i, dim=1, stable=True)               # index asc
        ids, sc, key_i = ids.gather(1, o), sc.gather(1, o), key_i.gather(1, o)
        dup = torch.zeros_like(ids, dtype=torch.bool)
        dup[:, 1:] = (key_i[:, 1:] == key_i[:, :-1]) & (ids[:, 1:] >= 0)
        s_key = torch.where((ids < 0) | dup, torch.full_like(sc, -np.inf), sc)
        o = torch.argsort(-s_key, dim=1, stable=True)               # score desc, ties keep index asc
        ids, s_key = ids.gather(1, o)[:, :K], s_key.gather(1, o)[:, :K]
        ok = s_key > -np.inf
        return torch.where(ok, ids, torch.full_like(ids, -1)), torch.where(ok, s_key, torch.zeros_like(s_key))

    def _p2p(self, send_tensors, recv_tensors):
        """Send to rank+1 and receive from rank-1.  NCCL moves device tensors
        over NVLink; other backends (gloo in the tests) go through host copies."""
        dist = self.dist
        nxt, prv = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        if dist.get_backend(self.group) != "nccl":
            host_recv = [t.cpu() for t in recv_tensors]
            ops = [dist.P2POp(dist.isend, t.cpu(), nxt, group=self.group) for t in send_tensors]
            ops += [dist.P2POp(dist.irecv, t, prv, group=self.group) for t in host_recv]
            reqs = dist.batch_isend_irecv(ops)
            for r in reqs:
                r.wait()
            for dst, src in zip(recv_tensors, host_recv):
                dst.copy_(src)
            return []
        ops = [dist.P2POp(dist.isend, t, nxt, group=self.group) for t in send_tensors]
        ops += [dist.P2POp(dist.irecv, t, prv, group=self.group) for t in recv_tensors]
        return dist.batch_isend_irecv(ops)

    def ring_start(self, block):
        torch = self.torch
        arrays = list(block[1:4]) if block[0] == "csr" else [block[1]]
        hdr = torch.tensor([a.numel() for a in arrays] + ([block[4]] if block[0] == "csr"
                                                          else list(block[1].shape)),
                           dtype=torch.int64, device="cuda")
        rh = torch.empty_like(hdr)
        for r in self._p2p([hdr], [rh]):
            r.wait()
        sizes = rh.cpu().tolist()
        if block[0] == "csr":
            bufs = [torch.empty(sizes[0], dtype=torch.int64, device="cuda"),
                    torch.empty(sizes[1], dtype=torch.int32, device="cuda"),
                    torch.empty(sizes[2], dtype=torch.float64, device="cuda")]
            meta = ("csr", sizes[3])
        else:
            bufs = [torch.empty((sizes[1], sizes[2]), dtype=torch.float64, device="cuda")]
            meta = ("dense",)
        reqs = self._p2p(arrays, bufs)
        return reqs, bufs, meta

    def ring_finish(self, pending):
        reqs, bufs, meta = pending
        for r in reqs:
            r.wait()
        return ("csr", bufs[0], bufs[1], bufs[2], meta[1]) if meta[0] == "csr" else ("dense", bufs[0])

    def knn_graph_rows(self, ids, scores, n, r0, r1):
        from ._device import DeviceCSR
        from .knn import build_knn_graph_device
        A, P, zero = build_knn_graph_device(ids.int(), scores, n)
        rp = P.rowptr[r0: r1 + 1]
        b, e = int(rp[0]), int(rp[-1])
        loc = DeviceCSR(r1 - r0, n, (rp - b).contiguous(), P.colidx[b:e], P.val64[b:e], P.val32[b:e])
        return loc, zero.cpu().numpy().astype(bool)

    def spmm(self, S, s_src, Kc, k_src, beta, selfloop, self_src, row_offset, tag, tagval, scale,
             c, dtype):
        torch, _lib = self.torch, self._lib
        f64 = dtype == "f64"
        dt = torch.float64 if f64 else torch.float32
        rows = S.rows
        out = torch.empty((rows, self._ld(c, dtype)), dtype=dt, device="cuda")
        code = _lib.F64 if f64 else _lib.F32

        def cast(x):
            return None if x is None else (x if x.dtype == dt else x.to(dt))
        s_src, k_src, self_src = cast(s_src), cast(k_src), cast(self_src)
        beta_t, tagval_t = cast(beta), cast(tagval)
        import ctypes
        Sst = S.struct(code)
        Kst = Kc.struct(code) if Kc is not None else None
        _lib.call("ancka_spmm2", code, rows, c, ctypes.byref(Sst), s_src.data_ptr(),
                  s_src.stride(0), ctypes.byref(Kst) if Kst is not None else None,
                  k_src.data_ptr() if k_src is not None else None,
                  k_src.stride(0) if k_src is not None else 0,
                  beta_t.data_ptr() if beta_t is not None else None,
                  selfloop.data_ptr() if selfloop is not None else None,
                  self_src.data_ptr() if self_src is not None else None,
                  self_src.stride(0) if self_src is not None else 0, row_offset,
                  tag.data_ptr() if tag is not None else None,
                  tagval_t.data_ptr() if tagval_t is not None else None, float(scale),
                  out.data_ptr(), out.stride(0), _lib.stream())
        return out

    def gram(self, Z, c):
        from ._device import WORKSPACE
        torch, _lib = self.torch, self._lib
        G = torch.empty(c * (c + 1) // 2, dtype=torch.float64, device="cuda")
        ws = WORKSPACE.get("dist_orth", _lib.load().ancka_orth_workspace_size(None, c))
        _lib.call("ancka_gram_f32", Z.data_ptr(), Z.shape[0], Z.stride(0), c, G.data_ptr(),
                  ws.data_ptr(), ws.numel(), _lib.stream())
        return G.cpu().numpy()

    def cholqr_apply(self, Z, Qprev, G, c):
        from ._device import WORKSPACE
        torch, _lib = self.torch, self._lib
        Gt = torch.as_tensor(G, device="cuda")
        Qn = torch.empty_like(Z)
        stats = torch.tensor([0.0, 1.0, 0.0, 0.0], dtype=torch.float64, device="cuda")
        ws = WORKSPACE.get("dist_orth", _lib.load().ancka_orth_workspace_size(None, c))
        _lib.call("ancka_cholqr_apply_f32", Z.data_ptr(), Qprev.data_ptr(), Qn.data_ptr(),
                  Z.shape[0], Z.stride(0), c, Gt.data_ptr(), stats.data_ptr(), ws.data_ptr(),
                  ws.numel(), _lib.stream())
        return Qn, float(stats[0].item())

    def argmax_rows(self, P, k):
        return self.torch.argmax(P[:, :k], dim=1).int()

    def trace_labels(self, F, labels_loc, yhat):
        torch = self.torch
        lab = torch.as_tensor(labels_loc, device="cuda").long()
        vals = F[torch.arange(F.shape[0], device="cuda"), lab].double()
        return float((vals * torch.as_tensor(yhat, device="cuda")[lab]).sum().item())

    def exact_qr_step(self, Z_full, rng):
        from ._device import padded
        from .engine import _qr_f64_inplace
        torch = self.torch
        c = Z_full.shape[1]
        z = padded(torch.from_numpy(Z_full), torch.float64)
        q = z.clone()
        d = _qr_f64_inplace(q, c)
        bad = d < 1e-12 * max(1.0, d.max() if d.size else 1.0)
        if bad.any():
            warnings.warn(f"rank-deficient iterate; perturbing {int(bad.sum())} column(s)")
            noise = rng.standard_normal((Z_full.shape[0], int(bad.sum())))
            cols = torch.from_numpy(np.flatnonzero(bad)).to("cuda")
            z[:, cols] += 1e-8 * torch.from_numpy(noise).to("cuda")
            q = z.clone()
            _qr_f64_inplace(q, c)
        return q[:, :c].cpu().numpy()

    # --- row-partitioned discretisation primitives (discretize_dist)
    def disc_prepare(self, Q_loc, col0, k):
        torch, _lib = self.torch, self._lib
        from ._device import ld_for
        n = Q_loc.shape[0]
        ldt = ld_for(k, torch.float32)
        st = {"k": k, "ldt": ldt, "n": n,
              "qt": torch.empty((n, ldt), dtype=torch.float32, device="cuda"),
              "zero": torch.zeros(1, dtype=torch.int32, device="cuda"),
              "R": torch.zeros((k, ldt), dtype=torch.float32, device="cuda"),
              "acc": torch.zeros(max(n, 1), dtype=torch.float64, device="cuda"),
              "rcol": torch.zeros(k, dtype=torch.float64, device="cuda"),
              "S": torch.empty(k * k, dtype=torch.int64, device="cuda"),
              "cnt": torch.empty(k, dtype=torch.int64, device="cuda")}
        bits = int(np.ceil(np.log2(max(self.all_reduce(np.array([float(n)]))[0], 1) + 1)))
        st["scale"] = float(2.0 ** (61 - bits))
        if n:
            _lib.call("ancka_disc_normalize", Q_loc.data_ptr(), Q_loc.stride(0), col0, n, k,
                      st["qt"].data_ptr(), ldt, st["zero"].data_ptr(), _lib.stream())
        return st

    def disc_score(self, st, R):
        torch, _lib = self.torch, self._lib
        k, n = st["k"], st["n"]
        st["R"][:, :k] = torch.from_numpy(R.astype(np.float32)).cuda()
        lab = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
        margin = torch.zeros(max(n, 1), dtype=torch.float32, device="cuda")
        if n:
            _lib.call("ancka_disc_score", st["qt"].data_ptr(), st["ldt"], n, k, st["R"].data_ptr(),
                      st["ldt"], lab.data_ptr(), margin.data_ptr(), _lib.stream())
        return lab[:n], margin[:n]

    def disc_counts(self, lab, k):
        return self.torch.bincount(lab.long(), minlength=k).cpu().numpy()

    def disc_best_movable(self, lab, margin, sizes):
        torch = self.torch
        if lab.numel() == 0:
            return -np.inf, -1, 0
        sz = torch.from_numpy(sizes).cuda()
        movable = sz[lab.long()] >= 2
        if not bool(movable.any()):
            return -np.inf, -1, 0
        cand = torch.where(movable, margin.double(), torch.full_like(margin, -np.inf).double())
        i = int(torch.argmax(cand))                      # first maximum
        return float(cand[i]), i, int(lab[i])

    def disc_set_label(self, lab, i, c):
        lab[i] = c

    def disc_cluster_sums(self, st, lab, k):
        torch, _lib = self.torch, self._lib
        n = st["n"]
        if n:
            _lib.call("ancka_disc_accumulate", st["qt"].data_ptr(), st["ldt"], n, k, lab.data_ptr(),
                      st["scale"], st["S"].data_ptr(), st["cnt"].data_ptr(), _lib.stream())
        else:
            st["S"].zero_()
            st["cnt"].zero_()
        both = torch.cat([st["S"], st["cnt"]])
        if self.world > 1:                               # int64 sums: exact, order free
            self.dist.all_reduce(both, group=self.group)
        h = both.cpu().numpy()
        return h[:k * k].reshape(k, k).astype(np.float64) / st["scale"], h[k * k:].astype(np.float64)

    def disc_proto_reset(self, st):
        st["acc"].zero_()

    def disc_proto_pass(self, st, rcol):
        torch, _lib = self.torch, self._lib
        n, k = st["n"], st["k"]
        if n == 0:
            return np.inf, -1
        st["rcol"].copy_(torch.from_numpy(rcol))
        _lib.call("ancka_disc_proto_pass", st["qt"].data_ptr(), st["ldt"], n, k,
                  st["rcol"].data_ptr(), st["acc"].data_ptr(), _lib.stream())
        i = int(torch.argmin(st["acc"][:n]))             # first minimum
        return float(st["acc"][i]), i

    def disc_row(self, st, i):
        return st["qt"][i, :st["k"]].double().cpu().numpy()

    def disc_labels_host(self, lab):
        return lab.cpu().numpy().astype(np.int64)

    def all_gather_small(self, a):
        torch = self.torch
        t = torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")
        if self.world == 1:
            return [t.cpu().numpy()]
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    def all_gather_labels(self, lab_loc, counts):
        t = self.torch.as_tensor(lab_loc.astype(np.float64), device="cuda")[:, None]
        return self.all_gather_rows(t, counts)[:, 0].cpu().numpy().astype(np.int64)
