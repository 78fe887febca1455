"""Row-partitioned multi-GPU ANCKA.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank r
owns a contiguous block of node rows [r0, r1) (balanced by operator
nonzeros) and, for hypergraphs, a block of hyperedges [e0, e1).  No rank
materialises a whole-graph factor, the whole KNN graph or a whole f64 block:

* factors   each rank normalises only its rows (ShardFactors): P_N / P_V rows
            [r0, r1), P_E rows [e0, e1), and the transposed factors of the
            init walk as column-scaled local slices (P_N^T rows = A rows * D^-1
            for the symmetrised A; P_V^T rows = H rows * D_V^-1; P_E^T rows =
            H^T rows * D_E^-1) -- walk.py:38-79, 153-174 restricted to rows.
* KNN       query-stationary key ring (knn.py:112-140): own rows x own rows
            once, then own rows x each visiting shard only (the kernels take a
            key-row range), the lists merged per row on the device by
            (score desc, id asc) with de-duplication.  The shards travel
            around the ring (P2P send/recv, the next transfer posted before
            the kernel runs).
* KNN graph A_K = M + M^T by rows (knn.py:294-324): every list entry (i, j, s)
            is kept as (i, j, s) by owner(i) and sent as (j, i, s) to owner(j)
            in one all-to-all; each rank sums duplicates and row-normalises
            its rows on the device (same sums as the single-GPU kernel).
* init      T_i restart walks (engine.py:87-127) over column chunks of the
            centres (f64, each chunk n x <= 32 gathered per step), with a
            running first-max argmax on the device.
* step 1    (rank deficient) f64 apply of Q^(0) -- rebuilt on
            every rank from the labels, in column chunks -- then CGS2 over
            the local rows with all-reduced column dots, the reference's rank
            test on |R_jj| and its replicated seeded noise (engine.py:130-149).
* loop      per f32 step: all-gather of Q (n x c), local rows of Z, local Gram
            all-reduced on the device, every rank factors the same Gram and
            applies R^-1 to its rows; ||dQ||^2 and the suspect-pivot count stay
            on the device until the tau sample (one small read-back).  A
            suspect pivot in a tau-block replays the block with exact f64
            steps, as the single-GPU engine does.
* MHC       gamma all-gathers plus an all-reduced trace (engine.py:291-299).
* discretisation is row-partitioned: argmax and cluster sums local, the
            k x k sums all-reduced (exact 64-bit fixed point), the k x k SVD
            replicated (engine.py:183-263).

The orchestration is backend-generic: `CudaBackend` drives libancka_b200
kernels and NCCL; the CPU tests drive the same code with a numpy backend over
gloo (tests/test_dist.py), which is how the N>1 logic is verified without
several GPUs.
"""
from __future__ import annotations

import os
import warnings
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .network import (AttributedNetwork, ClusterParams, NetworkError, NetworkKind,
                      default_knn_k, symmetrize_union, validate_network)

#: centre columns per chunk of the init walk / step-1 apply (bounds the f64
#: n x chunk block each rank holds: Papers100M 111M x 32 x 8 B = 28 GB)
INIT_CHUNK = 32
#: f64 bytes of one gathered n x chunk block allowed before chunking at INIT_CHUNK
INIT_CHUNK_BYTES = 4 << 30


def _f64_chunk(n: int, cols: int) -> int:
    """Columns per f64 walk / step-1 chunk: all of them when the gathered
    n x cols f64 block fits INIT_CHUNK_BYTES, else INIT_CHUNK."""
    return cols if n * cols * 8 <= INIT_CHUNK_BYTES else INIT_CHUNK


# ----------------------------------------------------------------------------
def partition_rows(cost: np.ndarray, world: int) -> np.ndarray:
    """Contiguous row blocks with ~equal total cost: boundaries[world + 1]."""
    n = cost.size
    c = np.concatenate([[0.0], np.cumsum(cost, dtype=np.float64)])
    targets = c[-1] * np.arange(1, world) / world
    cuts = np.searchsorted(c, targets, side="left")
    b = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    return np.maximum.accumulate(np.clip(b, 0, n))


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


def _binary(m: sp.csr_matrix) -> sp.csr_matrix:
    m = sp.csr_matrix(m)
    m.sort_indices()
    return m


class ShardFactors:
    """The validated structure with the global per-node / per-edge degree
    vectors (O(n + m)), from which each rank cuts its row slices.  The full
    normalised factors and their transposes are never formed."""

    def __init__(self, net: AttributedNetwork, degrees: np.ndarray):
        self.kind = net.kind
        self.n = net.n
        self.degrees = np.asarray(degrees, dtype=np.float64)
        if net.kind is NetworkKind.HYPERGRAPH:
            self.h = _binary(net.incidence)                   # m x n
            self.m = self.h.shape[0]
            # reference row sums of H^T (node degrees) and of H (edge sizes)
            self.dv = np.asarray(self.h.sum(axis=0)).ravel()
            self.de = np.asarray(self.h.sum(axis=1)).ravel()
            self.row_nnz = np.bincount(self.h.indices, minlength=self.n).astype(np.float64)
        else:
            a = symmetrize_union(net.adjacency) if net.directed else net.adjacency
            self.a = _binary(a)
            self.m = 0
            self.da = np.asarray(self.a.sum(axis=1)).ravel()
            self.row_nnz = np.diff(self.a.indptr).astype(np.float64)

    def row_cost(self, K: int) -> np.ndarray:
        return self.row_nnz + 2 * K + 1

    def edge_cost(self) -> np.ndarray:
        return np.diff(self.h.indptr).astype(np.float64) + 1


def _raw_row_cost(net: AttributedNetwork, K: int) -> np.ndarray:
    """Row costs from the unvalidated input's pattern (degrees + 2K + 1)."""
    if net.kind is NetworkKind.HYPERGRAPH:
        deg = np.bincount(net.incidence.indices, minlength=net.n)
    else:
        a = net.adjacency
        deg = np.diff(a.indptr)
        if net.directed:
            deg = deg + np.bincount(a.indices, minlength=net.n)
    return deg.astype(np.float64) + 2 * K + 1


def make_plan(fac: ShardFactors, K: int, rank: int, world: int) -> Plan:
    rows = partition_rows(fac.row_cost(K), world)
    if fac.kind is NetworkKind.HYPERGRAPH:
        edges = partition_rows(fac.edge_cost(), world)
    else:
        edges = np.zeros(world + 1, dtype=np.int64)
    return Plan(rank, world, fac.n, fac.m, rows, edges)


def _inv(v: np.ndarray) -> np.ndarray:
    return np.divide(1.0, v, out=np.zeros_like(v, dtype=np.float64), where=v != 0)


# ----------------------------------------------------------------------------
class DistOperator:
    """A rank's share of the joint-walk operator (row slices, backend handles)."""

    def __init__(self, B, fac: ShardFactors, plan: Plan, p_k_rows, beta_loc: np.ndarray,
                 selfloop_loc: np.ndarray, alpha: float, gamma: int):
        self.B, self.plan, self.kind = B, plan, fac.kind
        self.alpha, self.gamma = alpha, gamma
        r0, r1 = plan.r0, plan.r1
        if fac.kind is NetworkKind.HYPERGRAPH:
            hloc = fac.h[plan.e0:plan.e1]                     # m_loc x n
            htl = sp.csr_matrix(fac.h[:, r0:r1].T)            # H^T rows: n_loc x m
            htl.sort_indices()
            self.S = B.csr_rownorm(htl)                       # P_V rows: n_loc x m, gathers T
            self.E = B.csr_rownorm(hloc)                      # P_E rows: m_loc x n, gathers Q
            self.TA = B.csr_colscale(hloc, _inv(fac.dv))      # P_V^T rows: m_loc x n
            self.TB = B.csr_colscale(htl, _inv(fac.de))       # P_E^T rows: n_loc x m
        else:
            aloc = fac.a[r0:r1]
            self.S = B.csr_rownorm(aloc)                      # P_N rows
            self.TA = B.csr_colscale(aloc, _inv(fac.da))      # P_N^T rows (A symmetric)
        self.K = p_k_rows
        self.beta = B.vec(beta_loc)
        self.selfloop = B.mask(selfloop_loc)
        self.order = None     # f32 row order (locality), refreshed at every sample

    def set_order(self, labels_loc, k):
        if hasattr(self.B, "locality_order"):
            self.order = self.B.locality_order(labels_loc, k)

    # -- joint apply (walk.py:177-190) on the local rows; Q_full gathered
    def apply(self, Q_full, c, dtype, tag=None, tagval=None, scale=1.0):
        B, pl = self.B, self.plan
        if self.kind is NetworkKind.HYPERGRAPH:
            T_loc = B.spmm(self.E, Q_full, None, None, None, None, None, 0, None, None, 1.0, c, dtype)
            src = B.all_gather_rows(T_loc, pl.edge_counts())
        else:
            src = Q_full
        if self.order is not None and dtype == "f32":
            return B.spmm(self.S, src, self.K, Q_full, self.beta, self.selfloop, Q_full, pl.r0,
                          tag, tagval, scale, c, dtype, order=self.order)
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
    """Exact top-K of rows [r0, r1) against all n keys with only the own shard
    and one visiting shard of X resident (SURVEY.md §8(e) KNN ring): own x own
    once, then own x visiting per step; every key is ranked against the own
    rows exactly once, and the per-row merge by (score desc, id asc) keeps the
    global top-K (knn.py:83-98)."""
    rank, world = plan.rank, plan.world
    r0, r1 = plan.r0, plan.r1
    mine = B.x_shard(X, r0, r1)
    level = B.knn_level(mine)
    ids, sc = B.knn_own(mine, K, r0, level)
    block, src = mine, rank
    pending = B.ring_start(block) if world > 1 else None
    for step in range(1, world):
        block, src = B.ring_finish(pending), (src - 1) % world
        pending = B.ring_start(block) if step < world - 1 else None   # overlaps the kernel
        if B.shard_rows(block) == 0 or r1 == r0:
            continue
        i2, s2 = B.knn_cross(mine, block, K, r0, int(plan.rows[src]), level)
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
            S, cnt = B.disc_cluster_sums(qt, lab, k)
            sizes = cnt.astype(np.int64)
            if (sizes == 0).any() and k >= 2:
                for c in np.flatnonzero(sizes == 0):            # _reseed_empty_columns
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


# ANCKA_DW_* ops of ancka_discw_dist_op (include/ancka_b200.h)
(DW_START, DW_ROUND_LOCAL, DW_SNAP, DW_CHECK_EMPTY, DW_POLAR, DW_CLEAR_PAUSE, DW_MARGINS,
 DW_MOVE_ROW, DW_PROTO_PASS, DW_PROTO_PICK, DW_PROTO_SETCOL, DW_FLAGS, DW_FINISH,
 DW_RESEED_CAND) = range(14)

#: discretisation mode of the row-partitioned path: "auto" replicates the
#: device discretisation on every rank (the gathered n x c f32 block, the
#: single-GPU kernels, no host round trips) when that block is at most
#: DISC_REPLICATED_BYTES, else runs the device row-partitioned rounds
#: (`CudaBackend.disc_partitioned`, 8 < k <= 192) or the host rounds
#: (`discretize_dist`); "replicated" / "partitioned" / "host" force one
DISC_MODE = "auto"
DISC_REPLICATED_BYTES = 16 << 30


def _replicated_disc(B, n: int, c: int) -> bool:
    if not hasattr(B, "disc_replicated") or DISC_MODE in ("partitioned", "host"):
        return False
    return DISC_MODE == "replicated" or n * ((c + 3) // 4 * 4) * 4 <= DISC_REPLICATED_BYTES


def _device_partitioned_disc(B, k: int, plan) -> bool:
    """The device row-partitioned rounds cover 8 < k <= 192 with every rank
    holding rows; otherwise (and with DISC_MODE "host") the host rounds."""
    return (hasattr(B, "disc_partitioned") and DISC_MODE != "host" and 8 < k <= 192
            and int(np.min(plan.row_counts())) >= 1)


def _centers(deg: np.ndarray, k: int) -> np.ndarray:
    """Top-k degree nodes, ties to the smaller index, sorted (engine.py:97-110)."""
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
    replays: int = 0
    timings_ms: dict | None = None


def _q0_chunk(B, labels: np.ndarray, sizes: np.ndarray, n: int, c: int, c0: int, cc: int):
    if hasattr(B, "q0_chunk"):                 # built on the device from the labels
        return B.q0_chunk(labels, sizes, n, c, c0, cc)
    return _q0_chunk_host(B, labels, sizes, n, c, c0, cc)


def _q0_chunk_host(B, labels: np.ndarray, sizes: np.ndarray, n: int, c: int, c0: int, cc: int):
    """Columns [c0, c0 + cc) of Q^(0) = [1/sqrt(n) | Yhat0] (engine.py:368-371)
    for all n rows, built from the replicated labels (no gather)."""
    q = np.zeros((n, cc))
    if c0 == 0:
        q[:, 0] = 1.0 / np.sqrt(n)
    col = labels + 1 - c0
    ok = (col >= 0) & (col < cc) & (labels + 1 < c)
    q[np.flatnonzero(ok), col[ok]] = 1.0 / np.sqrt(sizes[labels[ok]])
    return B.rows_from_host(q, "f64")


def exact_step_dist(B, op: DistOperator, plan: Plan, Q_src, c: int, rng, labels0=None,
                    sizes0=None):
    """orthogonal_step (engine.py:130-149) in f64, row-partitioned: the apply
    by column chunks (all-gathered, or rebuilt from the labels for Q^(0)),
    CGS2 over the local rows with all-reduced column dots, the reference's
    rank test on |R_jj|, its seeded noise on flagged columns (the same
    n x b draw on every rank, each adding its rows), and the re-factorisation.
    Returns (Q_loc f64, Z_loc f64)."""
    n = plan.n
    parts = []
    ch = _f64_chunk(n, c)
    for c0 in range(0, c, ch):
        cc = min(ch, c - c0)
        if Q_src is None:
            full = _q0_chunk(B, labels0, sizes0, n, c, c0, cc)
        else:
            full = B.all_gather_rows(B.cols(Q_src, c0, cc, "f64"), plan.row_counts())
        parts.append(op.apply(full, cc, "f64"))
    Z = B.hcat(parts, c)
    Q, d = B.cgs2(Z, c, B.all_reduce_vec)
    bad = d < 1e-12 * max(1.0, d.max() if d.size else 1.0)
    if bad.any():
        warnings.warn(f"rank-deficient iterate; perturbing {int(bad.sum())} column(s)")
        noise = rng.standard_normal((n, int(bad.sum())))
        Z = B.add_cols(Z, np.flatnonzero(bad), 1e-8 * noise[plan.r0:plan.r1])
        Q, _ = B.cgs2(Z, c, B.all_reduce_vec)
    return Q, Z


#: phase wall times in DistResult.timings_ms (synchronises at phase ends)
DIST_TIMING = False


class _Phases:
    def __init__(self, B, on: bool):
        import time
        self.B, self.on, self.t = B, on, {}
        self._clock = time.perf_counter
        self._t0 = self._clock() if on else 0.0

    def mark(self, key):
        if not self.on:
            return
        sync = getattr(self.B, "synchronize", None)
        if sync is not None:
            sync()
        now = self._clock()
        self.t[key] = self.t.get(key, 0.0) + (now - self._t0) * 1e3
        self._t0 = now


#: reuse the last evaluated MHC for a relabelled partition (ANCKA_MHC_REUSE=0 disables)
MHC_REUSE = os.environ.get("ANCKA_MHC_REUSE", "1") != "0"


def same_partition(a: np.ndarray, b: np.ndarray, k: int) -> bool:
    """a and b (labels in [0, k), replicated on every rank) are the same
    partition up to relabelling: k distinct (a, b) pairs and k clusters on
    each side (the k x k pair histogram; k <= 4096, else False)."""
    if k > 4096 or a.shape != b.shape:
        return False
    pairs = np.bincount(a.astype(np.int64) * k + b, minlength=k * k)
    return (int(np.count_nonzero(pairs)) == k
            and int(np.count_nonzero(pairs.reshape(k, k).sum(axis=1))) == k
            and int(np.count_nonzero(pairs.reshape(k, k).sum(axis=0))) == k)


def run_ancka_dist(net: AttributedNetwork, params: ClusterParams, B, early_stop: bool = True) -> DistResult:
    """run_ancka (engine.py:343-437) row-partitioned over the backend's ranks."""
    rank, world = B.rank, B.world
    ph = _Phases(B, DIST_TIMING)
    if net.kind is NetworkKind.MULTIPLEX:
        raise NetworkError("the row-partitioned path covers graphs and hypergraphs")
    params.validate_for(net.n)
    n, k = net.n, params.k
    K = params.knn_k if params.knn_k is not None else default_knn_k(net.kind, n)
    K = min(K, n - 1)
    # rows are balanced on the input's pattern (any split is correct), so the
    # KNN ring starts before the host validation, which then overlaps it
    # (the attributes the ring reads are not changed by validation)
    rows = partition_rows(_raw_row_cost(net, K), world)
    plan = Plan(rank, world, n, 0, rows, np.zeros(world + 1, dtype=np.int64))
    r0, r1 = plan.r0, plan.r1

    # ---- KNN: key ring, then A_K / P_K rows from an all-to-all of triples
    ids_loc, sc_loc = knn_ring(B, net.attributes, K, plan)
    net, report = validate_network(net)
    fac = ShardFactors(net, report.degrees)
    if fac.kind is NetworkKind.HYPERGRAPH:
        plan = Plan(rank, world, n, fac.m, rows, partition_rows(fac.edge_cost(), world))
    ph.mark("knn_ms")
    pk_rows, zero_loc = B.knn_graph_rows(ids_loc, sc_loc, plan, K)

    # beta_vector / self-loops (walk.py:47-57, 121-123) on the local rows
    deg = fac.degrees
    beta = np.full(r1 - r0, float(params.beta))
    beta[deg[r0:r1] == 0] = 1.0
    beta[zero_loc] = 0.0
    selfloop = (deg[r0:r1] == 0) & (beta == 0.0)
    op = DistOperator(B, fac, plan, pk_rows, beta, selfloop, params.alpha, params.gamma)
    ph.mark("graph_operator_ms")

    # ---- greedy init (engine.py:87-127): T_i transposed restart walks per
    # chunk of centres, running first-max argmax over the chunks
    centers = _centers(deg, k)
    center_of = np.full(n, -1, dtype=np.int64)
    center_of[centers] = np.arange(k)
    best_v, best_i = None, None
    ch = _f64_chunk(n, k)
    for c0 in range(0, k, ch):
        cc = min(ch, k - c0)
        loc = center_of[r0:r1] - c0
        loc = np.where((center_of[r0:r1] >= 0) & (loc >= 0) & (loc < cc), loc, -1)
        tag_loc = B.ivec(loc)
        tagval = B.vec(np.full(cc, params.alpha))
        P_loc = B.tagged(tag_loc, tagval, cc, "f64")
        for _ in range(params.t_i):
            P_full = B.all_gather_rows(P_loc, plan.row_counts())
            P_loc = op.apply_t(P_full, cc, tag_loc, tagval, 1.0 - params.alpha)
        best_v, best_i = B.argmax_update(P_loc, cc, c0, best_v, best_i)
    lab0 = B.to_host_i(B.all_gather_rows(B.as_rows(best_i), plan.row_counts()))
    if (np.bincount(lab0, minlength=k) == 0).any():
        warnings.warn("greedy init left empty cluster(s); pinning centers")
        lab0 = lab0.copy()
        lab0[centers] = np.arange(k)

    def mhc(labels: np.ndarray, dtype: str):
        """calc_mhc (engine.py:291-299), row-partitioned; the trace stays a
        backend scalar until read."""
        sizes = np.bincount(labels, minlength=k)
        if (sizes == 0).any():
            raise NetworkError("empty cluster: normalization undefined")
        yhat = 1.0 / np.sqrt(sizes.astype(np.float64))
        tag = B.ivec(labels[r0:r1].astype(np.int32))
        tv = B.vec(params.alpha * yhat)
        F_loc = B.tagged(tag, tv, k, dtype)
        for _ in range(params.gamma):
            F_full = B.all_gather_rows(F_loc, plan.row_counts())
            F_loc = op.apply(F_full, k, dtype, tag, tv, 1.0 - params.alpha)
        tr = B.sync_scalars([B.trace_labels(F_loc, tag, yhat)])[0]
        return 1.0 - tr / k

    # MHC reuse (as engine.run_prepared): a sample whose labels are the last
    # evaluated partition under new ids repeats its phi exactly; the labels
    # are replicated, so every rank decides the same on the host
    mhc_prev = [None, 0.0]

    def mhc_sample(labels: np.ndarray) -> float:
        prev = mhc_prev[0]
        if MHC_REUSE and prev is not None and same_partition(prev, labels, k):
            return mhc_prev[1]
        phi_s = mhc(labels, "f32")
        mhc_prev[0], mhc_prev[1] = labels.copy(), phi_s
        return phi_s

    ph.mark("init_ms")
    rng = np.random.default_rng(params.seed)
    c = min(k + 1, n)
    sizes0 = np.bincount(lab0, minlength=k)
    best_phi = mhc(lab0, "f64")
    ph.mark("mhc_ms")
    best = lab0.copy()
    hist = [(0, best_phi)]

    op.set_order(lab0[r0:r1], k)
    # ---- t = 1: exact f64 step from the replicated labels (no gather of Q0)
    Q1, _ = exact_step_dist(B, op, plan, None, c, rng, labels0=lab0, sizes0=sizes0)
    if hasattr(B, "q0_chunk"):                 # local rows, 1/sqrt(n) with the global n
        q0_loc = B.q0_chunk(lab0[r0:r1], sizes0, n, c, 0, c)
    else:
        q0_loc = _q0_chunk_host(B, lab0[r0:r1], sizes0, r1 - r0, c, 0, c)
        if r1 > r0:
            q0_loc = B.fix_q0_rows(q0_loc, n)  # the 1/sqrt(n) column uses the global n
    dq = float(np.sqrt(B.sync_scalars([B.diff2(Q1, q0_loc, c)])[0]))
    Q_loc = B.to_f32(Q1, c)
    ph.mark("step1_ms")
    stop, converged, t, err, replays = "max_iterations", False, 1, None, 0
    kd = c - 1
    try:
        block_start, Q_save, bad_acc, dq2 = 1, None, None, None
        while True:
            if t % params.tau == 0:
                if t > 1:
                    dq2_g, bad_g = B.sync_scalars([dq2, bad_acc])
                    if bad_g > 0:
                        # a suspect Cholesky pivot: replay the block with exact f64 steps
                        warnings.warn("ill-conditioned iterate; replaying tau-block in f64")
                        replays += 1
                        Q64 = B.to_f64(Q_save, c)
                        prev = Q64
                        for _ in range(t - block_start):
                            prev = Q64
                            Q64, _ = exact_step_dist(B, op, plan, Q64, c, rng)
                        dq2_g = B.sync_scalars([B.diff2(Q64, prev, c)])[0]
                        Q_loc = B.to_f32(Q64, c)
                    dq = float(np.sqrt(dq2_g))
                ph.mark("ortho_ms")
                if kd < 1:
                    raise NetworkError("discretize expects an n x k block with k >= 1")
                if _replicated_disc(B, n, c):
                    labels, empties = B.disc_replicated(Q_loc, plan.row_counts(), 1, kd)
                elif _device_partitioned_disc(B, kd, plan):
                    lab_loc, empties = B.disc_partitioned(Q_loc, plan, 1, kd)
                    labels = None
                else:
                    lab_loc, empties = discretize_dist(B, Q_loc, kd, plan)
                    labels = None
                if empties > 0:
                    raise NetworkError("cannot repair empty clusters: no movable nodes")
                if labels is None:
                    labels = B.all_gather_labels(lab_loc, plan.row_counts())
                if kd < k:                                     # k == n (engine.py:392-394)
                    raise NetworkError("the row-partitioned path needs k < n")
                ph.mark("discretize_ms")
                phi = mhc_sample(labels)
                ph.mark("mhc_ms")
                op.set_order(labels[r0:r1], k)
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
            if t % params.tau == 0 or t == 1:      # a new tau-block starts at t + 1
                block_start, Q_save, bad_acc = t, B.copy(Q_loc), B.scalar(0.0)
            # one f32 orthogonal step (engine.py:130-149), row-partitioned
            Q_full = B.all_gather_rows(Q_loc, plan.row_counts())
            Z_loc = op.apply(Q_full, c, "f32")
            G = B.all_reduce_dev(B.gram(Z_loc, c))
            Q_loc, stats = B.cholqr_apply(Z_loc, Q_loc, G, c)
            dq2, bad_acc = stats[0], bad_acc + stats[2]
            t += 1
            if t % params.tau != 0 and t < params.t_a:
                continue
            if t % params.tau != 0:                 # t_a reached between samples
                break
    except NetworkError as exc:
        err, stop = str(exc), "error"
    ph.mark("ortho_ms")
    return DistResult(best, best_phi, t, stop, hist, converged, err, replays,
                      {k_: round(v, 1) for k_, v in ph.t.items()} if ph.on else None)


# ----------------------------------------------------------------------------
class CudaBackend:
    """libancka_b200 kernels + NCCL collectives (one rank per GPU).  Blocks,
    Grams and step statistics are device tensors; host reads happen at the
    tau samples and inside the discretisation rounds only."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib
        self.torch, self.dist, self._lib, self.group = torch, dist, _lib, group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        _lib.require_device()

    @property
    def _nccl(self):
        return self.world > 1 and self.dist.get_backend(self.group) == "nccl"

    # --- data
    def _t(self, a, dtype):
        return self.torch.as_tensor(a, dtype=dtype).to("cuda")

    def vec(self, a):
        return self._t(np.asarray(a, dtype=np.float64), self.torch.float64)

    def ivec(self, a):
        return self._t(np.asarray(a, dtype=np.int32), self.torch.int32)

    def mask(self, a):
        return self._t(np.asarray(a, dtype=np.uint8), self.torch.uint8)

    def _pattern(self, m):
        """Device CSR of a row slice, uploaded once per slice object: its
        row-normalised and column-scaled value arrays are both formed on the
        device from the same rowptr / colidx / values."""
        from ._device import DeviceCSR
        cache = self.__dict__.setdefault("_patterns", {})
        hit = cache.get(id(m))
        if hit is not None and hit[0] is m:
            return hit[1]
        mm = sp.csr_matrix(m)
        if not mm.has_sorted_indices:
            mm = mm.copy()
            mm.sort_indices()
        torch = self.torch
        rp = torch.from_numpy(np.ascontiguousarray(mm.indptr, dtype=np.int64)).to("cuda")
        ci = torch.from_numpy(np.ascontiguousarray(mm.indices, dtype=np.int32)).to("cuda")
        v = torch.from_numpy(np.ascontiguousarray(mm.data, dtype=np.float64)).to("cuda")
        d = DeviceCSR(mm.shape[0], mm.shape[1], rp, ci, v, None)
        if len(cache) > 8:
            cache.clear()
        cache[id(m)] = (m, d)
        return d

    def csr_rownorm(self, m):
        """Row-normalised device CSR of a (binary) row slice, numpy's row-sum
        order (ancka_csr_row_normalize)."""
        from ._device import DeviceCSR
        base = self._pattern(m)
        out = self.torch.empty_like(base.val64)
        if base.nnz:
            self._lib.call("ancka_csr_row_normalize", base.struct(self._lib.F64), out.data_ptr(),
                           None, self._lib.stream())
        return DeviceCSR(base.rows, base.cols, base.rowptr, base.colidx, out,
                         out.to(self.torch.float32))

    def csr_colscale(self, m, col_scale):
        from ._device import DeviceCSR
        base = self._pattern(m)
        out = self.torch.empty_like(base.val64)
        cs = self.vec(col_scale)
        if base.nnz:
            self._lib.call("ancka_csr_col_scale", base.struct(self._lib.F64), cs.data_ptr(),
                           out.data_ptr(), self._lib.stream())
        return DeviceCSR(base.rows, base.cols, base.rowptr, base.colidx, out,
                         out.to(self.torch.float32))

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
        return a.cpu().numpy().astype(np.int64).reshape(-1)

    def as_rows(self, v):
        return v.reshape(-1, 1)

    def tagged(self, tag, tagval, c, dtype):
        torch = self.torch
        dt = torch.float32 if dtype == "f32" else torch.float64
        out = torch.zeros((tag.numel(), self._ld(c, dtype)), dtype=dt, device="cuda")
        rows = torch.nonzero(tag >= 0).flatten()
        out[rows, tag[rows].long()] = tagval[tag[rows].long()].to(dt)
        return out

    def cols(self, Q, c0, cc, dtype):
        from ._device import padded
        return padded(Q[:, c0:c0 + cc], self.torch.float64 if dtype == "f64" else self.torch.float32)

    def hcat(self, parts, c):
        torch = self.torch
        n = parts[0].shape[0]
        out = torch.zeros((n, self._ld(c, "f64")), dtype=torch.float64, device="cuda")
        c0 = 0
        for p in parts:
            cc = min(p.shape[1], c - c0)
            out[:, c0:c0 + cc] = p[:, :cc]
            c0 += cc
            if c0 >= c:
                break
        return out

    def add_cols(self, Z, cols, noise):
        Z = Z.clone()
        idx = self.torch.from_numpy(cols).to("cuda")
        Z[:, idx] += self.torch.from_numpy(np.ascontiguousarray(noise)).to("cuda")
        return Z

    def fix_q0_rows(self, q, n):
        return q

    def q0_chunk(self, labels, sizes, n, c, c0, cc):
        """_q0_chunk on the device: columns [c0, c0 + cc) of [1/sqrt(n) | Yhat0]
        (n = the global node count of the first column) for the given rows'
        labels, without a host-built dense block or its upload."""
        torch = self.torch
        rows = int(labels.shape[0])
        from ._device import ld_for
        q = torch.zeros((rows, ld_for(cc, torch.float64)), dtype=torch.float64, device="cuda")
        if rows == 0:
            return q
        if c0 == 0:
            q[:, 0] = 1.0 / np.sqrt(n)
        lab = torch.as_tensor(np.asarray(labels, dtype=np.int64), device="cuda")
        inv = torch.as_tensor(1.0 / np.sqrt(np.maximum(np.asarray(sizes, dtype=np.float64), 1.0)),
                              device="cuda")
        col = lab + 1 - c0
        ok = (col >= 0) & (col < cc) & (lab + 1 < c)
        idx = torch.nonzero(ok, as_tuple=True)[0]
        q[idx, col[idx]] = inv[lab[idx]]
        return q

    def copy(self, a):
        return a.clone()

    def scalar(self, v):
        return self.torch.tensor(float(v), dtype=self.torch.float64, device="cuda")

    def to_f32(self, Q, c):
        from ._device import padded
        return padded(Q[:, :c], self.torch.float32)

    def to_f64(self, Q, c):
        from ._device import padded
        return padded(Q[:, :c], self.torch.float64)

    def diff2(self, A, Bm, c):
        return ((A[:, :c].double() - Bm[:, :c].double()) ** 2).sum()

    # --- collectives
    def all_gather_rows(self, x, counts):
        torch = self.torch
        if self.world == 1:
            return x
        mx = int(np.max(counts))
        buf = torch.zeros((mx,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        buf[: x.shape[0]] = x
        if self._nccl:
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

    def synchronize(self):
        self.torch.cuda.synchronize()

    def all_reduce_dev(self, t):
        """In-place sum over ranks of a device tensor (no host round trip)."""
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return t

    def all_reduce_vec(self, t):
        return self.all_reduce_dev(t)

    def sync_scalars(self, vals):
        """Sum over ranks of a few device scalars, read back once."""
        torch = self.torch
        t = torch.stack([v if isinstance(v, torch.Tensor) else self.scalar(v) for v in vals])
        t = t.to(torch.float64)
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    # --- KNN key ring: shards are ("csr", indptr, indices, data, d) or ("dense", X)
    def x_shard(self, X, r0, r1):
        torch = self.torch
        if sp.issparse(X):
            x = sp.csr_matrix(X)[r0:r1]
            return ("csr", torch.from_numpy(x.indptr.astype(np.int64)).cuda(),
                    torch.from_numpy(x.indices.astype(np.int32)).cuda(),
                    torch.from_numpy(x.data.astype(np.float64)).cuda(), X.shape[1])
        return ("dense", torch.from_numpy(np.ascontiguousarray(X[r0:r1], dtype=np.float64)).cuda())

    def shard_rows(self, s):
        return int(s[1].numel() - 1) if s[0] == "csr" else int(s[1].shape[0])

    def knn_level(self, mine):
        """Tensor-core path of the whole X: the minimum shard level over ranks."""
        from .knn import DeviceAttributes
        if self.shard_rows(mine) == 0:
            lv = 2.0
        elif mine[0] == "csr":
            lv = DeviceAttributes.from_device_csr(mine[1], mine[2], mine[3],
                                                  (self.shard_rows(mine), mine[4])).level
        else:
            lv = DeviceAttributes.from_device_dense(mine[1]).level
        t = self.torch.tensor([float(lv)], device="cuda")
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    def _attrs(self, s, level):
        from .knn import DeviceAttributes
        if s[0] == "csr":
            if level > 0:
                xa = DeviceAttributes.__new__(DeviceAttributes)
                xa.shape, xa.dense = (self.shard_rows(s), s[4]), None
                xa.indptr, xa.indices, xa.data, xa.level = s[1], s[2], s[3], level
                return xa
            t = self.torch.sparse_csr_tensor(s[1], s[2].long(), s[3],
                                             size=(self.shard_rows(s), s[4]))
            return DeviceAttributes.from_device_dense(t.to_dense())
        return DeviceAttributes.from_device_dense(s[1])

    def knn_own(self, mine, K, r0, level):
        from .knn import knn_search_exact_device
        nq = self.shard_rows(mine)
        torch = self.torch
        if nq == 0:
            return (torch.empty((0, K), dtype=torch.int32, device="cuda"),
                    torch.empty((0, K), dtype=torch.float64, device="cuda"))
        if nq <= 1:
            return (torch.full((nq, K), -1, dtype=torch.int32, device="cuda"),
                    torch.zeros((nq, K), dtype=torch.float64, device="cuda"))
        xa = self._attrs(mine, level)
        kk = min(K, nq - 1)
        ids, sc = knn_search_exact_device(xa, kk, integer=level)
        ids = torch.where(ids >= 0, ids + r0, ids)
        if kk < K:
            ids = torch.cat([ids, torch.full((nq, K - kk), -1, dtype=ids.dtype, device="cuda")], 1)
            sc = torch.cat([sc, torch.zeros((nq, K - kk), dtype=sc.dtype, device="cuda")], 1)
        return ids.contiguous(), sc.contiguous()

    def _concat_padded(self, a, b, pad_rows):
        """[a rows, zero rows up to pad_rows, b rows] (the key block starts on a 256-row tile)."""
        torch = self.torch
        na = self.shard_rows(a)
        if a[0] == "csr":
            ip_a = torch.cat([a[1], a[1][-1:].repeat(pad_rows - na)])
            ip = torch.cat([ip_a, b[1][1:] + ip_a[-1]])
            return ("csr", ip, torch.cat([a[2], b[2]]), torch.cat([a[3], b[3]]), a[4])
        d = a[1].shape[1]
        return ("dense", torch.cat([a[1], torch.zeros((pad_rows - na, d), dtype=a[1].dtype,
                                                       device="cuda"), b[1]]))

    def knn_cross(self, mine, block, K, r0, boff, level):
        """Top-K of the own rows over the visiting block's keys only
        (ancka_knn_exact_keys on [own | pad | visiting])."""
        from ._device import WORKSPACE
        torch, _lib = self.torch, self._lib
        nq, nb = self.shard_rows(mine), self.shard_rows(block)
        qpad = (nq + 255) // 256 * 256
        x = self._concat_padded(mine, block, qpad)
        n = qpad + nb
        kk = min(K, n - 1)
        ids = torch.empty((nq, kk), dtype=torch.int32, device="cuda")
        sc = torch.empty((nq, kk), dtype=torch.float64, device="cuda")
        if x[0] == "csr" and level > 0:
            d = x[4]
            ws = WORKSPACE.get("knn_ring", _lib.load().ancka_knn_workspace_size(n, d, kk, level))
            _lib.call("ancka_knn_exact_csr_keys", x[1].data_ptr(), x[2].data_ptr(), x[3].data_ptr(),
                      n, d, kk, level, 0, nq, qpad, n, ids.data_ptr(), sc.data_ptr(),
                      ws.data_ptr(), ws.numel(), _lib.stream())
        else:
            xa = self._attrs(x, level)
            xd = xa.dense
            d = xd.shape[1]
            lv = level if level >= 0 else 0
            ws = WORKSPACE.get("knn_ring", _lib.load().ancka_knn_workspace_size(n, d, kk, lv))
            _lib.call("ancka_knn_exact_keys", xd.data_ptr(), n, d, xd.stride(0), kk, lv, 0, nq,
                      qpad, n, ids.data_ptr(), sc.data_ptr(), ws.data_ptr(), ws.numel(),
                      _lib.stream())
        ids = ids.long()
        g = torch.where(ids >= qpad, ids - qpad + boff, ids + r0)
        g = torch.where(ids < 0, torch.full_like(ids, -1), g).to(torch.int32)
        if kk < K:
            g = torch.cat([g, torch.full((nq, K - kk), -1, dtype=g.dtype, device="cuda")], 1)
            sc = torch.cat([sc, torch.zeros((nq, K - kk), dtype=sc.dtype, device="cuda")], 1)
        return g.contiguous(), sc.contiguous()

    def merge_lists(self, ia, sa, ib, sb, K):
        """Per row: first K of the union by (score desc, id asc), de-duplicated
        (ancka_knn_merge_lists, in place)."""
        ia, sa = ia.contiguous(), sa.contiguous()
        self._lib.call("ancka_knn_merge_lists", ia.data_ptr(), sa.data_ptr(), ib.data_ptr(),
                       sb.data_ptr(), ia.shape[0], K, self._lib.stream())
        return ia, sa

    def _p2p(self, send_tensors, recv_tensors):
        """Send to rank+1 and receive from rank-1.  NCCL moves device tensors
        over NVLink; other backends (gloo in the tests) go through host copies."""
        dist = self.dist
        nxt, prv = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        if not self._nccl:
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

    def _all_to_all(self, send: np.ndarray | None, sendt, dest):
        """Exchange rows of `sendt` (device, [E, w]) grouped by destination rank."""
        torch, dist = self.torch, self.dist
        order = torch.argsort(dest, stable=True)
        sendt = sendt[order]
        counts = torch.bincount(dest, minlength=self.world)
        if self.world == 1:
            return sendt
        rc = torch.empty_like(counts)
        if self._nccl:
            dist.all_to_all_single(rc, counts, group=self.group)
            sc, rcl = counts.cpu().tolist(), rc.cpu().tolist()
            out = torch.empty((sum(rcl), sendt.shape[1]), dtype=sendt.dtype, device="cuda")
            dist.all_to_all_single(out, sendt.contiguous(), output_split_sizes=rcl,
                                   input_split_sizes=sc, group=self.group)
            return out
        # gloo (tests): all-gather the variable-size parts through the host
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(self.world)]
        dist.all_gather(sizes, torch.tensor([sendt.shape[0]], dtype=torch.int64), group=self.group)
        mx = max(int(s.item()) for s in sizes)
        cnt = counts.cpu()
        buf = torch.zeros((mx, sendt.shape[1]), dtype=sendt.dtype)
        buf[: sendt.shape[0]] = sendt.cpu()
        dbuf = torch.full((mx,), -1, dtype=torch.int64)
        dbuf[: sendt.shape[0]] = dest[order].cpu()
        lst = [torch.empty_like(buf) for _ in range(self.world)]
        dl = [torch.empty_like(dbuf) for _ in range(self.world)]
        dist.all_gather(lst, buf, group=self.group)
        dist.all_gather(dl, dbuf, group=self.group)
        del cnt
        parts = [lst[r][dl[r] == self.rank] for r in range(self.world)]
        return torch.cat(parts).to("cuda")

    def knn_graph_rows(self, ids_loc, sc_loc, plan, K):
        """Rows [r0, r1) of A_K = M + M^T and P_K (knn.py:294-324): own list
        entries stay, transposed entries go to the owner of their column."""
        from ._device import WORKSPACE, DeviceCSR
        torch, _lib = self.torch, self._lib
        r0, r1, n = plan.r0, plan.r1, plan.n
        nloc = r1 - r0
        i = torch.arange(r0, r1, device="cuda", dtype=torch.int64)[:, None].expand(-1, K)
        j = ids_loc.long()
        ok = j >= 0
        i, j, s = i[ok], j[ok], sc_loc[ok]
        bounds = torch.from_numpy(plan.rows[1:-1].astype(np.int64)).to("cuda")
        dest = torch.bucketize(j, bounds, right=True)
        trip = torch.stack([j.double(), i.double(), s], 1)      # (row j, col i, s) to owner(j)
        recv = self._all_to_all(None, trip, dest)
        rows = torch.cat([i - r0, recv[:, 0].long() - r0]).to(torch.int32)
        cols = torch.cat([j, recv[:, 1].long()]).to(torch.int32)
        vals = torch.cat([s, recv[:, 2]])
        E = int(rows.numel())
        rp = torch.empty(nloc + 1, dtype=torch.int64, device="cuda")
        ci = torch.empty(max(E, 1), dtype=torch.int32, device="cuda")
        ak = torch.empty(max(E, 1), dtype=torch.float64, device="cuda")
        p64 = torch.empty_like(ak)
        p32 = torch.empty(max(E, 1), dtype=torch.float32, device="cuda")
        zero = torch.empty(max(nloc, 1), dtype=torch.uint8, device="cuda")
        nnz = torch.zeros(1, dtype=torch.int64, device="cuda")
        if nloc:
            ws = WORKSPACE.get("knn_graph_coo", _lib.load().ancka_knn_graph_coo_workspace_size(E))
            _lib.call("ancka_knn_graph_coo", rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), E,
                      nloc, n, rp.data_ptr(), ci.data_ptr(), ak.data_ptr(), p64.data_ptr(),
                      p32.data_ptr(), zero.data_ptr(), nnz.data_ptr(), ws.data_ptr(), ws.numel(),
                      _lib.stream())
        else:
            rp.zero_()
        m = int(nnz.item())
        P = DeviceCSR(nloc, n, rp, ci[:m], p64[:m], p32[:m])
        return P, zero[:nloc].cpu().numpy().astype(bool)

    def spmm(self, S, s_src, Kc, k_src, beta, selfloop, self_src, row_offset, tag, tagval, scale,
             c, dtype, order=None):
        torch, _lib = self.torch, self._lib
        f64 = dtype == "f64"
        dt = torch.float64 if f64 else torch.float32
        rows = S.rows
        out = torch.empty((rows, self._ld(c, dtype)), dtype=dt, device="cuda")
        if rows == 0:
            return out
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
                  out.data_ptr(), out.stride(0),
                  order.data_ptr() if (order is not None and not f64) else None, _lib.stream())
        return out

    def locality_order(self, labels_loc, k):
        """Local rows grouped by cluster label (ancka_locality_order): the
        processing order of the f32 row pass, so the rows in flight gather
        mostly their own cluster's rows of Q from L2 (sums unchanged)."""
        torch, _lib = self.torch, self._lib
        n = int(labels_loc.shape[0])
        if n == 0:
            return None
        lab = torch.as_tensor(np.asarray(labels_loc, dtype=np.int32), device="cuda")
        order = torch.empty(n, dtype=torch.int32, device="cuda")
        ws = torch.empty(int(_lib.load().ancka_locality_order_workspace_size(n)), dtype=torch.uint8,
                         device="cuda")
        _lib.call("ancka_locality_order", lab.data_ptr(), n, k, order.data_ptr(), ws.data_ptr(),
                  ws.numel(), _lib.stream())
        return order

    def gram(self, Z, c):
        """Local Gram Z^T Z (packed upper, f64) on the device (ancka_gram_f32)."""
        from ._device import WORKSPACE
        torch, _lib = self.torch, self._lib
        G = torch.zeros(c * (c + 1) // 2, dtype=torch.float64, device="cuda")
        if Z.shape[0]:
            ws = WORKSPACE.get("dist_orth", _lib.load().ancka_orth_workspace_size(None, c))
            _lib.call("ancka_gram_f32", Z.data_ptr(), Z.shape[0], Z.stride(0), c, G.data_ptr(),
                      ws.data_ptr(), ws.numel(), _lib.stream())
        return G

    def cholqr_apply(self, Z, Qprev, G, c):
        """Every rank factors the same all-reduced Gram (device) and applies
        R^-1 to its rows; stats = [||dQ_loc||^2, min pivot ratio, suspect
        pivots] stay on the device."""
        from ._device import WORKSPACE
        torch, _lib = self.torch, self._lib
        Qn = torch.empty_like(Z)
        stats = torch.tensor([0.0, 1.0, 0.0, 0.0], dtype=torch.float64, device="cuda")
        ws = WORKSPACE.get("dist_orth", _lib.load().ancka_orth_workspace_size(None, c))
        _lib.call("ancka_cholqr_apply_f32", Z.data_ptr(), Qprev.data_ptr(), Qn.data_ptr(),
                  Z.shape[0], Z.stride(0), c, G.data_ptr(), stats.data_ptr(), ws.data_ptr(),
                  ws.numel(), _lib.stream())
        return Qn, stats

    def cgs2(self, Z, c, allreduce):
        """Classical Gram-Schmidt with reorthogonalisation over the local rows,
        column dots all-reduced (f64): Q and |R_jj|."""
        torch = self.torch
        Q = torch.zeros_like(Z)
        d = np.zeros(c)
        for j in range(c):
            z = Z[:, j].clone()
            for _ in range(2):
                if j:
                    h = allreduce(Q[:, :j].T @ z)
                    z = z - Q[:, :j] @ h
            r = float(np.sqrt(max(float(allreduce((z * z).sum().reshape(1))[0].item()), 0.0)))
            d[j] = r
            Q[:, j] = z / r if r > 0 else z * 0.0
        return Q, d

    def argmax_update(self, P, cc, c0, best_v, best_i):
        """Running first-max argmax over centre chunks (engine.py:119)."""
        torch = self.torch
        v, i = torch.max(P[:, :cc], dim=1)
        i = i.to(torch.int64) + c0
        if best_v is None:
            return v, i
        take = v > best_v                     # strict: the earlier chunk wins ties
        return torch.where(take, v, best_v), torch.where(take, i, best_i)

    def trace_labels(self, F, labels_loc, yhat):
        """sum_i yhat[l_i] F[i, l_i] (labels: the device tag vector or host)."""
        torch = self.torch
        lab = torch.as_tensor(labels_loc, device="cuda").long()
        vals = F[torch.arange(F.shape[0], device="cuda"), lab].double()
        return (vals * torch.as_tensor(yhat, device="cuda")[lab]).sum()

    def disc_replicated(self, Q_loc, counts, col0, k):
        """discretize (engine.py:183-263) on every rank from the gathered
        block with the single-GPU device kernels: the same input on every
        rank gives the same labels (deterministic kernels).  Returns (host
        labels, empties left)."""
        torch = self.torch
        from .engine import DISCRETIZE_MAX_ITER, DISCRETIZE_TOL, _discretize_device
        q = self.all_gather_rows(Q_loc, counts).contiguous()
        n = q.shape[0]
        labels = torch.empty(n, dtype=torch.int32, device="cuda")
        info = torch.zeros(8 + 2 * DISCRETIZE_MAX_ITER + 2 * k * k, dtype=torch.float64,
                           device="cuda")
        _discretize_device(q, col0, k, DISCRETIZE_MAX_ITER, DISCRETIZE_TOL, labels, info)
        return labels.cpu().numpy().astype(np.int64), int(info[4].item())

    def disc_partitioned(self, Q_loc, plan, col0, k):
        """discretize (engine.py:162-263) over this rank's rows on the device
        (`disc_wide_dev.cu`, ANCKA_DW_* ops): the wide path's rounds with the
        cluster totals summed over the ranks by an integer all-reduce, the
        rotation replicated, the prototype passes as (value, row) all-gathers
        plus one summed row, and the empty-cluster reseed as a host loop of
        global (margin, row) choices -- no host SVD, one read-back per 8
        rounds.  8 < k <= 192.  Returns (local labels as numpy, empties)."""
        torch, _lib = self.torch, self._lib
        from .engine import DISCRETIZE_MAX_ITER as MI, DISCRETIZE_TOL as TOL
        n_loc, world = int(Q_loc.shape[0]), self.world
        dv = "cuda"
        tots = torch.zeros(k * k + k, dtype=torch.int64, device=dv)
        rvec = torch.zeros(k, dtype=torch.float64, device=dv)
        loc = torch.zeros(3, dtype=torch.float64, device=dv)
        gath = torch.zeros(3 * world, dtype=torch.float64, device=dv)
        labels = torch.empty(n_loc, dtype=torch.int32, device=dv)
        info = torch.zeros(8 + 2 * MI + 2 * k * k, dtype=torch.float64, device=dv)
        flags = torch.zeros(6, dtype=torch.int32, device=dv)
        sizes_dev = torch.zeros(k, dtype=torch.int64, device=dv)
        ws = torch.empty(int(_lib.load().ancka_discw_dist_workspace_size(n_loc, k)),
                         dtype=torch.uint8, device=dv)
        st = _lib.stream()
        _lib.call("ancka_discw_dist_init", Q_loc.data_ptr(), Q_loc.stride(0), col0, n_loc, plan.n,
                  plan.r0, k, MI, float(TOL), tots.data_ptr(), rvec.data_ptr(), loc.data_ptr(),
                  labels.data_ptr(), info.data_ptr(), ws.data_ptr(), ws.numel(), st)

        def op(code, a=0, b=0, ptr=None):
            _lib.call("ancka_discw_dist_op", ws.data_ptr(), code, a, b, ptr, st)

        def summed(t):
            if world > 1:
                self.dist.all_reduce(t, group=self.group)

        def gathered():
            if world == 1:
                gath.copy_(loc)
            else:
                self.dist.all_gather_into_tensor(gath, loc, group=self.group) if self._nccl else \
                    gath.copy_(torch.cat(self._gather_list(loc)))

        def reseed():
            sizes = tots[k * k:].cpu().numpy().astype(np.int64)
            op(DW_MARGINS)
            for c in np.flatnonzero(sizes == 0):
                sizes_dev.copy_(torch.from_numpy(sizes))
                op(DW_RESEED_CAND, 0, 0, sizes_dev.data_ptr())
                gathered()
                g = gath.view(world, 3).cpu().numpy()
                ok = g[:, 1] >= 0
                if not ok.any():
                    break                               # no movable node left
                cand = g[ok]
                w = np.lexsort((cand[:, 1], -cand[:, 0]))[0]    # margin desc, row asc
                row, old = int(cand[w, 1]), int(cand[w, 2])
                if plan.r0 <= row < plan.r1:
                    op(DW_MOVE_ROW, int(c), row - plan.r0)
                sizes[old] -= 1
                sizes[c] += 1
            op(DW_SNAP)
            summed(tots)

        for run in (0, 1):
            op(DW_START, run)
            if run == 1:                                    # _prototype_rotation
                op(DW_PROTO_PICK, world, 0, gath.data_ptr())
                summed(rvec)
                op(DW_PROTO_SETCOL, 1, 0)
                for j in range(1, k):
                    op(DW_PROTO_PASS, 1, j)
                    gathered()
                    op(DW_PROTO_PICK, world, -1, gath.data_ptr())
                    summed(rvec)
                    op(DW_PROTO_SETCOL, 1, j)
            first = run == 0
            while True:
                for _ in range(8):
                    op(DW_ROUND_LOCAL, run, int(first))
                    first = False
                    summed(tots)
                    op(DW_CHECK_EMPTY, run)
                    op(DW_POLAR, run)
                op(DW_FLAGS, 0, 0, flags.data_ptr())
                f = flags.cpu().numpy()
                if f[2]:                                    # an empty cluster: reseed, then rotate
                    reseed()
                    op(DW_CLEAR_PAUSE)
                    op(DW_POLAR, run)
                    continue
                if f[run]:
                    break
        op(DW_FINISH)
        inf = info[:8].cpu().numpy()
        return labels.cpu().numpy().astype(np.int64), int(inf[4])

    def _gather_list(self, t):
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return out

    # --- row-partitioned discretisation primitives (discretize_dist)
    def disc_prepare(self, Q_loc, col0, k):
        torch, _lib = self.torch, self._lib
        from ._device import ld_for
        n = Q_loc.shape[0]
        ldt = ld_for(k, torch.float32)
        st = {"k": k, "ldt": ldt, "n": n,
              "qt": torch.empty((max(n, 1), ldt), dtype=torch.float32, device="cuda"),
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
        """k x k sums and k counts of this round: 64-bit fixed point on the
        device, all-reduced as integers (exact, order free), one read-back."""
        torch, _lib = self.torch, self._lib
        n = st["n"]
        if n:
            _lib.call("ancka_disc_accumulate", st["qt"].data_ptr(), st["ldt"], n, k, lab.data_ptr(),
                      st["scale"], st["S"].data_ptr(), st["cnt"].data_ptr(), _lib.stream())
        else:
            st["S"].zero_()
            st["cnt"].zero_()
        both = torch.cat([st["S"], st["cnt"]])
        if self.world > 1:
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
