"""CPU oracle for the ANCKA clustering hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy/scipy, the algorithm of the reference
package (`/root/reference/pkg/src/ancka`, v0.1.0).  Every function cites
the reference file:line it follows.  It exists for three callers only:

* `tests/` (parity checker for the CUDA path),
* `__graft_entry__.smoke()` (one tiny CUDA-vs-oracle check),
* `bench.py` (`cpu_baseline` leg and `--impl reference`).

The product package `paper_2408_05459_b200` never imports it: the product
path has no CPU fallback.

Parity pinning: `tests/golden/make_golden.py` runs the *reference itself*
(importable in the build container from /root/reference) on seeded inputs
and freezes its outputs as `tests/golden/*.npz`; `tests/test_oracle_golden.py`
checks this restatement against every one of them (bit-exact for integer
outputs, <=1e-12 for floating point).

Data model: plain arrays.  A network is a dict
    {"kind": "graph"|"hypergraph"|"multiplex", "S": csr (A n x n, or H m x n),
     "layers": [csr n x n, ...] (multiplex), "directed": bool, "X": ndarray or csr}
"""
from __future__ import annotations

import warnings

import numpy as np
import scipy.sparse as sp

ALPHA, BETA, GAMMA = 0.2, 0.5, 3
DISC_ROUNDS, DISC_TOL = 100, 1e-10          # engine.py:37-38


class OracleError(ValueError):
    """Mirrors ancka.NetworkError (network.py:39-40)."""


# ----------------------------------------------------------------------------
# network.py
# ----------------------------------------------------------------------------
def canon_csr(m, what="matrix"):
    """check_sparse_nonneg (network.py:43-63): sorted, deduplicated, no zeros."""
    m = sp.csr_matrix(m, copy=True)
    if m.nnz and (m.indices.min() < 0 or m.indices.max() >= m.shape[1]):
        raise OracleError(f"{what}: column index out of range")
    m.sum_duplicates()
    m.sort_indices()
    m.eliminate_zeros()
    if m.nnz:
        if not np.isfinite(m.data).all():
            raise OracleError(f"{what}: non-finite values are not allowed")
        if (m.data < 0).any():
            raise OracleError(f"{what}: negative values are not allowed")
    return m


def sym_union(a):
    """symmetrize_union (network.py:261-263): pattern union max(A, A^T)."""
    return canon_csr(a.maximum(a.T), "adjacency")


def clean_network(net):
    """validate_network (network.py:266-313), structural cleanup only
    (multiplex layers are only canonicalised, network.py:107-126)."""
    net = dict(net)
    if net["kind"] == "multiplex":
        net["layers"] = [canon_csr(a, f"layer {i}") for i, a in enumerate(net["layers"])]
        return net
    s = canon_csr(net["S"], "structure")
    if net["kind"] == "hypergraph":
        keep = np.diff(s.indptr) >= 2
        if not keep.all():
            s = canon_csr(s[keep], "incidence")
    else:
        dups = int((s.data > 1).sum())
        loops = int(s.diagonal().astype(bool).sum())
        if dups or loops:
            s = s.copy()
            s.data = np.minimum(s.data, 1.0)
            s.setdiag(0)
            s = canon_csr(s, "adjacency")
    net["S"] = s
    return net


def structural_degree(net):
    """node_degrees (network.py:316-328): pattern counts (multiplex: summed
    over layers, layer_degrees network.py:331-337)."""
    if net["kind"] == "multiplex":
        return np.sum([np.asarray((a != 0).sum(axis=1)).ravel().astype(np.float64)
                       for a in net["layers"]], axis=0)
    s = net["S"]
    if net["kind"] == "hypergraph":
        return np.asarray((s != 0).sum(axis=0)).ravel().astype(np.float64)
    a = sym_union(s) if net.get("directed") else s
    return np.asarray((a != 0).sum(axis=1)).ravel().astype(np.float64)


def default_K(kind, n):
    """default_knn_k (network.py:232-235)."""
    return 10 if (kind == "hypergraph" or n > 100_000) else 50


# ----------------------------------------------------------------------------
# knn.py (exact mode)
# ----------------------------------------------------------------------------
def unit_rows(x):
    """_normalize_rows (knn.py:54-65): L2-normalise, zero rows stay zero."""
    if sp.issparse(x):
        x = x.tocsr().astype(np.float64)
        nrm = np.sqrt(np.asarray(x.multiply(x).sum(axis=1)).ravel())
        scale = np.where(nrm > 0, 1.0 / np.where(nrm > 0, nrm, 1.0), 0.0)
        return (sp.diags(scale) @ x).tocsr(), nrm
    x = np.asarray(x, dtype=np.float64)
    nrm = np.linalg.norm(x, axis=1)
    scale = np.where(nrm > 0, 1.0 / np.where(nrm > 0, nrm, 1.0), 0.0)
    return x * scale[:, None], nrm


def _select_row(sims_row, K):
    """_ordered_top_k (knn.py:83-98): keep strictly positive entries; above K
    of them, partition at the K-th largest value, keep everything above it
    and the smallest-index ties at it; order by a stable sort on -value
    (so (value desc, index asc)).  Same selection work as the reference
    (partition, then a sort of K entries), so the CPU arm is timed fairly."""
    pos = np.flatnonzero(sims_row > 0)
    if pos.size > K:
        vals = sims_row[pos]
        kth = np.partition(vals, vals.size - K)[vals.size - K]
        above = pos[vals > kth]
        ties = pos[vals == kth]
        pos = np.concatenate([above, ties[: K - above.size]])
        pos.sort()
    order = np.argsort(-sims_row[pos], kind="stable")
    return pos[order]


def knn_rows(X, rows, K, normalized=None):
    """Exact lists of the query rows `rows` against all n keys, the blocked
    scan of knn.py:112-140 restricted to a row sample (the reference's own
    sampled form is knn._exact_rows_for, knn.py:227-239).  Used to time the
    CPU KNN on a bounded sample and to check sampled GPU rows."""
    xn, nrm = unit_rows(X) if normalized is None else normalized
    n = xn.shape[0]
    rows = np.asarray(rows, dtype=np.int64)
    right = xn.T.tocsc() if sp.issparse(xn) else xn.T
    block = max(16, min(4096, int(2.5e7 // max(n, 1))))
    ids = np.full((rows.size, K), -1, dtype=np.int64)
    scores = np.zeros((rows.size, K), dtype=np.float64)
    for lo in range(0, rows.size, block):
        chunk = rows[lo: lo + block]
        blk = xn[chunk] @ right
        blk = blk.toarray() if sp.issparse(blk) else np.asarray(blk)
        blk[np.arange(chunk.size), chunk] = -1.0
        for r in range(chunk.size):
            if nrm[chunk[r]] == 0.0:
                continue
            sel = _select_row(blk[r], K)
            ids[lo + r, : sel.size] = sel
            scores[lo + r, : sel.size] = np.minimum(blk[r, sel], 1.0)
    return ids, scores


def knn_exact(X, K, block_rows=None):
    """knn_search_exact (knn.py:112-140).  Returns (ids int64 (n,K) padded -1,
    scores f64 (n,K) padded 0)."""
    xn, nrm = unit_rows(X)
    n = xn.shape[0]
    if K >= n:
        raise OracleError(f"K={K} must be smaller than n={n}")
    if block_rows is None:
        block_rows = max(16, min(4096, int(2.5e7 // max(n, 1))))
    right = xn.T.tocsc() if sp.issparse(xn) else xn.T
    ids = np.full((n, K), -1, dtype=np.int64)
    scores = np.zeros((n, K), dtype=np.float64)
    for lo in range(0, n, block_rows):
        hi = min(lo + block_rows, n)
        blk = xn[lo:hi] @ right
        blk = blk.toarray() if sp.issparse(blk) else np.asarray(blk)
        blk[np.arange(hi - lo), np.arange(lo, hi)] = -1.0
        for r in range(hi - lo):
            if nrm[lo + r] == 0.0:
                continue
            sel = _select_row(blk[r], K)
            ids[lo + r, : sel.size] = sel
            scores[lo + r, : sel.size] = np.minimum(blk[r, sel], 1.0)
    return ids, scores


# ----------------------------------------------------------------------------
# knn.py (approximate mode: inverted-file index, knn.py:143-280)
# ----------------------------------------------------------------------------
def ivf_defaults(n, nlist=None, nprobe=None):
    """knn.py:181-187."""
    if nlist is None:
        nlist = int(min(4096, max(8, round(np.sqrt(n)))))
    nlist = min(nlist, n)
    if nprobe is None:
        nprobe = max(4, nlist // 32)
    return nlist, min(nprobe, nlist)


def ivf_unit_f32(X):
    """knn.py:172-175: the f32 dense copy of the normalised rows."""
    xn, nrm = unit_rows(X)
    if sp.issparse(xn):
        xn = np.asarray(xn.todense())
    return np.ascontiguousarray(xn, dtype=np.float32), nrm


def ivf_train(xn, nlist, seed):
    """_train_ivf (knn.py:143-153): sklearn KMeans on at most 50 nlist rows."""
    from sklearn.cluster import KMeans
    sample = xn
    if xn.shape[0] > 50 * nlist:
        rng = np.random.default_rng(seed)
        sample = xn[rng.choice(xn.shape[0], size=50 * nlist, replace=False)]
    km = KMeans(n_clusters=nlist, n_init=1, max_iter=25, random_state=seed)
    km.fit(sample)
    return km.cluster_centers_.astype(xn.dtype)


def ivf_assign(xn, centroids):
    """_batched_argmax_assign (knn.py:216-222)."""
    n = xn.shape[0]
    out = np.empty(n, dtype=np.int64)
    step = max(1, int(2.5e7 // max(centroids.shape[0], 1)))
    for lo in range(0, n, step):
        out[lo: lo + step] = np.argmax(xn[lo: lo + step] @ centroids.T, axis=1)
    return out


def ivf_lists(labels, nlist):
    """knn.py:198-203: member rows of each list, ascending."""
    order = np.argsort(labels, kind="stable")
    cuts = np.searchsorted(labels[order], np.arange(nlist + 1))
    return [order[cuts[c]: cuts[c + 1]] for c in range(nlist)]


def ivf_probes(xn, centroids, rows, nprobe):
    """The probe sets of knn.py:246-250 (as sets; argpartition's order is not
    part of the contract) plus the f32 centroid scores."""
    cd = xn[rows] @ centroids.T
    return np.argpartition(-cd, nprobe - 1, axis=1)[:, :nprobe], cd


def ivf_search_all(xn, nrm, centroids, lists, K, nprobe):
    """_ivf_search_all (knn.py:236-262): (ids (n,K) padded -1, scores)."""
    n, nlist = xn.shape[0], centroids.shape[0]
    ids = np.full((n, K), -1, dtype=np.int64)
    scores = np.zeros((n, K), dtype=np.float64)
    step = max(1, int(2.5e7 // max(nlist, 1)))
    for lo in range(0, n, step):
        hi = min(lo + step, n)
        cd = xn[lo:hi] @ centroids.T
        probes = None if nprobe >= nlist else np.argpartition(-cd, nprobe - 1, axis=1)[:, :nprobe]
        for r in range(hi - lo):
            q = lo + r
            if nrm[q] == 0.0:
                continue
            cand = np.arange(n) if probes is None else np.sort(np.concatenate(
                [lists[c] for c in probes[r]]))
            sims = xn[cand] @ xn[q]
            sims[cand == q] = -1.0
            sel = _select_row(sims.astype(np.float64), K)
            ids[q, : sel.size] = cand[sel]
            scores[q, : sel.size] = np.minimum(sims[sel].astype(np.float64), 1.0)
    return ids, scores


def ivf_exact_rows(xn, nrm, rows, K):
    """_exact_rows_for (knn.py:225-233): f32 similarities of the audit rows."""
    out = {}
    step = max(1, int(2.5e7 // max(xn.shape[0], 1)))
    for lo in range(0, rows.size, step):
        chunk = rows[lo: lo + step]
        sims = xn[chunk] @ xn.T
        sims[np.arange(chunk.size), chunk] = -1.0
        for j, i in enumerate(chunk):
            out[int(i)] = (np.empty(0, dtype=np.int64) if nrm[i] == 0.0
                           else _select_row(sims[j].astype(np.float64), K).astype(np.int64))
    return out


def ivf_recall(ids, truth, rows):
    """_audit_recall (knn.py:265-274)."""
    hits = []
    for i in rows:
        t = truth[int(i)]
        if t.size == 0:
            continue
        got = ids[int(i)]
        hits.append(np.isin(t, got[got >= 0]).mean())
    return float(np.mean(hits)) if hits else 1.0


def knn_approx(X, K, recall_target=0.9, seed=0, nlist=None, nprobe=None, audit_size=1000,
               centroids=None):
    """knn_search_approx (knn.py:156-213).  Returns (ids, scores, info) with
    info = {nlist, nprobe (final), recall, escalations, centroids}."""
    xn, nrm = ivf_unit_f32(X)
    n = xn.shape[0]
    if K >= n:
        raise OracleError(f"K={K} must be smaller than n={n}")
    if centroids is not None:
        nlist = centroids.shape[0]
    nlist, nprobe = ivf_defaults(n, nlist, nprobe)
    C = ivf_train(xn, nlist, seed) if centroids is None else np.asarray(centroids, np.float32)
    lists = ivf_lists(ivf_assign(xn, C), nlist)
    rng = np.random.default_rng(seed)
    m = min(n, max(audit_size, 1000))
    audit = np.sort(rng.choice(n, size=m, replace=False))
    truth = ivf_exact_rows(xn, nrm, audit, K)
    esc = 0
    while True:
        ids, scores = ivf_search_all(xn, nrm, C, lists, K, nprobe)
        recall = ivf_recall(ids, truth, audit)
        if recall >= recall_target or nprobe >= nlist:
            break
        nprobe = min(nlist, nprobe * 2)
        esc += 1
    return ids, scores, {"nlist": nlist, "nprobe": nprobe, "recall": recall, "escalations": esc,
                         "centroids": C}


def knn_adjacency(ids, scores):
    """build_knn_adjacency (knn.py:294-309): A_K = M + M^T, sorted CSR."""
    n = ids.shape[0]
    ok = ids != -1
    rows = np.repeat(np.arange(n), ok.sum(axis=1))
    m = sp.csr_matrix((scores[ok], (rows, ids[ok])), shape=(n, n))
    a = (m + m.T).tocsr()
    a.sort_indices()
    return a


def row_stochastic(a):
    """_row_normalize (walk.py:38-44) == knn_transition (knn.py:312-324)."""
    rs = np.asarray(a.sum(axis=1)).ravel()
    inv = np.divide(1.0, rs, out=np.zeros_like(rs), where=rs > 0)
    p = (sp.diags(inv) @ a).tocsr()
    p.sort_indices()
    return p, rs == 0


# ----------------------------------------------------------------------------
# walk.py
# ----------------------------------------------------------------------------
def make_operator(net, p_k, knn_zero, alpha=ALPHA, beta=BETA, gamma=GAMMA):
    """build_walk_operator (walk.py:107-132) with beta_vector (walk.py:47-57),
    hypergraph_factors (walk.py:60-71), graph_transition (walk.py:74-79)."""
    deg = structural_degree(net)
    n = deg.size
    b = np.full(n, float(beta))
    b[deg == 0] = 1.0
    b[np.asarray(knn_zero, dtype=bool)] = 0.0
    op = {"kind": net["kind"], "n": n, "alpha": float(alpha), "gamma": int(gamma),
          "beta": b, "p_k": p_k, "degrees": deg,
          "selfloop": np.flatnonzero((deg == 0) & (b == 0.0))}
    if net["kind"] == "multiplex":   # multiplex_transition (walk.py:82-86)
        op["layers"] = [row_stochastic(a)[0] for a in net["layers"]]
        return op
    s = net["S"]
    if net["kind"] == "hypergraph":
        op["p_v"], _ = row_stochastic(s.T.tocsr())
        op["p_e"], _ = row_stochastic(s)
    else:
        op["p_n"], _ = row_stochastic(sym_union(s) if net.get("directed") else s)
    return op


def structure_apply(op, m):
    """apply_structure (walk.py:135-150)."""
    if m.shape[0] != op["n"]:
        raise OracleError("block/operator size mismatch")
    if op["kind"] == "multiplex":   # layer average (walk.py:143-147)
        out = op["layers"][0] @ m
        for p in op["layers"][1:]:
            out += p @ m
        out /= len(op["layers"])
    elif op["kind"] == "hypergraph":
        out = op["p_v"] @ (op["p_e"] @ m)
    else:
        out = op["p_n"] @ m
    sl = op["selfloop"]
    if sl.size:
        out[sl] += m[sl]
    return out


def structure_apply_t(op, m):
    """apply_structure_rowvec (walk.py:153-174): (c x n) block times P_struct."""
    mt = np.ascontiguousarray(m.T)
    if op["kind"] == "multiplex":   # walk.py:168-172
        acc = op["layers"][0].T @ mt
        for p in op["layers"][1:]:
            acc += p.T @ mt
        out = acc.T / len(op["layers"])
    elif op["kind"] == "hypergraph":
        out = (op["p_e"].T @ (op["p_v"].T @ mt)).T
    else:
        out = (op["p_n"].T @ mt).T
    out = np.ascontiguousarray(out)
    sl = op["selfloop"]
    if sl.size:
        out[:, sl] += m[:, sl]
    return out


def joint_apply(op, m):
    """apply_joint_transition (walk.py:177-190): (I-B) P_N M + B P_K M."""
    m = np.asarray(m, dtype=np.float64)
    vec = m.ndim == 1
    if vec:
        m = m[:, None]
    b = op["beta"][:, None]
    out = (1.0 - b) * structure_apply(op, m) + b * (op["p_k"] @ m)
    return out.ravel() if vec else out


def dense_P(op):
    """dense_transition (walk.py:193-208), small n only."""
    if op["kind"] == "multiplex":
        pn = sum(p.toarray() for p in op["layers"]) / len(op["layers"])
    elif op["kind"] == "hypergraph":
        pn = (op["p_v"] @ op["p_e"]).toarray()
    else:
        pn = op["p_n"].toarray()
    sl = op["selfloop"]
    if sl.size:
        pn[sl, sl] += 1.0
    b = op["beta"][:, None]
    return (1.0 - b) * pn + b * op["p_k"].toarray()


# ----------------------------------------------------------------------------
# engine.py
# ----------------------------------------------------------------------------
def sizes_of(labels, k):
    return np.bincount(labels, minlength=k)


def unit_membership(labels, k):
    """normalize_bcm (engine.py:75-84)."""
    sz = sizes_of(labels, k)
    if (sz == 0).any():
        raise OracleError("empty cluster: normalization undefined")
    y = np.zeros((labels.size, k))
    y[np.arange(labels.size), labels] = 1.0 / np.sqrt(sz[labels])
    return y


def greedy_init(op, k, t_i, alpha):
    """init_bcm (engine.py:87-127).  Returns (labels, centers)."""
    n, deg = op["n"], op["degrees"]
    if k > n:
        raise OracleError(f"k={k} exceeds node count n={n}")
    rank = np.lexsort((np.arange(n), -deg))
    live = int((deg > 0).sum())
    if k > live:
        warnings.warn("too few nonzero-degree nodes; filling centers in index order")
        chosen = set(rank[:live].tolist())
        fill = [i for i in range(n) if i not in chosen][: k - live]
        centers = np.sort(np.array(sorted(chosen) + fill, dtype=np.int64))
    else:
        centers = np.sort(rank[:k])
    pi0 = np.zeros((k, n))
    pi0[np.arange(k), centers] = alpha
    pi = pi0.copy()
    for _ in range(t_i):
        pi = (1.0 - alpha) * structure_apply_t(op, pi) + pi0
    labels = np.argmax(pi, axis=0).astype(np.int64)
    if (sizes_of(labels, k) == 0).any():
        warnings.warn("greedy init left empty cluster(s); pinning centers")
        labels = labels.copy()
        labels[centers] = np.arange(k)
    return labels, centers


def qr_step(op, q_prev, rng):
    """orthogonal_step (engine.py:130-149): apply, Householder QR, noise on
    rank-deficient columns, sign fix so diag(R) >= 0."""
    z = joint_apply(op, q_prev)
    q, r = np.linalg.qr(z)
    dg = np.abs(np.diag(r))
    bad = dg < 1e-12 * max(1.0, dg.max() if dg.size else 1.0)
    if bad.any():
        warnings.warn(f"rank-deficient iterate; perturbing {int(bad.sum())} column(s)")
        z = z.copy()
        z[:, bad] += 1e-8 * rng.standard_normal((z.shape[0], int(bad.sum())))
        q, r = np.linalg.qr(z)
    sgn = np.where(np.diag(r) < 0, -1.0, 1.0)
    return q * sgn, r * sgn[:, None]


def _second_best(scores):
    return np.partition(scores, -2, axis=1)[:, -2]


def _refill_empty(labels, scores, k):
    """_reseed_empty_columns (engine.py:162-180)."""
    empties = np.flatnonzero(sizes_of(labels, k) == 0)
    if empties.size == 0 or k < 2 or scores.shape[1] < 2:
        return labels
    labels = labels.copy()
    margin = _second_best(scores)
    for c in empties:
        movable = sizes_of(labels, k)[labels] >= 2
        if not movable.any():
            break
        labels[int(np.argmax(np.where(movable, margin, -np.inf)))] = c
    return labels


def _rounding_run(qt, rot, rounds, tol):
    """_alternate_rounding (engine.py:183-206)."""
    n, k = qt.shape
    objs = []
    labels = np.zeros(n, dtype=np.int64)
    scores = qt @ rot
    done = False
    for _ in range(rounds):
        scores = qt @ rot
        labels = _refill_empty(np.argmax(scores, axis=1), scores, k)
        sz = sizes_of(labels, k).astype(np.float64)
        w = np.divide(1.0, sz[labels], out=np.zeros(n), where=sz[labels] > 0)
        ytil = np.zeros((n, k))
        ytil[np.arange(n), labels] = w
        u, om, vh = np.linalg.svd(ytil.T @ qt)
        objs.append(n - 2.0 * float(om.sum()))
        if len(objs) >= 2 and abs(objs[-1] - objs[-2]) < tol:
            done = True
            break
        rot = vh.T @ u.T
    return labels, scores, objs, done


def _prototype_start(qt, k):
    """_prototype_rotation (engine.py:209-218)."""
    rot = np.zeros((k, k))
    rot[:, 0] = qt[0]
    acc = np.zeros(qt.shape[0])
    for j in range(1, k):
        acc += np.abs(qt @ rot[:, j - 1])
        rot[:, j] = qt[int(np.argmin(acc))]
    return rot


def discretize(q, rounds=DISC_ROUNDS, tol=DISC_TOL):
    """discretize (engine.py:221-263).  Returns dict(labels, scores, objs,
    converged, runs)."""
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 2 or q.shape[1] < 1:
        raise OracleError("discretize expects an n x k block with k >= 1")
    n, k = q.shape
    nrm = np.linalg.norm(q, axis=1)
    if (nrm == 0).any():
        warnings.warn(f"{int((nrm == 0).sum())} all-zero row(s); assigning to cluster 0")
    qt = np.divide(q, nrm[:, None], out=np.zeros_like(q), where=nrm[:, None] > 0)
    best, runs = None, []
    for name, rot in (("identity", np.eye(k)), ("prototype", _prototype_start(qt, k))):
        res = _rounding_run(qt, rot, rounds, tol)
        runs.append((name, res[2]))
        if best is None or res[2][-1] < best[2][-1] - 1e-15:
            best = res
    labels, scores, objs, done = best
    return {"labels": labels, "scores": scores, "objs": objs, "converged": done,
            "runs": runs}


def repair(labels, scores, k):
    """repair_empty_clusters (engine.py:266-288)."""
    empties = np.flatnonzero(sizes_of(labels, k) == 0)
    if empties.size == 0:
        return labels
    warnings.warn(f"re-seeding {empties.size} empty cluster(s) after discretization")
    labels = labels.copy()
    margin = _second_best(scores) if scores.shape[1] >= 2 else scores[:, 0]
    for c in empties:
        movable = sizes_of(labels, k)[labels] >= 2
        if not movable.any():
            raise OracleError("cannot repair empty clusters: no movable nodes")
        labels[int(np.argmax(np.where(movable, margin, -np.inf)))] = c
    return labels


def mhc(op, labels, k):
    """calc_mhc (engine.py:291-299)."""
    yh = unit_membership(labels, k)
    f0 = op["alpha"] * yh
    f = f0.copy()
    for _ in range(op["gamma"]):
        f = (1.0 - op["alpha"]) * joint_apply(op, f) + f0
    return 1.0 - float(np.einsum("ij,ij->", yh, f)) / k


def build(net, k, knn_k=None, alpha=ALPHA, beta=BETA, gamma=GAMMA, knn=None):
    """build_pipeline (engine.py:302-340), exact KNN only.  `knn`=(ids, scores)
    injects neighbour lists the way the reference's .aknn cache does."""
    net = clean_network(net)
    deg_n = structural_degree(net).size
    if k > deg_n:
        raise OracleError(f"k={k} exceeds node count n={deg_n}")
    K = knn_k if knn_k is not None else default_K(net["kind"], deg_n)
    K = min(K, deg_n - 1)
    if knn is None:
        ids, scores = knn_exact(net["X"], K)
    else:
        ids, scores = knn
    adj = knn_adjacency(ids, scores)
    p_k, zero = row_stochastic(adj)
    return make_operator(net, p_k, zero, alpha, beta, gamma), (ids, scores, adj)


def run(net, k, knn_k=None, alpha=ALPHA, beta=BETA, gamma=GAMMA, eps_q=0.005,
        t_a=1000, t_i=25, tau=5, seed=0, early_stop=True, knn=None):
    """run_ancka (engine.py:343-437).  Returns a dict with labels, mhc,
    iterations, stop_reason, history and the operator."""
    import time
    tm = {"knn_ms": 0.0, "init_ms": 0.0, "ortho_ms": 0.0, "discretize_ms": 0.0, "mhc_ms": 0.0}
    calls = {"ortho": 0, "discretize": 0, "mhc": 0}
    t0 = time.perf_counter()
    op, knn_out = build(net, k, knn_k, alpha, beta, gamma, knn)
    t1 = time.perf_counter()
    tm["knn_ms"] = (t1 - t0) * 1e3
    labels0, _ = greedy_init(op, k, t_i, alpha)
    tm["init_ms"] = (time.perf_counter() - t1) * 1e3
    rng = np.random.default_rng(seed)
    n = op["n"]
    q = np.concatenate([np.full((n, 1), 1.0 / np.sqrt(n)), unit_membership(labels0, k)], axis=1)
    q = q[:, :n]
    t1 = time.perf_counter()
    best_phi = mhc(op, labels0, k)
    tm["mhc_ms"] += (time.perf_counter() - t1) * 1e3
    calls["mhc"] += 1
    best = labels0
    hist = [(0, best_phi)]
    stop, it, err = "max_iterations", 0, None
    try:
        for t in range(1, t_a + 1):
            it = t
            q_prev = q
            t1 = time.perf_counter()
            q, _ = qr_step(op, q_prev, rng)
            tm["ortho_ms"] += (time.perf_counter() - t1) * 1e3
            calls["ortho"] += 1
            if t % tau:
                continue
            t1 = time.perf_counter()
            d = discretize(q[:, 1:])
            lab = repair(d["labels"], d["scores"], k)
            t2 = time.perf_counter()
            phi = mhc(op, lab, k)
            tm["discretize_ms"] += (t2 - t1) * 1e3
            tm["mhc_ms"] += (time.perf_counter() - t2) * 1e3
            calls["discretize"] += 1
            calls["mhc"] += 1
            hist.append((t, phi))
            if phi < best_phi:
                best_phi, best = phi, lab
            if float(np.linalg.norm(q - q_prev)) < eps_q:
                stop = "subspace_converged"
                break
            if early_stop and len(hist) >= 3 and hist[-3][1] < hist[-2][1] < hist[-1][1]:
                stop = "mhc_rising"
                break
    except OracleError as exc:
        err, stop = str(exc), "error"
    return {"labels": best, "mhc": best_phi, "iterations": it, "stop_reason": stop,
            "history": hist, "q": q, "op": op, "knn": knn_out, "labels0": labels0,
            "error": err, "timings_ms": tm, "calls": calls}
