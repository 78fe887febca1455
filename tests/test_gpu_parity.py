"""CUDA path vs the oracle and the reference's golden outputs (needs a B200).

Tolerances (north star): f64 operator application is
bit-identical to scipy (asserted <= 1e-15 absolute here); f32 operator
outputs within 1e-5 relative; KNN index sets exact up to exact ties at the
K-th value; labels at ARI >= 0.99.
"""
from __future__ import annotations

import warnings

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from conftest import load_csr, load_x, oracle_net, random_seeds
from oracle import ancka_cpu as oc

pytestmark = pytest.mark.gpu
warnings.simplefilter("ignore")

ancka = pytest.importorskip("paper_2408_05459_b200")
from paper_2408_05459_b200 import _lib  # noqa: E402
from paper_2408_05459_b200._device import DeviceCSR, padded  # noqa: E402
from paper_2408_05459_b200.knn import build_knn_graph_device  # noqa: E402


def ari(a, b):
    from sklearn.metrics import adjusted_rand_score
    return adjusted_rand_score(a, b)


def _net(z, p):
    kind = str(z[p + "kind"])
    X = load_x(z, p + "X")
    if kind == "multiplex":
        from conftest import load_layers
        return ancka.AttributedNetwork.multiplex(load_layers(z, p), X)
    S = load_csr(z, p + "S")
    if kind == "hypergraph":
        return ancka.AttributedNetwork.hypergraph(S, X)
    return ancka.AttributedNetwork.graph(S, X, directed=bool(z[p + "directed"]))


def _op_from_golden(z, p):
    net, _ = ancka.validate_network(_net(z, p))
    pk = load_csr(z, p + "PK")
    zero = np.asarray(pk.sum(axis=1)).ravel() == 0
    return ancka.build_walk_operator(net, pk, zero, 0.2, float(z[p + "beta"]), int(z[p + "gamma"]))


def _cases(z):
    return [s for s in random_seeds(z) if not bool(z[f"s{s}_skip"])]


def knn_sets_match(ids_a, ids_b, X, K):
    """Tie-aware comparison: rows may differ only by members of the exact tie
    group at the K-th similarity (f64 cosines, |s - s_K| <= 1e-12)."""
    xn, _ = oc.unit_rows(X)
    xn = xn.toarray() if sp.issparse(xn) else xn
    bad = 0
    for i in range(ids_a.shape[0]):
        a = set(ids_a[i][ids_a[i] >= 0].tolist())
        b = set(ids_b[i][ids_b[i] >= 0].tolist())
        if a == b:
            continue
        if len(a) != len(b):
            bad += 1
            continue
        s = xn @ xn[i]
        members = sorted(a | b, key=lambda j: -s[j])
        kth = min(s[j] for j in b)
        diff = a ^ b
        if not all(abs(s[j] - kth) <= 1e-12 for j in diff):
            bad += 1
    return bad


def test_device_present():
    _lib.require_device()
    assert _lib.load().ancka_abi_version() == 1


def test_apply_f64_bit_exact(golden_random):
    z = golden_random
    worst = 0.0
    for s in _cases(z):
        p = f"s{s}_"
        op = _op_from_golden(z, p)
        np.testing.assert_array_equal(op.beta, z[p + "beta_vec"])
        out = ancka.apply_joint_transition(op, z[p + "M"])
        worst = max(worst, float(np.abs(out - z[p + "apply"]).max()))
        out_t = ancka.apply_structure_rowvec(op, z[p + "M"].T.copy())
        worst = max(worst, float(np.abs(out_t - z[p + "apply_t"]).max()))
    assert worst <= 1e-15, worst


def test_apply_f32_within_1e5(golden_random):
    z = golden_random
    for s in _cases(z):
        p = f"s{s}_"
        op = _op_from_golden(z, p)
        m = z[p + "M"]
        q = padded(torch.from_numpy(m), torch.float32)
        out = torch.empty_like(q)
        scr = op.scratch(3, torch.float32)
        _lib.call("ancka_op_apply", op.struct(_lib.F32), q.data_ptr(), q.stride(0), 3,
                  out.data_ptr(), out.stride(0), scr.data_ptr(), _lib.stream())
        got = out[:, :3].double().cpu().numpy()
        ref = z[p + "apply"]
        rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
        assert rel <= 1e-5, (s, rel)
        # elementwise: 1e-5 relative to (|Z_ij| + rms(Z)); the f32 rounding of
        # M alone is ~6e-8 of max|M| before any cancellation in the average
        floor = np.sqrt(np.mean(ref ** 2))
        assert np.all(np.abs(got - ref) <= 1e-5 * (np.abs(ref) + floor)), s


def test_knn_matches_reference(golden_random):
    z = golden_random
    for s in _cases(z):
        p = f"s{s}_"
        X = load_x(z, p + "X")
        n = X.shape[0]
        K = min(4, n - 1)
        lists = ancka.knn_search_exact(X, K)
        assert knn_sets_match(lists.ids, z[p + "knn_ids"], X, K) == 0, s
        ok = z[p + "knn_ids"] >= 0
        assert np.array_equal(lists.ids >= 0, ok)


def test_knn_graph_bit_exact(golden_random):
    z = golden_random
    for s in _cases(z):
        p = f"s{s}_"
        ids = torch.from_numpy(z[p + "knn_ids"].astype(np.int32)).cuda()
        sc = torch.from_numpy(z[p + "knn_scores"]).cuda()
        A, P, zero = build_knn_graph_device(ids, sc, ids.shape[0])
        ak, pk = load_csr(z, p + "AK"), load_csr(z, p + "PK")
        a_mine, p_mine = A.to_scipy(), P.to_scipy()
        assert np.array_equal(a_mine.indptr, ak.indptr) and np.array_equal(a_mine.indices, ak.indices)
        np.testing.assert_array_equal(a_mine.data, ak.data)
        np.testing.assert_array_equal(p_mine.data, pk.data)


def test_init_mhc_step_discretize(golden_random):
    z = golden_random
    for s in _cases(z):
        p = f"s{s}_"
        op = _op_from_golden(z, p)
        n = op.n
        k = min(3, n)
        y0 = ancka.init_bcm(op, k, 5, 0.2)
        assert np.array_equal(y0.assignment, z[p + "init"]), s
        phi = ancka.calc_mhc(op, ancka.BcmMatrix(z[p + "lab"], k))
        assert abs(phi - float(z[p + "mhc"])) < 1e-13, s
        if p + "q0" in z:
            q1, r1 = ancka.orthogonal_step(op, z[p + "q0"], np.random.default_rng(s))
            np.testing.assert_allclose(q1, z[p + "q1"], atol=1e-10)
        d = ancka.discretize(z[p + "qd"])
        ref = z[p + "disc_labels"]
        assert ari(d.y.assignment, ref) >= 0.99 or np.array_equal(d.y.assignment, ref), s


@pytest.mark.parametrize("i", range(6))
def test_run_ancka_matches_reference(golden_runs, i):
    z, meta = golden_runs
    m = meta[i]
    p = f"r{i}_"
    S, X = load_csr(z, p + "S"), load_x(z, p + "X")
    net = (ancka.AttributedNetwork.hypergraph(S, X) if m["kind"] == "hypergraph"
           else ancka.AttributedNetwork.graph(S, X))
    params = ancka.ClusterParams(k=m["k"], knn_k=10, seed=m["seed"], t_a=m["t_a"],
                                 knn_mode=ancka.KnnMode.EXACT)
    res = ancka.run_ancka(net, params, early_stop=m["early_stop"])
    assert res.error is None, res.error
    a = ari(res.y.assignment, z[p + "labels"])
    assert a >= 0.99, (i, a, res.iterations, int(z[p + "iterations"]), res.stop_reason)
    assert abs(res.mhc - float(z[p + "mhc"])) < 1e-3


def canonical_knn(X, K):
    """Exact rational top-K for integer X: order (c/sqrt(a) desc, j asc),
    strictly positive only.  Ties are resolved with exact integer arithmetic."""
    Xd = X.toarray() if sp.issparse(X) else np.asarray(X)
    Xi = np.rint(Xd).astype(np.int64)
    a = (Xi * Xi).sum(axis=1)
    C = Xi @ Xi.T
    n = Xi.shape[0]
    ids = np.full((n, K), -1, dtype=np.int64)
    from functools import cmp_to_key
    for i in range(n):
        c = C[i].copy()
        c[i] = 0
        cand = np.flatnonzero(c > 0)
        if a[i] == 0 or cand.size == 0:
            continue
        key = c[cand] / np.sqrt(a[cand])
        order = cand[np.lexsort((cand, -key))][: 4 * K + 8]

        def cmp(x, y):
            lx, ly = int(c[x]) ** 2 * int(a[y]), int(c[y]) ** 2 * int(a[x])
            if lx != ly:
                return -1 if lx > ly else 1
            return -1 if x < y else 1
        best = sorted(order.tolist(), key=cmp_to_key(cmp))[:K]
        ids[i, : len(best)] = best
    return ids


@pytest.mark.parametrize("shape,n,words,K", [("cora", 1500, 18, 10), ("dblp", 2100, 20, 10),
                                             ("citeseer", 700, 32, 10), ("cora", 900, 18, 12),
                                             ("dblp", 800, 20, 16), ("cora", 600, 18, 24)])
def test_tensor_core_knn_exact(shape, n, words, K):
    """Every list-slot instantiation (K <= 10, 12, 16, 32) of the integer
    tcgen05 kernel against exact rational top-K."""
    from paper_2408_05459_b200 import synth
    from paper_2408_05459_b200.knn import integer_exact, knn_search_exact_device
    inst = synth.make(shape, seed=3, n=n, words=words)
    X = inst.X
    assert integer_exact(X) == 2
    ids_fp8, sc_fp8 = knn_search_exact_device(X, K, integer=2)
    ids_bf16, sc_bf16 = knn_search_exact_device(X, K, integer=1)
    ref = canonical_knn(X, K)
    got8 = ids_fp8.cpu().numpy().astype(np.int64)
    got16 = ids_bf16.cpu().numpy().astype(np.int64)
    assert np.array_equal(got8, ref), int((got8 != ref).any(axis=1).sum())
    assert np.array_equal(got16, ref)
    # scores: cosines of the selected pairs (f64, vs numpy f64 formula)
    Xd = X.toarray()
    nrm = np.linalg.norm(Xd, axis=1)
    ok = ref >= 0
    rows = np.repeat(np.arange(n)[:, None], K, axis=1)
    cos = np.zeros_like(sc_fp8.cpu().numpy())
    cos[ok] = (Xd[rows[ok]] * Xd[ref[ok]]).sum(1) / (nrm[rows[ok]] * nrm[ref[ok]])
    np.testing.assert_allclose(sc_fp8.cpu().numpy(), np.minimum(cos, 1.0), atol=1e-14)
    # the f64 CUDA-core path agrees up to exact ties at the K-th value
    ids_f64, _ = knn_search_exact_device(X, K, integer=0)
    assert knn_sets_match(ids_f64.cpu().numpy(), ref, X, K) == 0


@pytest.mark.parametrize("i", [0, 2, 3])
def test_fused_and_graph_paths_agree(golden_runs, i):
    """The fused cooperative orthogonal block and the per-step graph path give
    the same clustering (labels identical up to f32 rounding decisions)."""
    z, meta = golden_runs
    m = meta[i]
    p = f"r{i}_"
    S, X = load_csr(z, p + "S"), load_x(z, p + "X")
    net = (ancka.AttributedNetwork.hypergraph(S, X) if m["kind"] == "hypergraph"
           else ancka.AttributedNetwork.graph(S, X))
    params = ancka.ClusterParams(k=m["k"], knn_k=10, seed=m["seed"], t_a=m["t_a"],
                                 knn_mode=ancka.KnnMode.EXACT)
    a = ancka.run_ancka(net, params, early_stop=m["early_stop"], fused=True)
    b = ancka.run_ancka(net, params, early_stop=m["early_stop"], fused=False)
    assert ari(a.y.assignment, b.y.assignment) >= 0.99
    q = a.state.q
    assert np.abs(q.T @ q - np.eye(q.shape[1])).max() < 1e-5   # orthonormal block


@pytest.mark.parametrize("n,d,K,dup", [(3000, 100, 10, 0), (1100, 128, 10, 40), (700, 37, 20, 0),
                                       (257, 300, 5, 0)])
def test_real_valued_knn_certified(n, d, K, dup):
    """Real-valued attributes: tcgen05 split-bf16 candidates + f64 re-rank
    (level 0) must select the reference's sets (tie-aware, f64) and agree with
    the f64 CUDA-core scan (level -1); duplicated rows force uncertified rows
    through the fallback scan."""
    from paper_2408_05459_b200 import knn as kn
    rng = np.random.default_rng(n + d)
    lab = rng.integers(0, 7, n)
    mu = rng.normal(0.0, 2.0, size=(7, d))
    X = np.abs(mu[lab] + rng.standard_normal((n, d)))
    if dup:
        X[n - dup:] = X[0]                      # a tie group of dup+1 identical rows
        X[5] = 0.0                              # and a zero row
    ids0, sc0 = kn.knn_search_exact_device(X, K, integer=0)
    fallback = kn.LAST_STATS.get("fallback_rows")
    ids1, sc1 = kn.knn_search_exact_device(X, K, integer=-1)
    ref_ids, ref_sc = oc.knn_exact(X, K)
    a0 = ids0.cpu().numpy().astype(np.int64)
    a1 = ids1.cpu().numpy().astype(np.int64)
    assert knn_sets_match(a0, ref_ids, X, K) == 0
    assert knn_sets_match(a1, ref_ids, X, K) == 0
    np.testing.assert_allclose(sc0.cpu().numpy(), ref_sc, rtol=0, atol=1e-14)
    if dup:
        assert fallback > 0
        assert np.all(a0[5] == -1)
    else:
        assert fallback == 0


@pytest.mark.parametrize("path", ["device", "host"])
@pytest.mark.parametrize("n,k,noise", [(3000, 20, 0.25), (2500, 47, 0.2), (3000, 72, 0.1),
                                       (4000, 172, 0.05)])
def test_wide_discretize_matches_oracle(n, k, noise, path, monkeypatch):
    """Wide rounds against the oracle restatement of engine.py:221-263, forced
    here for every k: "device" = disc_wide_dev.cu's device-driven rounds (the
    path for 64 < k <= 192: tensor-core scoring with certified f64
    rescoring, incremental fixed-point totals, device Newton-Schulz polar
    factor, no host SVD); "host" = the host-driven rounds kept for k > 192
    (device scoring / accumulation, host SVD)."""
    from sklearn.metrics import adjusted_rand_score as ari_

    from paper_2408_05459_b200 import engine
    if path == "host":
        monkeypatch.setattr(engine, "WIDE_DISCRETIZE_K", 16)
    else:
        monkeypatch.setenv("ANCKA_DISC_WIDE_MIN", "8")
    rng = np.random.default_rng(k)
    lab = rng.integers(0, k, n)
    q = np.zeros((n, k))
    q[np.arange(n), lab] = 1.0
    q += noise * rng.standard_normal((n, k))
    q[7] = 0.0                                    # an all-zero row -> cluster 0
    q32 = q.astype(np.float32).astype(np.float64)   # the device sees f32 input
    d = ancka.discretize(q32)
    ref = oc.discretize(q32)
    assert ari_(ref["labels"], d.y.assignment) >= 0.99
    assert d.y.assignment[7] == ref["labels"][7]
    assert abs(d.objectives[-1] - ref["objs"][-1]) <= 1e-5 * max(1.0, abs(ref["objs"][-1]))


@pytest.mark.parametrize("k", [12, 20, 47, 62])
def test_discretize_kernel_windows(k):
    """Cooperative kernel for 8 < k <= 64 against the oracle, and bit-identical
    across the column offset of the block inside Q (the kernel stages an
    aligned column window) and across aligned / unaligned row strides
    (16-byte vs 4-byte staging)."""
    from paper_2408_05459_b200 import engine
    n = 3000
    rng = np.random.default_rng(100 + k)
    lab = rng.integers(0, k, n)
    q = np.zeros((n, k))
    q[np.arange(n), lab] = 1.0
    q += 0.25 * rng.standard_normal((n, k))
    q[5] = 0.0
    q32 = q.astype(np.float32).astype(np.float64)
    d = ancka.discretize(q32)
    ref = oc.discretize(q32)
    assert ari(ref["labels"], d.y.assignment) >= 0.99
    assert abs(d.objectives[-1] - ref["objs"][-1]) <= 1e-5 * max(1.0, abs(ref["objs"][-1]))
    base = None
    for col0 in (0, 1, 2, 3):
        for ld in (((col0 + k + 3) // 4) * 4, col0 + k + (1 if (col0 + k) % 4 == 0 else 0)):
            Q = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
            Q[:, col0:col0 + k] = torch.as_tensor(q32, dtype=torch.float32, device="cuda")
            labels = torch.empty(n, dtype=torch.int32, device="cuda")
            info = torch.zeros(8 + 2 * 100 + 2 * k * k, dtype=torch.float64, device="cuda")
            engine._discretize_device(Q, col0, k, 100, 1e-10, labels, info)
            got = (labels.cpu().numpy(), info[:8].cpu().numpy())
            if base is None:
                base = got
                assert ari(ref["labels"], got[0]) >= 0.99
                continue
            np.testing.assert_array_equal(got[0], base[0], err_msg=f"col0={col0} ld={ld}")
            np.testing.assert_array_equal(got[1], base[1], err_msg=f"col0={col0} ld={ld}")


def test_run_ancka_wide_k_matches_oracle():
    """k = 70 (c = 71 > 64): CholQR on wide blocks, the wide discretisation,
    MHC and init at large k, end to end against the oracle on a
    well-separated planted instance."""
    from sklearn.metrics import adjusted_rand_score as ari_
    rng = np.random.default_rng(11)
    k, per, d = 70, 60, 32
    n = k * per
    lab = np.repeat(np.arange(k), per)
    rows, cols = [], []
    for b in range(k):
        idx = np.arange(b * per, (b + 1) * per)
        e = rng.integers(0, per, size=(6 * per, 2))
        rows += list(idx[e[:, 0]])
        cols += list(idx[e[:, 1]])
    a = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))
    a = ((a + a.T) > 0).astype(np.float64)
    a.setdiag(0)
    a.eliminate_zeros()
    mu = rng.normal(0, 2.0, size=(k, d))
    X = np.abs(mu[lab] + 0.5 * rng.standard_normal((n, d)))
    net = ancka.AttributedNetwork.graph(sp.csr_matrix(a), X)
    params = ancka.ClusterParams(k=k, knn_k=10, seed=3, knn_mode=ancka.KnnMode.EXACT)
    res = ancka.run_ancka(net, params)
    assert res.error is None, res.error
    ref = oc.run({"kind": "graph", "S": sp.csr_matrix(a), "X": X}, k, knn_k=10, seed=3)
    assert ari_(ref["labels"], res.y.assignment) >= 0.99, (ari_(lab, res.y.assignment),
                                                           ari_(lab, ref["labels"]))
    assert abs(res.mhc - ref["mhc"]) < 1e-3


@pytest.mark.parametrize("i", range(2))
def test_run_ancka_multiplex_matches_reference(golden_multiplex, i):
    """multiplex networks (layer-averaged structural
    walk) end to end against the reference's golden runs."""
    from conftest import load_layers
    z, meta = golden_multiplex
    m = meta[i]
    p = f"m{i}_"
    net = ancka.AttributedNetwork.multiplex(load_layers(z, p), load_x(z, p + "X"))
    params = ancka.ClusterParams(k=m["k"], knn_k=10, seed=m["seed"], t_a=m["t_a"],
                                 knn_mode=ancka.KnnMode.EXACT)
    res = ancka.run_ancka(net, params, early_stop=m["early_stop"])
    assert res.error is None, res.error
    assert ari(res.y.assignment, z[p + "labels"]) >= 0.99
    assert abs(res.mhc - float(z[p + "mhc"])) < 1e-3


def _split_plan_torch(srp, krp, thr):
    """Torch restatement of the row-split plan (the former host-side builder)."""
    cost = (srp[1:] - srp[:-1]) + (krp[1:] - krp[:-1])
    order = torch.sort(cost, descending=True, stable=True).indices.to(torch.int32)
    long_rows = torch.nonzero(cost > thr).flatten().to(torch.int32)
    return order, long_rows


@pytest.mark.parametrize("hubs", [0, 7])
def test_row_split_plan_and_hub_rows(hubs):
    """plan.cu (cost order, long rows) against the torch restatement on a
    graph with `hubs` star nodes, and the f32 apply with hub rows summed by
    whole warps against the oracle (1e-5 relative)."""
    rng = np.random.default_rng(hubs)
    n = 3000
    a = sp.random(n, n, density=0.002, random_state=rng, format="csr")
    a.data[:] = 1.0
    for h in range(hubs):
        a[h * 11, rng.choice(n, 400, replace=False)] = 1.0
    a = ((a + a.T) > 0).astype(np.float64).tocsr()
    a.setdiag(0)
    a.eliminate_zeros()
    X = np.abs(rng.normal(size=(n, 8)))
    X[: n // 2] += 3.0 * np.eye(8)[0]
    net = ancka.AttributedNetwork.graph(a, X)
    params = ancka.ClusterParams(k=4, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
    from paper_2408_05459_b200.engine import build_pipeline
    op, _, _ = build_pipeline(net, params)
    split = op._split_plan()
    sf = op._f["p_n"]
    thr = max(op.LONG_ROW, op.HUB_FACTOR * (sf.nnz + op.p_k_dev.nnz) / n)
    order, long_rows = _split_plan_torch(sf.rowptr, op.p_k_dev.rowptr, thr)
    assert torch.equal(op._order.cpu(), order.cpu())
    assert split.n_long == long_rows.numel()
    assert hubs == 0 or split.n_long >= hubs
    if split.n_long:
        assert torch.equal(op._plan["long_rows"][: split.n_long].cpu(), long_rows.cpu())
    # the f32 apply (hub rows by warps) against the f64 oracle apply
    c = 5
    m = rng.standard_normal((n, c))
    q = padded(torch.from_numpy(m), torch.float32)
    out = torch.empty_like(q)
    scr = op.scratch(c, torch.float32)
    _lib.call("ancka_op_apply", op.struct(_lib.F32), q.data_ptr(), q.stride(0), c,
              out.data_ptr(), out.stride(0), scr.data_ptr(), _lib.stream())
    got = out[:, :c].double().cpu().numpy()
    ref = ancka.apply_joint_transition(op, m)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 1e-5, rel
    floor = np.sqrt(np.mean(ref ** 2))
    assert np.all(np.abs(got - ref) <= 1e-5 * (np.abs(ref) + floor))


def test_graph_replay_matches_eager():
    """The tau-block CUDA-graph path of the unfused loop (c > 8) replays the
    same kernels: labels and iteration count identical to eager launches."""
    rng = np.random.default_rng(21)
    k, per = 12, 80
    n = k * per
    lab = np.repeat(np.arange(k), per)
    rows, cols = [], []
    for b in range(k):
        idx = np.arange(b * per, (b + 1) * per)
        e = rng.integers(0, per, size=(5 * per, 2))
        rows += list(idx[e[:, 0]])
        cols += list(idx[e[:, 1]])
    a = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))
    a = ((a + a.T) > 0).astype(np.float64)
    a.setdiag(0)
    a.eliminate_zeros()
    X = np.abs(rng.normal(0, 2.0, size=(k, 16))[lab] + 0.7 * rng.standard_normal((n, 16)))
    net = ancka.AttributedNetwork.graph(sp.csr_matrix(a), X)
    params = ancka.ClusterParams(k=k, knn_k=10, seed=2, knn_mode=ancka.KnnMode.EXACT)
    r0 = ancka.run_ancka(net, params, use_graphs=False)
    r1 = ancka.run_ancka(net, params, use_graphs=True)
    assert r0.iterations == r1.iterations
    assert np.array_equal(r0.y.assignment, r1.y.assignment)
    assert r0.mhc == r1.mhc


@pytest.mark.parametrize("c", [12, 41, 48, 173])
def test_cholqr_wide_blocks(c):
    """Cholesky-QR of a tall block (engine.py:130-149) on the tensor-core
    Gram / apply kernels: Q matches the sign-fixed Householder QR of the same
    f32 block and is orthonormal (||Q^T Q - I||_F <= 1e-6 at c = 48 and 173
    for a block of condition ~10); ||Q - Q_prev||^2 is reported exactly."""
    from paper_2408_05459_b200._device import WORKSPACE, ld_for
    n = 200_000
    rng = np.random.default_rng(c)
    q0, _ = np.linalg.qr(rng.standard_normal((n, c)))
    r0 = np.triu(rng.standard_normal((c, c))) + 4.0 * np.eye(c) * np.sqrt(c)
    z = (q0 @ r0).astype(np.float32)
    ld = ld_for(c, torch.float32)
    Z = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
    Z[:, :c] = torch.from_numpy(z).cuda()
    Qp = torch.zeros_like(Z)
    Qp[:, :c] = torch.from_numpy(q0.astype(np.float32)).cuda()
    Qn = torch.full_like(Z, 7.0)
    G = torch.empty(c * (c + 1) // 2, dtype=torch.float64, device="cuda")
    stats = torch.tensor([0.0, 1.0, 0.0, 0.0], dtype=torch.float64, device="cuda")
    ws = WORKSPACE.get("test_orth", _lib.load().ancka_orth_workspace_size(None, c))
    _lib.call("ancka_gram_f32", Z.data_ptr(), n, ld, c, G.data_ptr(), ws.data_ptr(), ws.numel(),
              _lib.stream())
    zd = z.astype(np.float64)
    gfull = zd.T @ zd
    g_ref = gfull[np.triu_indices(c)]
    scale = np.sqrt(np.outer(np.diag(gfull), np.diag(gfull)))[np.triu_indices(c)]
    assert np.all(np.abs(G.cpu().numpy() - g_ref) <= 1e-6 * scale)   # f32-data Gram accuracy
    _lib.call("ancka_cholqr_apply_f32", Z.data_ptr(), Qp.data_ptr(), Qn.data_ptr(), n, ld, c,
              G.data_ptr(), stats.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    q = Qn[:, :c].double().cpu().numpy()
    assert np.all(Qn[:, c:].cpu().numpy() == 0.0)          # padding columns stay zero
    qr_, rr = np.linalg.qr(zd)
    qr_ = qr_ * np.where(np.diag(rr) < 0, -1.0, 1.0)
    assert np.abs(q - qr_).max() < 1e-5
    orth = np.linalg.norm(q.T @ q - np.eye(c))
    assert orth <= 1e-6, orth
    dq2 = float(((q - q0.astype(np.float32).astype(np.float64)) ** 2).sum())
    assert abs(float(stats[0]) - dq2) <= 1e-6 * max(dq2, 1.0)
    assert float(stats[2]) == 0.0
