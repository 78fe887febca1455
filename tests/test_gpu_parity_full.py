"""Full-size parity on the shapes the CPU can finish, and the reference's
edge cases (needs a B200).

* Cora (graph, n=2,708, d=1,433, K=10), Citeseer (hypergraph, n=3,312,
  d=3,703) and DBLP (hypergraph, n=41,302, d=1,425) at their full
  BASELINE.json sizes.  Both sides use the same neighbour lists: the GPU run
  writes the reference's `.aknn` cache (knn.py:327-382; f32 scores), a
  second GPU run reads it, and the oracle is given the same lists (the
  reference's own injection hook, engine.py:320-327).  Asserted: labels at
  ARI >= 0.99, equal iteration counts and stop reasons, |dphi| <= 1e-6;
  plus a lockstep run (early_stop=False, t_a = the oracle's count).
* SPEC.md edge cases: k = 1 -> phi = 0.4096, two isolated
  cliques with beta = 0 -> 0.4096, k = n does not crash
  (SPEC.md:345), planted Y0 R0 recovery >= 48/50,
  determinism, calc_mhc = brute_mhc_oracle within 1e-9
  (SPEC.md:538), and a discretisation input whose argmax leaves a column
  empty, so the in-loop reseed (engine.py:162-180) fires in the
  cooperative kernel and in the wide (k > 64) path.
"""
from __future__ import annotations

import warnings

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import load_csr, oracle_net, random_seeds
from oracle import ancka_cpu as oc

pytestmark = pytest.mark.gpu
warnings.simplefilter("ignore")

ancka = pytest.importorskip("paper_2408_05459_b200")
from paper_2408_05459_b200 import synth  # noqa: E402
from paper_2408_05459_b200.knn import cache_key, load_neighbor_cache  # noqa: E402

PHI_TOL = 1e-6


def ari(a, b):
    from sklearn.metrics import adjusted_rand_score
    return adjusted_rand_score(a, b)


def _net(inst):
    if inst.kind == "hypergraph":
        return ancka.AttributedNetwork.hypergraph(inst.structure, inst.X)
    return ancka.AttributedNetwork.graph(inst.structure, inst.X)


@pytest.mark.parametrize("shape", ["cora", "citeseer", "dblp"])
def test_full_shape_parity(shape, tmp_path):
    inst = synth.make(shape, seed=0)
    net = _net(inst)
    params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
    first = ancka.run_ancka(net, params, knn_cache_dir=tmp_path)        # writes the .aknn
    assert first.error is None, first.error
    path = tmp_path / f"{cache_key(net.attributes, 10, ancka.KnnMode.EXACT)}.aknn"
    lists, _ = load_neighbor_cache(path)
    res = ancka.run_ancka(net, params, knn_cache_dir=tmp_path)          # reads it
    assert res.error is None, res.error
    onet = {"kind": inst.kind, "S": inst.structure, "X": inst.X}
    ref = oc.run(onet, inst.k, knn_k=10, seed=0, knn=(lists.ids, lists.scores))
    a = ari(ref["labels"], res.y.assignment)
    info = (shape, a, res.iterations, ref["iterations"], res.stop_reason, ref["stop_reason"],
            res.mhc, ref["mhc"])
    assert a >= 0.99, info
    assert res.iterations == ref["iterations"], info
    assert res.stop_reason == ref["stop_reason"], info
    assert abs(res.mhc - ref["mhc"]) <= PHI_TOL, info
    # the run on the GPU's own lists (f64 scores) lands on the same clustering
    assert ari(first.y.assignment, res.y.assignment) >= 0.99
    # lockstep: no early stop, the oracle's iteration budget
    t_a = int(ref["iterations"])
    p2 = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, t_a=t_a, knn_mode=ancka.KnnMode.EXACT)
    res2 = ancka.run_ancka(net, p2, knn_cache_dir=tmp_path, early_stop=False)
    ref2 = oc.run(onet, inst.k, knn_k=10, seed=0, t_a=t_a, early_stop=False,
                  knn=(lists.ids, lists.scores))
    assert res2.iterations == ref2["iterations"] == t_a
    assert ari(ref2["labels"], res2.y.assignment) >= 0.99
    assert abs(res2.mhc - ref2["mhc"]) <= PHI_TOL, (res2.mhc, ref2["mhc"])


def _ring_graph(n, extra=0, seed=0):
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    rows, cols = [i, (i + 1) % n], [(i + 1) % n, i]
    if extra:
        u, v = rng.integers(0, n, extra), rng.integers(0, n, extra)
        keep = u != v
        rows += [u[keep], v[keep]]
        cols += [v[keep], u[keep]]
    a = sp.csr_matrix((np.ones(sum(r.size for r in rows)),
                       (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    return ((a + a.T) > 0).astype(np.float64).tocsr()


def test_mhc_single_cluster_is_04096():
    """one cluster, alpha = 0.2, gamma = 3, every row fully
    stochastic -> phi = 1 - 0.2 (1 + 0.8 + 0.64 + 0.512) = 0.4096."""
    n = 200
    a = _ring_graph(n, extra=300)
    X = np.abs(np.random.default_rng(1).normal(size=(n, 6))) + 0.1   # no empty KNN row
    net = ancka.AttributedNetwork.graph(a, X)
    op, _, _ = ancka.build_pipeline(net, ancka.ClusterParams(k=1, knn_k=5))
    phi = ancka.calc_mhc(op, ancka.BcmMatrix(np.zeros(n, dtype=np.int64), 1))
    assert abs(phi - 0.4096) < 1e-12, phi


def test_mhc_two_cliques_beta0():
    """two isolated cliques as two clusters, beta = 0 -> 0.4096."""
    n = 8
    a = np.zeros((n, n))
    a[:4, :4] = 1.0
    a[4:, 4:] = 1.0
    np.fill_diagonal(a, 0.0)
    X = np.abs(np.random.default_rng(2).normal(size=(n, 3))) + 0.1
    net = ancka.AttributedNetwork.graph(sp.csr_matrix(a), X)
    op, _, _ = ancka.build_pipeline(net, ancka.ClusterParams(k=2, knn_k=3, beta=0.0))
    y = ancka.BcmMatrix(np.array([0, 0, 0, 0, 1, 1, 1, 1]), 2)
    assert abs(ancka.calc_mhc(op, y) - 0.4096) < 1e-12
    assert abs(ancka.brute_mhc_oracle(op, y) - 0.4096) < 1e-12


@pytest.mark.parametrize("n", [5, 8, 12])
def test_k_equals_n_does_not_crash(n):
    """k = n; the discretised block has n - 1 columns and the
    post-pass repair (engine.py:266-288) fills the missing cluster.  Same
    outcome as the oracle (labels, phi, iterations, error)."""
    a = _ring_graph(n, extra=n, seed=n)
    X = np.abs(np.random.default_rng(n).normal(size=(n, 4))) + 0.05
    net = ancka.AttributedNetwork.graph(a, X)
    params = ancka.ClusterParams(k=n, knn_k=2, seed=0, t_a=40, knn_mode=ancka.KnnMode.EXACT)
    res = ancka.run_ancka(net, params)
    ref = oc.run({"kind": "graph", "S": a, "X": X}, n, knn_k=2, seed=0, t_a=40)
    assert (res.error is None) == (ref["error"] is None), (res.error, ref["error"])
    assert res.iterations == ref["iterations"]
    assert np.array_equal(np.sort(np.bincount(res.y.assignment, minlength=n)),
                          np.sort(np.bincount(ref["labels"], minlength=n)))
    assert abs(res.mhc - ref["mhc"]) <= PHI_TOL


def test_planted_rotation_recovery():
    """Q = Y0 R0 for a random orthogonal R0 and a balanced
    Y0 (n = 12, k = 3) is recovered up to column permutation in >= 48 of 50
    seeds (the reference recovers 50/50)."""
    ok = 0
    for seed in range(50):
        rng = np.random.default_rng(seed)
        lab = rng.permutation(np.repeat(np.arange(3), 4))
        y = np.zeros((12, 3))
        y[np.arange(12), lab] = 0.5                     # 1/sqrt(4)
        r0, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        d = ancka.discretize(y @ r0)
        ref = oc.discretize(y @ r0)
        assert ari(d.y.assignment, ref["labels"]) == 1.0, seed
        ok += int(ari(d.y.assignment, lab) == 1.0)
    assert ok >= 48, ok


def test_determinism_byte_identical():
    """the same seed twice gives byte-identical assignments
    (no float atomics; fixed-order or integer reductions only)."""
    inst = synth.make("dblp", seed=4, n=6000)
    net = _net(inst)
    params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=7, knn_mode=ancka.KnnMode.EXACT)
    r1 = ancka.run_ancka(net, params)
    r2 = ancka.run_ancka(net, params)
    assert r1.y.assignment.tobytes() == r2.y.assignment.tobytes()
    assert r1.mhc == r2.mhc and r1.iterations == r2.iterations
    assert [v for _, v in r1.state.mhc_history] == [v for _, v in r2.state.mhc_history]


def test_dense_oracles_match_golden(golden_random):
    """walk.py:193-242 on the device: dense_transition equals the reference's
    dense P (1e-12), brute_mhc_oracle equals the reference's (1e-9)
    and the iterative calc_mhc (1e-9)."""
    from test_gpu_parity import _op_from_golden
    z = golden_random
    for s in [s for s in random_seeds(z) if not bool(z[f"s{s}_skip"])]:
        p = f"s{s}_"
        op = _op_from_golden(z, p)
        np.testing.assert_allclose(ancka.dense_transition(op), z[p + "dense"], atol=1e-12)
        y = ancka.BcmMatrix(z[p + "lab"], min(3, op.n))
        b = ancka.brute_mhc_oracle(op, y)
        assert abs(b - float(z[p + "mhc_brute"])) < 1e-9, s
        assert abs(b - ancka.calc_mhc(op, y)) < 1e-9, s
        m = z[p + "M"]
        onet = oc.clean_network(oracle_net(z, p))
        pk = load_csr(z, p + "PK")
        zero = np.asarray(pk.sum(axis=1)).ravel() == 0
        oop = oc.make_operator(onet, pk, zero, 0.2, float(z[p + "beta"]), int(z[p + "gamma"]))
        np.testing.assert_array_equal(np.sort(oop["selfloop"]), op.selfloop)
        np.testing.assert_allclose(ancka.apply_structure(op, m), oc.structure_apply(oop, m),
                                   rtol=0, atol=1e-15)


def _starved_block(n, k, seed):
    """Rows one-hot on columns 0..k-2 plus noise, column k-1 never the row
    maximum: the first rounding round leaves cluster k-1 empty."""
    rng = np.random.default_rng(seed)
    lab = rng.integers(0, k - 1, n)
    q = np.zeros((n, k))
    q[np.arange(n), lab] = 1.0
    q[:, : k - 1] += 0.2 * rng.standard_normal((n, k - 1))
    q[:, k - 1] = -2.0 + 0.1 * rng.standard_normal(n)      # starved column
    return q.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("k,wide", [(6, None), (20, None), (47, None), (20, "host"),
                                    (20, "device"), (47, "device"), (80, "device")])
def test_empty_column_reseed(k, wide, monkeypatch):
    """engine.py:162-180: the in-loop reseed moves the node with the largest
    second-best score (from clusters of size >= 2) into the empty column.
    Device labels and objective against the oracle; the reseeded cluster is
    populated on both sides.  wide: the host-driven wide rounds, or the
    device-driven wide path (disc_wide_dev.cu) forced on narrower blocks."""
    from paper_2408_05459_b200 import engine
    if wide == "host":
        monkeypatch.setattr(engine, "WIDE_DISCRETIZE_K", 16)
    elif wide == "device":
        monkeypatch.setenv("ANCKA_DISC_WIDE_MIN", "8")
    q = _starved_block(1500, k, k)
    ref = oc.discretize(q)
    d = ancka.discretize(q)
    assert (np.bincount(ref["labels"], minlength=k) > 0).all()
    assert np.array_equal(d.y.assignment, ref["labels"]) or ari(d.y.assignment, ref["labels"]) >= 0.999
    assert (np.bincount(d.y.assignment, minlength=k) > 0).all()
    assert abs(d.objectives[-1] - ref["objs"][-1]) <= 1e-5 * max(1.0, abs(ref["objs"][-1]))


def test_planted_partition_end_to_end():
    """SPEC.md:345, 545 (criterion 12 restated): disconnected planted blocks
    with block-indicator attributes -> ACC = ARI = 1.0 for graphs and
    hypergraphs over several seeds."""
    for seed in range(4):
        rng = np.random.default_rng(seed)
        k, per = 4, 30
        n = k * per
        lab = np.repeat(np.arange(k), per)
        X = np.zeros((n, 2 * k))
        X[np.arange(n), 2 * lab] = 1.0
        X[np.arange(n), 2 * lab + 1] = 1.0
        rows, cols = [], []
        for b in range(k):
            idx = np.arange(b * per, (b + 1) * per)
            e = rng.integers(0, per, size=(4 * per, 2))
            rows += list(idx[e[:, 0]])
            cols += list(idx[e[:, 1]])
        a = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))
        a = ((a + a.T) > 0).astype(np.float64).tolil()
        a.setdiag(0)
        a = a.tocsr()
        a.eliminate_zeros()
        h_rows, h_cols = [], []
        for e in range(2 * n):
            b = e % k
            mem = rng.choice(np.arange(b * per, (b + 1) * per), size=3, replace=False)
            h_rows += [e] * 3
            h_cols += list(mem)
        h = sp.csr_matrix((np.ones(len(h_rows)), (h_rows, h_cols)), shape=(2 * n, n))
        for net in (ancka.AttributedNetwork.graph(a, X), ancka.AttributedNetwork.hypergraph(h, X)):
            res = ancka.run_ancka(net, ancka.ClusterParams(k=k, knn_k=10, seed=seed))
            assert res.error is None
            assert ari(res.y.assignment, lab) == 1.0, (seed, net.kind)


def test_cli_run_binary_matches_in_memory(tmp_path):
    """f3: `python -m ... run` over a binary directory (mapped arrays,
    validated in place) returns the in-memory run's labels and phi."""
    import json

    from paper_2408_05459_b200 import cli
    assert cli.main(["gen", "--shape", "dblp", "--n", "3000", "--out", str(tmp_path / "d")]) == 0
    out = tmp_path / "r.json"
    rc = cli.main(["run", "--net-dir", str(tmp_path / "d"), "-k", "6", "--knn-k", "10",
                   "--knn-mode", "exact", "-o", str(out)])
    assert rc == cli.EXIT_OK
    doc = json.loads(out.read_text())
    inst = synth.make("dblp", seed=0, n=3000)
    ref = ancka.run_ancka(_net(inst), ancka.ClusterParams(k=6, knn_k=10, seed=0,
                                                          knn_mode=ancka.KnnMode.EXACT))
    assert np.array_equal(np.asarray(doc["assignment"]), ref.y.assignment)
    assert doc["mhc"] == ref.mhc and doc["iterations"] == ref.iterations
    assert doc["stop_reason"] == ref.stop_reason and "load_ms" in doc
    assert set(doc["metrics"]) == {"ari", "nmi"}
