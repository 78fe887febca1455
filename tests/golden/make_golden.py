"""Freeze outputs of the REFERENCE package as golden fixtures.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference (`/root/reference/pkg/src/ancka`) and its
own test-fixture builders (`/root/reference/pkg/tests/conftest.py`), runs the
hot-path functions on seeded inputs and writes small .npz files next to this
script.  The oracle (`oracle/ancka_cpu.py`) is pinned against these files by
`tests/test_oracle_golden.py`; the CUDA path is then checked against the
oracle and against these files.  Nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import json
import sys
import warnings
from pathlib import Path

import numpy as np
import scipy.sparse as sp

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, str(HERE.parents[1]))

import ancka  # noqa: E402  (the reference)
from ancka import engine, knn, walk  # noqa: E402
from conftest import make_random_instance, random_membership  # noqa: E402

from paper_2408_05459_b200 import synth  # noqa: E402

warnings.simplefilter("ignore")


def _csr(prefix, m, out):
    m = sp.csr_matrix(m)
    out[prefix + "_indptr"] = m.indptr.astype(np.int64)
    out[prefix + "_indices"] = m.indices.astype(np.int64)
    out[prefix + "_data"] = m.data.astype(np.float64)
    out[prefix + "_shape"] = np.asarray(m.shape, dtype=np.int64)


def _x(prefix, x, out):
    if sp.issparse(x):
        _csr(prefix + "_csr", x, out)
    else:
        out[prefix + "_dense"] = np.asarray(x, dtype=np.float64)


def spec_examples():
    out = {}
    x = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    nl = ancka.knn_search_exact(x, 1)
    out["ex1_X"] = x
    out["ex1_ids"], out["ex1_scores"] = nl.ids, nl.scores
    g = ancka.build_knn_adjacency(nl, x)
    out["ex1_AK"] = g.adjacency.toarray()
    p, z = ancka.knn_transition(g)
    out["ex1_PK"] = p.toarray()
    x2 = np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0], [1.0, 0.1]])
    nl2 = ancka.knn_search_exact(x2, 2)
    out["ex2_X"], out["ex2_ids"], out["ex2_scores"] = x2, nl2.ids, nl2.scores
    np.savez_compressed(HERE / "spec_examples.npz", **out)


def random_instances(n_seeds=60):
    """Per-op outputs on conftest.make_random_instance(seed) (conftest.py:69-82)."""
    out = {}
    for seed in range(n_seeds):
        op, g, net = make_random_instance(seed)
        p = f"s{seed}_"
        rng = np.random.default_rng(1000 + seed)
        out[p + "kind"] = np.array(net.kind.value)
        out[p + "directed"] = np.array(bool(net.directed))
        out[p + "beta"] = np.array((0.0, 0.5, 1.0)[(seed // 3) % 3])   # conftest.py:80
        out[p + "beta_vec"] = op.beta
        out[p + "gamma"] = np.array(op.gamma)
        out[p + "skip"] = np.array(False)
        if net.kind is ancka.NetworkKind.MULTIPLEX:
            out[p + "n_layers"] = np.array(len(net.layers))
            for li, a in enumerate(net.layers):
                _csr(p + f"L{li}", a, out)
        else:
            struct = net.incidence if net.kind is ancka.NetworkKind.HYPERGRAPH else net.adjacency
            _csr(p + "S", struct, out)
        _x(p + "X", net.attributes, out)
        out[p + "knn_ids"] = g.neighbors.ids
        out[p + "knn_scores"] = g.neighbors.scores
        _csr(p + "AK", g.adjacency, out)
        _csr(p + "PK", op.p_k, out)
        out[p + "selfloop"] = op.selfloop
        n = op.n
        m = rng.standard_normal((n, 3))
        out[p + "M"] = m
        out[p + "apply"] = walk.apply_joint_transition(op, m)
        out[p + "apply_t"] = walk.apply_structure_rowvec(op, m.T.copy())
        out[p + "dense"] = walk.dense_transition(op)
        k = int(min(3, n))
        out[p + "init"] = engine.init_bcm(op, k, 5, 0.2).assignment
        lab = random_membership(rng, n, k)
        out[p + "lab"] = lab
        out[p + "mhc"] = np.array(engine.calc_mhc(op, ancka.BcmMatrix(lab, k)))
        out[p + "mhc_brute"] = np.array(walk.brute_mhc_oracle(op, ancka.BcmMatrix(lab, k)))
        q0 = np.linalg.qr(rng.standard_normal((n, k + 1)))[0] if n > k else None
        if q0 is not None:
            out[p + "q0"] = q0
            q1, r1 = engine.orthogonal_step(op, q0, np.random.default_rng(seed))
            out[p + "q1"], out[p + "r1"] = q1, r1
        qd = rng.standard_normal((n, k))
        d = engine.discretize(qd)
        out[p + "qd"] = qd
        out[p + "disc_labels"] = d.y.assignment
        out[p + "disc_objs"] = np.asarray(d.objectives)
        out[p + "disc_scores"] = d.scores
    np.savez_compressed(HERE / "random_instances.npz", **out)


def _net(inst):
    if inst.kind == "graph":
        return ancka.AttributedNetwork.graph(inst.structure, inst.X)
    return ancka.AttributedNetwork.hypergraph(inst.structure, inst.X)


RUNS = [  # (shape, seed, n, p_in, words, early_stop)
    ("cora", 0, 300, 0.8, 18, True),
    ("cora", 1, 400, 0.5, 8, True),
    ("citeseer", 0, 300, 0.8, 32, True),
    ("dblp", 2, 500, 0.8, 20, True),
    ("amazon2m", 0, 300, 0.8, None, True),
    ("cora", 3, 250, 0.8, 18, False),
]


def multiplex_split(inst, seed):
    """Two-layer multiplex from a graph instance: each edge goes to layer 0 or
    1 at random, and each layer gets a few extra intra-block edges."""
    rng = np.random.default_rng(seed)
    a = sp.triu(sp.csr_matrix(inst.structure), 1).tocoo()
    side = rng.random(a.nnz) < 0.55
    n = inst.structure.shape[0]
    layers = []
    for want in (True, False):
        keep = side == want
        r, c = a.row[keep], a.col[keep]
        extra = rng.integers(0, n, size=(n // 4, 2))
        same = inst.labels[extra[:, 0]] == inst.labels[extra[:, 1]]
        r = np.concatenate([r, extra[same, 0]])
        c = np.concatenate([c, extra[same, 1]])
        m = sp.csr_matrix((np.ones(r.size), (r, c)), shape=(n, n))
        m = ((m + m.T) > 0).astype(np.float64)
        m.setdiag(0)
        m.eliminate_zeros()
        layers.append(sp.csr_matrix(m))
    return layers


MPX_RUNS = [  # (shape, seed, n, early_stop)
    ("cora", 5, 300, True),
    ("amazon2m", 6, 300, True),
]


def end_to_end_multiplex():
    out, meta = {}, []
    for i, (shape, seed, n, early) in enumerate(MPX_RUNS):
        inst = synth.make(shape, seed=seed, n=n)
        layers = multiplex_split(inst, seed)
        p = f"m{i}_"
        out[p + "n_layers"] = np.array(len(layers))
        for li, a in enumerate(layers):
            _csr(p + f"L{li}", a, out)
        _x(p + "X", inst.X, out)
        params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=seed, knn_mode=ancka.KnnMode.EXACT)
        net = ancka.AttributedNetwork.multiplex(layers, inst.X)
        res = ancka.run_ancka(net, params, early_stop=early)
        out[p + "labels"] = res.y.assignment
        out[p + "mhc"] = np.array(res.mhc)
        out[p + "iterations"] = np.array(res.iterations)
        out[p + "planted"] = inst.labels
        meta.append({"shape": shape, "seed": seed, "n": n, "kind": "multiplex",
                     "n_layers": len(layers), "k": inst.k, "stop_reason": res.stop_reason,
                     "early_stop": early, "t_a": params.t_a,
                     "ari_vs_planted": float(ancka.ari(inst.labels, res.y.assignment))})
    np.savez_compressed(HERE / "multiplex.npz", **out)
    (HERE / "multiplex.json").write_text(json.dumps(meta, indent=1))


def end_to_end():
    out, meta = {}, []
    for i, (shape, seed, n, p_in, words, early) in enumerate(RUNS):
        inst = synth.make(shape, seed=seed, n=n, p_in=p_in, words=words)
        p = f"r{i}_"
        _csr(p + "S", inst.structure, out)
        _x(p + "X", inst.X, out)
        params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=seed,
                                     knn_mode=ancka.KnnMode.EXACT,
                                     t_a=60 if not early else 1000)
        res = ancka.run_ancka(_net(inst), params, early_stop=early)
        out[p + "labels"] = res.y.assignment
        out[p + "mhc"] = np.array(res.mhc)
        out[p + "iterations"] = np.array(res.iterations)
        out[p + "history"] = np.asarray(res.state.mhc_history, dtype=np.float64)
        out[p + "knn_ids"] = res.knn.neighbors.ids
        out[p + "knn_scores"] = res.knn.neighbors.scores
        out[p + "q"] = res.state.q
        out[p + "planted"] = inst.labels
        meta.append({"shape": shape, "seed": seed, "n": n, "p_in": p_in, "words": words,
                     "kind": inst.kind, "k": inst.k, "stop_reason": res.stop_reason,
                     "early_stop": early, "t_a": params.t_a,
                     "ari_vs_planted": float(ancka.ari(inst.labels, res.y.assignment))})
    np.savez_compressed(HERE / "end_to_end.npz", **out)
    (HERE / "end_to_end.json").write_text(json.dumps(meta, indent=1))


def aknn_cache():
    """The .aknn neighbour-cache wire format (knn.py:327-382): files written
    by the reference's save_neighbor_cache for its own exact lists, and its
    cache_key for each input, so the B200 reader/writer/key are pinned."""
    rng = np.random.default_rng(5)
    xs = {
        "binary_csr": sp.csr_matrix((rng.random((300, 120)) < 0.06).astype(np.float64)),
        "dense": np.abs(rng.normal(size=(250, 16))),
    }
    out, meta = {}, {}
    for name, x in xs.items():
        _x(name, x, out)
        nl = knn.knn_search_exact(x, 7)
        f = HERE / f"aknn_{name}.aknn"
        knn.save_neighbor_cache(f, nl, ancka.KnnMode.EXACT)
        meta[name] = {"K": 7, "file": f.name,
                      "key_exact": knn.cache_key(x, 7, ancka.KnnMode.EXACT),
                      "key_approx": knn.cache_key(x, 7, ancka.KnnMode.APPROX)}
    np.savez_compressed(HERE / "aknn.npz", **out)
    (HERE / "aknn.json").write_text(json.dumps(meta, indent=1))


def approx_knn():
    """Approximate KNN (knn.py:156-280): the reference's knn_search_approx
    lists, its trained centroids (knn._train_ivf on its own f32 copy) and
    the escalation count read from its warnings, on three seeded inputs --
    continuous dense, binary sparse, and a forced escalation."""
    cases = {
        "dense": (synth.make("amazon2m", seed=0, n=3000).X, 10, 0.9, None, 0),
        "binary": (synth.make("citeseer", seed=1, n=2500).X, 10, 0.9, None, 1),
        "escalate": (np.abs(np.random.default_rng(3).normal(size=(2000, 16))), 8, 0.99, 1, 2),
    }
    out, meta = {}, {}
    for name, (x, K, target, nprobe, seed) in cases.items():
        _x(name + "_X", x, out)
        with warnings.catch_warnings(record=True) as rec:
            warnings.simplefilter("always")
            nl = knn.knn_search_approx(x, K, recall_target=target, seed=seed, nprobe=nprobe)
        esc = sum("escalating probes" in str(w.message) for w in rec)
        xn, _ = knn._normalize_rows(x)
        if sp.issparse(xn):
            xn = np.asarray(xn.todense())
        xn = np.ascontiguousarray(xn, dtype=np.float32)
        n = xn.shape[0]
        nlist = int(min(4096, max(8, round(np.sqrt(n)))))
        out[name + "_centroids"] = knn._train_ivf(xn, nlist, seed)
        out[name + "_ids"], out[name + "_scores"] = nl.ids, nl.scores
        meta[name] = {"K": K, "recall_target": target, "nprobe": nprobe, "seed": seed,
                      "nlist": nlist, "escalations": esc}
    np.savez_compressed(HERE / "approx.npz", **out)
    (HERE / "approx.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    which = set(sys.argv[1:])
    if not which or "spec" in which:
        spec_examples()
    if not which or "random" in which:
        random_instances()
    if not which or "e2e" in which:
        end_to_end()
    if not which or "multiplex" in which:
        end_to_end_multiplex()
    if not which or "aknn" in which:
        aknn_cache()
    if not which or "approx" in which:
        approx_knn()
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)
