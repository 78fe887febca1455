"""Full-size parity (BASELINE.json configs 3 and 4: MAG-PM- and Amazon2M-shaped)
through size-independent properties and sampled rows.

At these sizes the CPU reference cannot run the whole path (one f64 apply of
the Amazon2M operator takes 38 s, exact KNN ~34 h), so the device pipeline
(`build_pipeline`: validation, KNN, KNN graph, operator -- the code
`run_ancka` runs) is
checked where the answer is cheap to compute exactly:

* KNN: sampled query rows against an exact scan of all n keys -- exact
  rational order with index tie-break for the binary MAG-PM attributes
  (knn.py:83-98 made canonical), f64 cosines tie-aware (|s - s_K| <= 1e-12)
  for the continuous Amazon2M attributes (knn.py:112-140);
* operator: P_K rebuilt on the host from the device lists by the oracle
  (knn.py:294-324), the structural factors by the oracle from the raw input
  (walk.py:38-79, network.py:266-313); sampled rows of the f64 apply agree to
  1e-12 relative and of the f32 apply to 1e-5 (walk.py:177-190);
* the walk is row-stochastic: P 1 = 1 on every row (f32, 1e-5).
"""
from __future__ import annotations

import warnings

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import ancka_cpu as oc

pytestmark = pytest.mark.gpu
warnings.simplefilter("ignore")

ancka = pytest.importorskip("paper_2408_05459_b200")
from paper_2408_05459_b200 import _lib, synth  # noqa: E402
from paper_2408_05459_b200._device import padded  # noqa: E402

SAMPLE = 48


def _canonical_row(X, a, i, K):
    """Exact top-K of row i for integer X: (c/sqrt(a) desc, j asc), c > 0."""
    c = np.rint((X @ X[i].T).toarray().ravel()).astype(np.int64)
    c[i] = 0
    cand = np.flatnonzero(c > 0)
    if a[i] == 0 or cand.size == 0:
        return []
    key = c[cand] / np.sqrt(a[cand])
    order = cand[np.lexsort((cand, -key))][: 4 * K + 8]
    from functools import cmp_to_key

    def cmp(x, y):
        lx, ly = int(c[x]) ** 2 * int(a[y]), int(c[y]) ** 2 * int(a[x])
        if lx != ly:
            return -1 if lx > ly else 1
        return -1 if x < y else 1
    return sorted(order.tolist(), key=cmp_to_key(cmp))[:K]


def _real_row_ok(xn, i, got, K):
    """Tie-aware f64 check of one real-valued row."""
    s = xn @ xn[i]
    s[i] = -np.inf
    s = np.where(s > 0, s, -np.inf)
    ref = np.argsort(-s, kind="stable")[:K]
    ref = [j for j in ref.tolist() if np.isfinite(s[j])]
    a, b = set(got), set(ref)
    if a == b:
        return True
    if len(a) != len(b):
        return False
    kth = min(s[j] for j in b)
    return all(abs(s[j] - kth) <= 1e-12 for j in a ^ b)


def _sampled_apply(op, m, rows):
    """Rows `rows` of oracle.joint_apply (walk.py:177-190) without forming the
    full n x c product."""
    if op["kind"] == "hypergraph":
        s = op["p_v"][rows] @ (op["p_e"] @ m)
    else:
        s = op["p_n"][rows] @ m
    sl = np.isin(rows, op["selfloop"])
    s[sl] += m[rows[sl]]
    b = op["beta"][rows][:, None]
    return (1.0 - b) * s + b * (op["p_k"][rows] @ m)


@pytest.mark.parametrize("shape", ["magpm", "amazon2m"])
def test_full_size_knn_and_operator(shape):
    _lib.require_device()
    inst = synth.make(shape, seed=0)
    X, S = inst.X, inst.structure
    net = (ancka.AttributedNetwork.hypergraph(S, X) if inst.kind == "hypergraph"
           else ancka.AttributedNetwork.graph(S, X))
    params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
    op, g, _ = ancka.build_pipeline(net, params)
    n, K = X.shape[0], 10
    ids = g.neighbors.ids.astype(np.int64)
    scores = g.neighbors.scores.astype(np.float64)
    rng = np.random.default_rng(7)
    rows = np.sort(rng.choice(n, SAMPLE, replace=False))

    # --- KNN: sampled rows against an exact scan of every key
    if sp.issparse(X):
        Xc = X.tocsr()
        a = np.rint(np.asarray(Xc.multiply(Xc).sum(axis=1)).ravel()).astype(np.int64)
        for i in rows:
            ref = _canonical_row(Xc, a, int(i), K)
            got = [j for j in ids[i].tolist() if j >= 0]
            assert got == ref, (shape, int(i), got, ref)
    else:
        xn = np.asarray(X, dtype=np.float64)
        nrm = np.linalg.norm(xn, axis=1)
        xn = xn / np.where(nrm > 0, nrm, 1.0)[:, None]
        bad = [int(i) for i in rows if not _real_row_ok(xn, int(i), [j for j in ids[i].tolist() if j >= 0], K)]
        assert not bad, (shape, bad)
        del xn

    # --- operator: oracle factors from the raw input and the device lists
    onet = oc.clean_network({"kind": inst.kind, "S": S, "X": X})
    p_k, knn_zero = oc.row_stochastic(oc.knn_adjacency(ids, scores))
    ref_op = oc.make_operator(onet, p_k, knn_zero, alpha=params.alpha, beta=params.beta,
                              gamma=params.gamma)
    np.testing.assert_array_equal(op.beta, ref_op["beta"])
    c = inst.k + 1
    m = rng.standard_normal((n, c))
    ref = _sampled_apply(ref_op, m, rows)
    got64 = ancka.apply_joint_transition(op, m)[rows]
    rel64 = np.linalg.norm(got64 - ref) / np.linalg.norm(ref)
    assert rel64 <= 1e-12, (shape, rel64)

    def apply32(block):
        q = padded(torch.from_numpy(block), torch.float32)
        out = torch.empty_like(q)
        scr = op.scratch(block.shape[1], torch.float32)
        _lib.call("ancka_op_apply", op.struct(_lib.F32), q.data_ptr(), q.stride(0), block.shape[1],
                  out.data_ptr(), out.stride(0), scr.data_ptr(), _lib.stream())
        return out[:, :block.shape[1]]

    got32 = apply32(m)[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    rel32 = np.linalg.norm(got32 - ref) / np.linalg.norm(ref)
    assert rel32 <= 1e-5, (shape, rel32)
    # row-stochastic walk: P 1 = 1 on every row
    ones = apply32(np.ones((n, 4)))
    dev = float((ones - 1.0).abs().max())
    assert dev <= 1e-5, (shape, dev)
