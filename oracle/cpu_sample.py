"""Bounded-sample timing of the reference CPU path -- BENCH INFRASTRUCTURE ONLY.

At the Amazon2M / MAG-PM shapes a full CPU clustering takes tens of hours
(exact KNN alone ~34 h at Amazon2M), so the CPU side of
`bench.py` follows BASELINE.md §4: time each reference kernel of the path
once on a bounded sample of the same instance and assemble a full-run
estimate from the kernel counts of a real run (iterations, discretisation
calls and rounds).  Every timed kernel is the oracle restatement
(oracle/ancka_cpu.py) of the reference function cited beside it.

Sampling (`row_frac` < 1): the per-row kernels (operator apply rows, QR,
discretisation rounds) are timed on a random row subset and scaled by
1/row_frac -- each is linear in the number of rows; the hypergraph P_E
pass is always timed in full.  Exact KNN is timed on `knn_rows` query rows
against all n keys and scaled by n / knn_rows (labelled "extrapolated").
"""
from __future__ import annotations

import os
import time

import numpy as np
import scipy.sparse as sp

from . import ancka_cpu as oc


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _planted_knn_lists(labels: np.ndarray, rows: np.ndarray, K: int, seed: int = 0):
    """KNN lists standing in for the exact ones when building the CPU
    operator rows: K distinct random same-block neighbours per row with
    positive scores.  The timed SpMM depends on nnz and layout only."""
    rng = np.random.default_rng(seed)
    order = np.argsort(labels, kind="stable")
    bounds = np.searchsorted(labels[order], np.arange(labels.max() + 2))
    lo, hi = bounds[labels[rows]], bounds[labels[rows] + 1]
    ids = order[lo[:, None] + (rng.random((rows.size, K)) * (hi - lo)[:, None]).astype(np.int64)]
    scores = 0.5 + 0.5 * rng.random((rows.size, K))
    return ids, scores


def _timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return time.perf_counter() - t0, out


def sample_timings(inst, K: int, row_frac: float = 1.0, knn_rows: int = 1000,
                   seed: int = 0, alpha: float = oc.ALPHA, beta: float = oc.BETA) -> dict:
    """Seconds per call of each reference kernel on the workload (scaled to
    all n rows when sampled)."""
    from threadpoolctl import threadpool_limits

    n = inst.X.shape[0]
    k = inst.k
    c = k + 1
    rng = np.random.default_rng(seed)
    rows = (np.arange(n) if row_frac >= 1.0 else
            np.sort(rng.choice(n, size=max(64, int(round(n * row_frac))), replace=False)))
    f = rows.size / n
    out = {"rows": int(rows.size), "row_frac": f, "knn_rows": int(knn_rows)}
    with threadpool_limits(limits=cores()):
        # exact KNN (knn.py:112-140) on query rows spread over the instance
        # (the one-off row normalisation is timed once, the scan per row)
        q = np.linspace(0, n - 1, knn_rows).astype(np.int64)
        t_norm, xnn = _timed(lambda: oc.unit_rows(inst.X))
        t, _ = _timed(lambda: oc.knn_rows(inst.X, q, K, normalized=xnn))
        out["knn_s"] = t_norm + t * n / knn_rows
        del xnn

        # operator rows (walk.py:38-79, knn.py:294-324): row normalisation is
        # row-local, so the sampled rows of P are the sampled rows of the
        # normalised sample
        ids, sc = _planted_knn_lists(inst.labels, rows, K, seed)
        pk_rows = sp.csr_matrix((sc.ravel(), (np.repeat(np.arange(rows.size), K), ids.ravel())),
                                shape=(rows.size, n))
        pk_rows, _ = oc.row_stochastic(pk_rows)
        Q = rng.standard_normal((n, c)) / np.sqrt(n)     # the apply's cost is value-blind
        if inst.kind == "hypergraph":
            h = inst.structure.tocsr()
            p_e, _ = oc.row_stochastic(h)
            p_v_rows, _ = oc.row_stochastic(h.T.tocsr()[rows])
            t_pe, T = _timed(lambda: p_e @ Q)                       # walk.py:139-140
            t_pv, S = _timed(lambda: p_v_rows @ T)
            t_struct = t_pe + t_pv / f
        else:
            p_n_rows, _ = oc.row_stochastic(inst.structure.tocsr()[rows])
            t_s, S = _timed(lambda: p_n_rows @ Q)                   # walk.py:141-142
            t_struct = t_s / f
        b = np.full((rows.size, 1), beta)

        def knn_mix():
            a = pk_rows @ Q                                          # walk.py:188
            return (1.0 - b) * S + b * a                             # walk.py:189
        t_mix, Z = _timed(knn_mix)
        out["apply_s"] = t_struct + t_mix / f                        # walk.py:177-190
        out["init_step_s"] = t_struct      # one T_i restart step (walk.py:153-174 is its transpose)

        # Householder QR of the tall-skinny block (engine.py:140)
        t, _ = _timed(lambda: np.linalg.qr(Z))
        out["qr_s"] = t / f

        # discretisation (engine.py:183-218): one rounding round, one prototype start
        qs = Z[:, 1:]
        nrm = np.linalg.norm(qs, axis=1)
        qt = np.divide(qs, nrm[:, None], out=np.zeros_like(qs), where=nrm[:, None] > 0)
        t, _ = _timed(lambda: oc._rounding_run(qt, np.eye(k), 1, oc.DISC_TOL))
        out["disc_round_s"] = t / f
        t, _ = _timed(lambda: oc._prototype_start(qt, k))
        out["disc_proto_s"] = t / f
    out["mhc_s"] = oc.GAMMA * out["apply_s"]                           # engine.py:291-299
    return out


def full_run_estimate(tm: dict, counts: dict, t_i: int = 25) -> float:
    """Seconds of one reference clustering with the run's kernel counts:
    KNN + T_i init steps + iterations x (apply + QR) + per sample
    (prototype start + rounds x round + gamma applies) + the initial MHC."""
    calls = counts["disc_calls"]
    return (tm["knn_s"] + t_i * tm["init_step_s"]
            + counts["iterations"] * (tm["apply_s"] + tm["qr_s"])
            + calls * tm["disc_proto_s"] + counts["disc_rounds"] * tm["disc_round_s"]
            + (calls + 1) * tm["mhc_s"])
