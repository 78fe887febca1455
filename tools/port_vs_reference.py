"""CPU arm fairness: the oracle port (the reference arm's code on the GPU box)
timed beside the unmodified reference on the same inputs, in this container
(the only place /root/reference exists).

    python tools/port_vs_reference.py > profiles/r02/port_vs_reference.json
"""
import json
import os
import sys
import time
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
warnings.simplefilter("ignore")

import numpy as np  # noqa: E402

import ancka  # noqa: E402  (the reference)
from ancka import engine as ref_engine, knn as ref_knn, walk as ref_walk  # noqa: E402
from oracle import ancka_cpu as oc  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402


def timed(fn, reps=1):
    best = None
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


res = {"cores": len(os.sched_getaffinity(0))}
inst = synth.make("dblp", seed=0)
X = inst.X
t_ref, nl = timed(lambda: ref_knn.knn_search_exact(X, 10))
t_port, (ids, sc) = timed(lambda: oc.knn_exact(X, 10))
res["dblp_knn_exact"] = {"reference_s": round(t_ref, 2), "port_s": round(t_port, 2),
                         "ratio_port_over_reference": round(t_port / t_ref, 3),
                         "same_ids": bool(np.array_equal(ids, nl.ids))}
# one joint apply and one orthogonal step on the reference operator
net = ancka.AttributedNetwork.hypergraph(inst.structure, X)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
op, g, _ = ref_engine.build_pipeline(net, params)
onet = {"kind": "hypergraph", "S": inst.structure, "X": X}
oop, _ = oc.build(onet, inst.k, knn_k=10, knn=(nl.ids, nl.scores))
m = np.random.default_rng(0).standard_normal((net.n, inst.k + 1))
t_ref, z_ref = timed(lambda: ref_walk.apply_joint_transition(op, m), 5)
t_port, z_port = timed(lambda: oc.joint_apply(oop, m), 5)
res["dblp_joint_apply"] = {"reference_s": round(t_ref, 4), "port_s": round(t_port, 4),
                           "ratio_port_over_reference": round(t_port / t_ref, 3),
                           "max_abs_diff": float(np.abs(z_ref - z_port).max())}
print(json.dumps(res, indent=1))
