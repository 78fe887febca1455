"""Discretize phase timers summed over every call of one clustering run:
ANCKA_DISC_TIMING=1 python tools/disc_profile_run.py [shape]"""
import os
import sys
import time
import warnings
from pathlib import Path

os.environ["ANCKA_DISC_TIMING"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "amazon2m"
inst = synth.make(shape, seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
t0 = time.perf_counter()
res = ancka.run_ancka(net, params)
print(f"run {time.perf_counter() - t0:.2f} s, iterations {res.iterations}",
      {k: round(v) for k, v in res.timings_ms.items()})
P = engine.DISC_PROFILE
ns = {"round_gap": 15, "sync_after_A": 1, "reduce": 2, "reseed+scale": 3, "polar": 4,
      "proto_iter": 5, "phaseA": 6}
print(f"calls {P['calls']} rounds {P['rounds']} NS iterations {P[7]}")
print("ms:", {n: round(P[i] / 1e6, 1) for n, i in ns.items()})
sub = ["wait+stage", "score+argmax", "rescore", "skipped rows", "accumulate"]
print("CTA0 Mclk:", {sub[j]: round(P[8 + j] / 1e6, 1) for j in range(5)},
      "flagged", P[14], "changed", P[13])
