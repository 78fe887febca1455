"""Where e2e time goes: run_ancka wall time vs its prepare / device parts."""
import gc
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, synth  # noqa: E402

inst = synth.make("dblp", seed=0)
net = ancka.AttributedNetwork.hypergraph(inst.structure, inst.X)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
for _ in range(4):
    ancka.run_ancka(net, params)
rows = []
for _ in range(8):
    gc.collect()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prep = engine.prepare_network(net, params)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r = engine.run_prepared(prep, params)
    t3 = time.perf_counter()
    lab = r.y.assignment
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    gc.collect()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    r2 = ancka.run_ancka(net, params)
    lab2 = r2.y.assignment
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t6 - t5))
a = np.median(np.array(rows), axis=0) * 1e3
print(f"prepare host {a[0]:.2f} + drain {a[1]:.2f} | run_prepared {a[2]:.2f} + tail {a[3]:.2f} | run_ancka {a[4]:.2f} ms")
