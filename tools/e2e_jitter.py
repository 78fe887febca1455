"""Host jitter of run_ancka(net, params) on the DBLP shape: prepare vs device
pipeline wall time over repeated calls (after bench-like warm-up)."""
import gc
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, synth  # noqa: E402

inst = synth.make("dblp", seed=0)
net = ancka.AttributedNetwork.hypergraph(inst.structure, inst.X)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
for _ in range(3):
    ancka.run_ancka(net, params)
rows = []
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 15):
    gc.collect()
    torch.cuda.synchronize()
    a0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    t0 = time.perf_counter()
    prep = engine.prepare_network(net, params)
    t1 = time.perf_counter()
    res = engine.run_prepared(prep, params)
    lab = res.y.assignment
    t2 = time.perf_counter()
    rows.append((t1 - t0, t2 - t1))
    a1 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    print(f"cudaMalloc {a1 - a0:3d}  prep {1e3 * (t1 - t0):6.2f} ms  run {1e3 * (t2 - t1):6.2f} ms  phases "
          f"{ {k: round(v, 1) for k, v in res.timings_ms.items()} }", flush=True)
