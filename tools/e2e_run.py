"""Wall-clock run_ancka(net, params) from host inputs (the bench's e2e leg):
python tools/e2e_run.py [shape] [reps]"""
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "amazon2m"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
inst = synth.make(shape, seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = ancka.run_ancka(net, params)
    lab = res.y.assignment
    dt = time.perf_counter() - t0
    print(f"run {r}: {dt:.3f} s iters={res.iterations}",
          {k: round(v) for k, v in res.timings_ms.items()}, flush=True)
