"""Host cost of capturing the tau-block CUDA graph of the unfused orthogonal
loop (first run(5) per parity) vs eager and replayed blocks."""
import os
import sys
import time
import warnings
from pathlib import Path

os.environ["ANCKA_ORTH_UNFUSED"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "dblp"
inst = synth.make(shape, seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
op, g = engine.build_pipeline_device(prep, params)
c = inst.k + 1
for graphs in (False, True):
    loop = engine._Loop(op, c, inst.k, 5, graphs, False)
    loop.Q[0][:, :c] = torch.randn(op.n, c, device="cuda")
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        loop.run(5)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"graphs={graphs} run {it}: host {1e3 * (t1 - t0):8.2f} ms  total {1e3 * (t2 - t0):8.2f} ms",
              flush=True)
