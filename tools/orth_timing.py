"""Phase timers of the fused orthogonal block (ANCKA_ORTH_TIMING=1)."""
import os
import sys
import warnings
from pathlib import Path

os.environ["ANCKA_ORTH_TIMING"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, synth  # noqa: E402

inst = synth.make(sys.argv[1] if len(sys.argv) > 1 else "dblp", seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
op, g = engine.build_pipeline_device(prep, params)
loop = engine._Loop(op, inst.k + 1, inst.k, 5, True, True)
loop.Q[0][:, : inst.k + 1] = torch.randn(op.n, inst.k + 1, device="cuda")
for rep in range(3):
    loop.stats.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    loop.run(20)
    b.record()
    b.synchronize()
    t = loop.stats[4:16].cpu().numpy().view(np.uint64)
    print("slowest P2 CTA:", int(t[11]) & 0xFFFFF, "dt us", (int(t[11]) >> 20) / 1000)
    names = ["P1", "sync1", "P2+gram", "-", "sync2", "chol", "apply", "sync3", "-",
             "P2max_sum_over_steps", "P2sum_all_ctas"]
    print(f"20 steps {a.elapsed_time(b)*1e3:.0f} us:", {nm: int(v) // 1000 for nm, v in zip(names, t)}, "us")
