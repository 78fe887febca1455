"""Host profile of prepare_network (validation + uploads) on the DBLP shape."""
import cProfile
import pstats
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
for _ in range(5):
    engine.prepare_network(net, params)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    engine.prepare_network(net, params)
    torch.cuda.synchronize()
    print(f"prepare {1e3 * (time.perf_counter() - t0):.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    engine.prepare_network(net, params)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
