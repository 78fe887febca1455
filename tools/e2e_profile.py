"""cProfile of one run_ancka(net, params) on the DBLP shape after warm-up:
where the host-side (e2e minus device pipeline) time goes."""
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
for _ in range(4):
    ancka.run_ancka(net, params)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    prep = engine.prepare_network(net, params)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = engine.run_prepared(prep, params)
    lab = r.y.assignment
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"prepare {1e3 * (t1 - t0):.2f} ms  run_prepared {1e3 * (t2 - t1):.2f} ms  "
          f"{ {k: round(v, 2) for k, v in r.timings_ms.items()} }")
pr = cProfile.Profile()
pr.enable()
r = ancka.run_ancka(net, params)
lab = r.y.assignment
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(40)
