"""Host-side timestamps of the device pipeline pieces (finds host stalls)."""
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, knn, synth, walk  # noqa: E402

inst = synth.make(sys.argv[1] if len(sys.argv) > 1 else "dblp", seed=0)
net = ancka.AttributedNetwork.hypergraph(inst.structure, inst.X)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
T = {}


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e3
        return r
    setattr(mod, name, g)


for m, n in [(engine, "knn_search_exact_device"), (engine, "build_knn_graph_device"),
             (engine, "build_walk_operator"), (engine, "_init_labels_device"),
             (engine, "_exact_step"), (engine, "_discretize_device"),
             (walk.WalkOperator, "_split_plan"), (engine._Loop, "run"), (engine._MhcRunner, "__call__")]:
    wrap(m, n)
for it in range(3):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = ancka.run_prepared(prep, params)
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) * 1e3
    print(f"run {it}: total {tot:.1f} ms", {k: round(v, 2) for k, v in T.items()}, res.timings_ms)
