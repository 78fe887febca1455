"""One DBLP-shaped clustering after a warm-up run (target for ncu launch lists)."""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "dblp"
what = sys.argv[2] if len(sys.argv) > 2 else "run"
inst = synth.make(shape, seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
if what == "knn":
    from paper_2408_05459_b200.knn import knn_search_exact_device
    for _ in range(2):
        knn_search_exact_device(prep.x_dev, prep.K, integer=prep.x_level)
    torch.cuda.synchronize()
else:
    for _ in range(2):
        res = ancka.run_prepared(prep, params)
    torch.cuda.synchronize()
    print(res.iterations, res.timings_ms)
