"""Host breakdown of run_ancka(net, params) from host inputs."""
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, knn, network, synth, walk  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "dblp"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
inst = synth.make(shape, seed=0)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
import gc, os
if os.environ.get("NOGC"): gc.disable()
for it in range(reps):
    T = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
           else ancka.AttributedNetwork.graph(inst.structure, inst.X))
    T["construct"] = time.perf_counter() - t0
    t = time.perf_counter(); vnet, _ = network.validate_network(net); T["validate"] = time.perf_counter() - t
    t = time.perf_counter(); xd = knn.attributes_to_device(vnet.attributes, None); lvl = xd.level; torch.cuda.synchronize(); T["x_to_dev+level"] = time.perf_counter() - t
    t = time.perf_counter(); fac = walk.StructureFactors(vnet); torch.cuda.synchronize(); T["factors"] = time.perf_counter() - t
    prep = engine.PreparedNetwork(vnet, 10, xd, lvl, fac)
    t = time.perf_counter(); res = ancka.run_prepared(prep, params); lab = res.y.assignment; T["run"] = time.perf_counter() - t
    print(f"iter {it}: total {(time.perf_counter()-t0)*1e3:.1f} ms", {k: round(v * 1e3, 2) for k, v in T.items()})
