"""One clustering of a full-size shape on 1 GPU with a phase breakdown.

    python tools/scale_run.py SHAPE [scale] [reps]   (KNN_MODE=exact|auto|approx, default exact)
"""
import os
import sys
import time
import warnings
from pathlib import Path

# large shapes (Papers100M/8 peaks at ~182 GB) need the allocator to grow
# segments instead of carving fixed ones: fragmentation otherwise fails an
# 18 GB block with 21 GB reserved but unallocated
if len(sys.argv) > 1 and sys.argv[1] == "papers100m":
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "magpm"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
t0 = time.perf_counter()
inst = synth.make(shape, seed=0, scale=scale)
print(f"generated {shape} n={inst.structure.shape[1]} nnz={inst.structure.nnz} "
      f"X nnz={getattr(inst.X, 'nnz', inst.X.size)} in {time.perf_counter() - t0:.1f}s", flush=True)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
mode = {"exact": ancka.KnnMode.EXACT, "auto": ancka.KnnMode.AUTO,
        "approx": ancka.KnnMode.APPROX}[os.environ.get("KNN_MODE", "exact")]
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=mode)
t0 = time.perf_counter()
prep = ancka.prepare_network(net, params)
torch.cuda.synchronize()
print(f"prepare {time.perf_counter() - t0:.2f}s level={prep.x_level}", flush=True)
for rep in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = ancka.run_prepared(prep, params)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    from sklearn.metrics import adjusted_rand_score
    print(f"run {rep}: {dt:.2f}s iters={res.iterations} stop={res.stop_reason} "
          f"err={res.error} ari_planted={adjusted_rand_score(inst.labels, res.y.assignment):.4f} "
          f"timings={ {k: round(v, 1) for k, v in res.timings_ms.items()} }", flush=True)
    if res.warnings:
        print("   warnings:", sorted(set(res.warnings)), flush=True)
print("max mem GB", torch.cuda.max_memory_allocated() / 1e9,
      "reserved GB", torch.cuda.max_memory_reserved() / 1e9, flush=True)
