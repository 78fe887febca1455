"""Phase wall times of the row-partitioned path at N = 1 (NCCL world 1).

    python tools/dist_phases.py amazon2m
"""
import json
import os
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import dist as D, synth  # noqa: E402

name = sys.argv[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
inst = synth.make(name, seed=0)
net = (ancka.AttributedNetwork.hypergraph if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph)(inst.structure, inst.X)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
D.DIST_TIMING = True
D.DISC_MODE = os.environ.get("DISC_MODE", "auto")
B = D.CudaBackend()
for rep in range(int(os.environ.get("REPS", "2"))):
    res = D.run_ancka_dist(net, params, B)
    print(json.dumps({"rep": rep, "iterations": res.iterations, "stop": res.stop_reason,
                      "timings_ms": res.timings_ms, "total_ms": round(sum(res.timings_ms.values()), 1)}))
dist.destroy_process_group()
