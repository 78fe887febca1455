"""Approximate-KNN timing at a named shape (device-trained centroids).

    python tools/approx_time.py amazon2m [scale]
"""
import json
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import knn as aknn, synth  # noqa: E402
from paper_2408_05459_b200.knn import attributes_to_device  # noqa: E402

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
inst = synth.make(name, seed=0, scale=scale)
xd = attributes_to_device(inst.X, None)
torch.cuda.synchronize()
out = {"shape": name, "n": inst.X.shape[0], "d": inst.X.shape[1]}
for rep in range(2):
    t0 = time.perf_counter()
    nl = ancka.knn_search_approx(xd, 10, seed=0)
    torch.cuda.synchronize()
    out[f"approx_s_{rep}"] = round(time.perf_counter() - t0, 3)
out["stats"] = {k: v for k, v in aknn.LAST_STATS["approx"].items()}
# phases of one search at the final nprobe
ix = aknn.build_ivf_index(xd, out["stats"]["nlist"], 0)
torch.cuda.synchronize()
t0 = time.perf_counter()
aknn.ivf_search_all_device(ix, 10, out["stats"]["nprobe"])
torch.cuda.synchronize()
out["search_all_s"] = round(time.perf_counter() - t0, 3)
t0 = time.perf_counter()
ids, _ = aknn.knn_search_exact_device(xd, 10)
torch.cuda.synchronize()
out["exact_s"] = round(time.perf_counter() - t0, 3)
ex = ids.cpu().numpy()
ap = nl.ids
hits = [np.isin(e[e >= 0], g[g >= 0]).mean() for e, g in zip(ex[::50], ap[::50]) if (e >= 0).any()]
out["recall_vs_exact_sampled"] = round(float(np.mean(hits)), 4)
print(json.dumps(out))
