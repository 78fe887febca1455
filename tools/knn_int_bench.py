"""Time the integer-exact tensor-core KNN on a DBLP-shaped matrix:
python tools/knn_int_bench.py [shape] [reps]  (ANCKA_KNN_DEBUG=1/2/3 variants)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2408_05459_b200 import knn as kn  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "dblp"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
inst = synth.make(shape, seed=0, scale=scale)
X = inst.X
xa = kn.DeviceAttributes(X, kn.integer_exact(X))
n, d = X.shape
ts = []
for r in range(reps + 2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    kn.knn_search_exact_device(xa, 10)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
ts = np.array(ts[2:])
print(f"{shape} n={n} d={d} level={xa.level}: min {ts.min():.3f} ms median {np.median(ts):.3f} ms "
      f"-> {2 * n * n * d / ts.min() / 1e9:.0f} TFLOP/s (2n^2d)")
