"""Row-length statistics of the device operator factors (hubness check)."""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import numpy as np  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "dblp"
inst = synth.make(shape, seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
op, g = ancka.engine.build_pipeline_device(prep, params)
for name, m in [("p_k", op.p_k_dev)] + list(op._f.items()):
    rl = np.diff(m.rowptr.cpu().numpy())
    print(f"{name}: rows={m.rows} nnz={m.nnz} mean={rl.mean():.1f} p50={np.percentile(rl,50):.0f} "
          f"p99={np.percentile(rl,99):.0f} p99.9={np.percentile(rl,99.9):.0f} max={rl.max()}")
