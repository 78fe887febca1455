"""Which Python call sites issue the torch glue ops of one DBLP run_prepared
(aten op counts grouped by the innermost package frames)."""
import sys
import warnings
from collections import Counter
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402

inst = synth.make("dblp", seed=0)
net = ancka.AttributedNetwork.hypergraph(inst.structure, inst.X)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
for _ in range(3):
    ancka.run_prepared(prep, params)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU], with_stack=True) as prof:
    ancka.run_prepared(prep, params)
    torch.cuda.synchronize()
sites, ops = Counter(), Counter()
for e in prof.events():
    if not e.name.startswith("aten::") or e.cpu_parent is not None and e.cpu_parent.name.startswith("aten::"):
        continue
    st = [f for f in (e.stack or []) if "paper_2408_05459_b200" in f]
    site = st[0].split("paper_2408_05459_b200/")[-1] if st else "?"
    sites[site] += 1
    ops[(site, e.name)] += 1
print("top-level aten ops by call site:")
for s, c in sites.most_common(40):
    print(f"{c:5d}  {s}")
print()
for (s, o), c in ops.most_common(40):
    print(f"{c:5d}  {o:30s} {s}")
