"""How many tau samples of one clustering see the same labels as the
previous sample (their MHC evaluation would repeat): python tools/mhc_repeat.py amazon2m"""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "amazon2m"
inst = synth.make(shape, seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
seen = []
orig = engine._MhcRunner.__call__


def spy(self, labels, phi_out=None):
    seen.append(labels.clone())
    return orig(self, labels, phi_out)


engine._MhcRunner.__call__ = spy
res = ancka.run_ancka(net, params)
same = sum(int(torch.equal(a, b)) for a, b in zip(seen[1:], seen[:-1]))
changed = [int((a != b).sum()) for a, b in zip(seen[1:], seen[:-1])]
# same partition up to relabelling: as many distinct (new, old) pairs as clusters
k = inst.k
pairs = [int(torch.unique(a.long() * k + b.long()).numel()) for a, b in zip(seen[1:], seen[:-1])]
print({"samples": len(seen), "same_labels": same, "iterations": res.iterations,
       "same_partition": sum(int(p == k) for p in pairs), "distinct_pairs": pairs,
       "changed_rows": changed})
