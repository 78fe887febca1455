"""Rounds per discretize call along a DBLP-shaped run."""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, synth  # noqa: E402

orig = engine._discretize_device
log = []


def spy(q32, col0, k, max_iter, tol, lab, info):
    orig(q32, col0, k, max_iter, tol, lab, info)
    inf = info[:8].cpu().numpy()
    log.append((int(inf[6]), int(inf[7]), int(inf[3])))


engine._discretize_device = spy
inst = synth.make(sys.argv[1] if len(sys.argv) > 1 else "dblp", seed=0)
net = ancka.AttributedNetwork.hypergraph(inst.structure, inst.X)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
res = ancka.run_ancka(net, params)
print("calls", len(log), "rounds (run0, run1, winner):", log)
