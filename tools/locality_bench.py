"""f32 joint apply at Amazon2M with and without the locality row order
(rows grouped by the greedy-init labels): python tools/locality_bench.py [shape]."""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import _lib, engine, synth  # noqa: E402
from paper_2408_05459_b200._device import ld_for  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "amazon2m"
inst = synth.make(shape, seed=0)
net = ancka.AttributedNetwork.graph(inst.structure, inst.X)
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
op, g = engine.build_pipeline_device(prep, params)
n, c = op.n, inst.k + 1
ld = ld_for(c, torch.float32)
Q = torch.randn((n, ld), dtype=torch.float32, device="cuda")
Q[:, c:] = 0
s32 = op.struct(_lib.F32)
scr = op.scratch(c, torch.float32)


def run(reps=20):
    Z = torch.empty_like(Q)
    for _ in range(3):
        _lib.call("ancka_op_apply", s32, Q.data_ptr(), ld, c, Z.data_ptr(), ld, scr.data_ptr(), _lib.stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        _lib.call("ancka_op_apply", s32, Q.data_ptr(), ld, c, Z.data_ptr(), ld, scr.data_ptr(), _lib.stream())
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps, Z


t0, z0 = run()
labels, _, _, _ = engine._init_labels_sizes(op, inst.k, 25, 0.2)
op.set_locality(labels, inst.k)
t1, z1 = run()
from sklearn.metrics import adjusted_rand_score
print(f"{shape}: apply {t0:.3f} ms (index order) -> {t1:.3f} ms (init-label order); "
      f"bit-identical: {bool(torch.equal(z0, z1))}; init ARI vs planted "
      f"{adjusted_rand_score(inst.labels, labels.cpu().numpy()):.3f}")
planted = torch.from_numpy(inst.labels.astype('int32')).cuda()
op.set_locality(planted, inst.k)
t2, z2 = run()
print(f"   planted-label order: {t2:.3f} ms; bit-identical: {bool(torch.equal(z0, z2))}")
