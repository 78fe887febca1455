"""Per-kernel timings of one orthogonal step on a full-size shape:
python tools/op_bench.py [shape] [scale]  -> SpMM (f32 apply), Gram+CholQR, MHC apply."""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import _lib, engine, synth  # noqa: E402
from paper_2408_05459_b200._device import WORKSPACE, ld_for  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "amazon2m"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
inst = synth.make(shape, seed=0, scale=scale)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
op, g = engine.build_pipeline_device(prep, params)
n, c = op.n, inst.k + 1
ld = ld_for(c, torch.float32)
Q = torch.randn((n, ld), dtype=torch.float32, device="cuda")
Q[:, c:] = 0
Z = torch.empty_like(Q)
Q2 = torch.empty_like(Q)
s32 = op.struct(_lib.F32)
scr = op.scratch(c, torch.float32)
stats = torch.tensor([0.0, 1.0, 0.0, 0.0] + [0.0] * 12, dtype=torch.float64, device="cuda")
ws = WORKSPACE.get("orth", _lib.load().ancka_orth_workspace_size(s32, c))
G = torch.empty(c * (c + 1) // 2, dtype=torch.float64, device="cuda")


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


st = _lib.stream
t_apply = timeit(lambda: _lib.call("ancka_op_apply", s32, Q.data_ptr(), ld, c, Z.data_ptr(), ld,
                                   scr.data_ptr(), st()))
t_gram = timeit(lambda: _lib.call("ancka_gram_f32", Z.data_ptr(), n, ld, c, G.data_ptr(),
                                  ws.data_ptr(), ws.numel(), st()))
t_chol = timeit(lambda: _lib.call("ancka_cholqr_apply_f32", Z.data_ptr(), Q.data_ptr(),
                                  Q2.data_ptr(), n, ld, c, G.data_ptr(), stats.data_ptr(),
                                  ws.data_ptr(), ws.numel(), st()))
t_step = timeit(lambda: _lib.call("ancka_orth_step_f32", s32, Q.data_ptr(), Q2.data_ptr(),
                                  Z.data_ptr(), ld, c, stats.data_ptr(), ws.data_ptr(), ws.numel(),
                                  st()))
nnz_k = int(op.p_k_dev.colidx.numel())
if inst.kind == "graph":
    nnz_a = int(inst.structure.nnz)
    b_op = 4 * nnz_a + 8 * nnz_k + 16 * (n + 1) + 8 * n + 4 * c * (nnz_a + nnz_k) + 4 * n * c
else:
    h = inst.structure
    m, nnz_h = h.shape[0], h.nnz
    b_op = (4 * nnz_h + 12 * m + 4 * c * nnz_h + 4 * m * c) + \
           (4 * nnz_h + 8 * nnz_k + 16 * n + 8 * n + 4 * c * (nnz_h + nnz_k) + 4 * n * c)
print(f"{shape} n={n} c={c} ld={ld} nnz_K={nnz_k}")
print(f"apply f32: {t_apply:.3f} ms  gather-model {b_op / 1e9:.2f} GB -> {b_op / t_apply / 1e6:.0f} GB/s")
print(f"gram: {t_gram:.3f} ms   cholqr_apply: {t_chol:.3f} ms   fused orth step: {t_step:.3f} ms")
print(f"QR bytes 12nc: {12 * n * c / 1e9:.2f} GB -> {12 * n * c / (t_gram + t_chol) / 1e6:.0f} GB/s")
