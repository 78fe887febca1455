"""Per-phase ns inside the discretize kernel (ANCKA_DISC_TIMING=1)."""
import os
import sys
import warnings
from pathlib import Path

os.environ["ANCKA_DISC_TIMING"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import engine, synth  # noqa: E402

if len(sys.argv) > 1:   # synthetic block: tools/disc_timing.py n k  (planted + noise)
    n, k = int(sys.argv[1]), int(sys.argv[2])
    g = torch.Generator(device="cuda").manual_seed(0)
    lab0 = torch.randint(0, k, (n,), device="cuda", generator=g)
    q = torch.zeros((n, 48 if k + 1 <= 48 else k + 1), dtype=torch.float32, device="cuda")
    q[:, 0] = n ** -0.5
    q[torch.arange(n, device="cuda"), lab0 + 1] = 1.0
    q[:, 1:k + 1] += 0.3 * torch.randn((n, k), device="cuda", generator=g)
else:
    shape = os.environ.get("SHAPE", "dblp")
    inst = synth.make(shape, seed=0)
    net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
           else ancka.AttributedNetwork.graph(inst.structure, inst.X))
    params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
    res = ancka.run_ancka(net, params)
    q = res.state.q_dev
    k = inst.k
lab = torch.empty(q.shape[0], dtype=torch.int32, device=q.device)
info = torch.zeros(8 + 200 + 2 * k * k + 16, dtype=torch.float64, device=q.device)
for rep in range(3):
    info.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    engine._discretize_device(q, 1, k, 100, 1e-10, lab, info)
    b.record()
    b.synchronize()
    t = info[8 + 200 + 2 * k * k:].cpu().numpy().view(np.uint64)
    names = ["to_round_start", "sync_after_A", "reduce", "reseed+scale", "polar", "proto_iter", "phaseA", "ns_iters"]
    inf = info[:8].cpu().numpy()
    print(f"total {a.elapsed_time(b)*1e3:.0f} us rounds={inf[6]:.0f}+{inf[7]:.0f}",
          {names[i]: int(t[i if i else 15]) // 1000 for i in (0, 1, 2, 3, 4, 5, 6)}, "us; NS iterations", int(t[7]))
    if len(t) > 8:
        sub = ["wait+stage", "score+argmax", "rescore", "skipped rows (CTA0)", "accumulate"]
        print("   CTA0 clocks (M):", {sub[j]: round(int(t[8 + j]) / 1e6, 2) for j in range(5)},
              "flagged rows (CTA0):", int(t[14]), "changed rows (CTA0):", int(t[13]))
