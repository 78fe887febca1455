"""Time one f32 MHC call (ancka_mhc) at a shape: python tools/mhc_timing.py [shape]
(ANCKA_MHC_UNFUSED=1 for the multi-launch path)."""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import _lib, engine, synth  # noqa: E402

inst = synth.make(sys.argv[1] if len(sys.argv) > 1 else "dblp", seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
op, g = engine.build_pipeline_device(prep, params)
labels = torch.from_numpy(inst.labels.astype(np.int32)).cuda()
run = engine._MhcRunner(op, inst.k, _lib.F32)
run64 = engine._MhcRunner(op, inst.k, _lib.F64)
reps = 20
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run(labels)
    b.record()
    b.synchronize()
    print(f"{a.elapsed_time(b) * 1e3 / reps:.1f} us per call, phi32 {float(run.phi):.9f} "
          f"phi64 {float(run64(labels)):.9f}")

import ctypes  # noqa: E402
import os  # noqa: E402
if os.environ.get("ANCKA_MHC_TIMING"):
    lib = _lib.load()
    buf = (ctypes.c_ulonglong * (64 + 9 * 1024))()
    lib.ancka_mhc_timing(ctypes.cast(buf, ctypes.c_void_p), 1)
    for rep in range(reps):
        run(labels)
    lib.ancka_mhc_timing(ctypes.cast(buf, ctypes.c_void_p), 1)
    names = ["hist", "F0"] + [f"{x}{g}" for g in range(3) for x in ("T", "rows")]
    print("per call, us (CTA0 work / max CTA work):",
          {nm: (round(buf[2 * q] / reps / 1e3, 1), round(buf[2 * q + 1] / 1e3, 1)) for q, nm in enumerate(names)})
    per = np.array(buf[64:64 + 8 * 1024], dtype=np.float64).reshape(8, 1024) / 1e3
    for q in (3, 5):
        v = per[q][:296]
        print(names[q], "per-CTA us: min %.1f med %.1f max %.1f; slowest CTAs" % (v.min(), np.median(v), v.max()),
              np.argsort(-v)[:12].tolist(), np.round(np.sort(v)[::-1][:12], 1).tolist())
    nz = np.array(buf[64 + 8 * 1024:64 + 8 * 1024 + 296], dtype=np.float64) / (reps * 3)
    print("nonzeros per CTA per row pass: min %d med %d max %d" % (nz.min(), np.median(nz), nz.max()))
    v = per[5][:296]
    print("corr(nnz, time) rows1: %.3f" % np.corrcoef(nz, v)[0, 1])
