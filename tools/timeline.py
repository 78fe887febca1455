"""GPU timeline of one DBLP-shaped run_prepared (torch.profiler / CUPTI):
busy vs idle time, top kernels, largest idle gaps (host stalls)."""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2408_05459_b200 as ancka  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "dblp"
inst = synth.make(shape, seed=0)
net = (ancka.AttributedNetwork.hypergraph(inst.structure, inst.X) if inst.kind == "hypergraph"
       else ancka.AttributedNetwork.graph(inst.structure, inst.X))
params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=0, knn_mode=ancka.KnnMode.EXACT)
prep = ancka.prepare_network(net, params)
for _ in range(3):
    ancka.run_prepared(prep, params)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ancka.run_prepared(prep, params)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy, last_end, gaps, prev = 0.0, t0, [], "-"
for e in ev:
    s, f = e.time_range.start, e.time_range.end
    if s > last_end:
        gaps.append((s - last_end, prev[:45] + "  ->  " + e.name[:45]))
    prev = e.name
    busy += max(0, f - max(s, last_end))
    last_end = max(last_end, f)
print(f"span {(t1 - t0) / 1e3:.2f} ms  busy {busy / 1e3:.2f} ms  idle {(t1 - t0 - busy) / 1e3:.2f} ms  events {len(ev)}")
agg = {}
for e in ev:
    a = agg.setdefault(e.name[:70], [0, 0.0])
    a[0] += 1
    a[1] += e.time_range.end - e.time_range.start
for name, (cnt, tot) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{tot / 1e3:8.3f} ms  x{cnt:4d}  {name}")
gaps.sort(reverse=True)
print("largest idle gaps (us, next event):")
for g, name in gaps[:12]:
    print(f"  {g:8.1f}  {name}")
print(f"gaps > 20us: {sum(1 for g, _ in gaps if g > 20)} totalling {sum(g for g, _ in gaps if g > 20) / 1e3:.2f} ms")
# idle time attributed to where it happens: before the first orth_fused launch
# (KNN / operator / init) vs inside the iteration loop, by (prev -> next) pair
first_loop = next((e.time_range.start for e in ev if "orth_fused" in e.name or "cgs2" in e.name), t1)
pre = sum(g for g, _ in [(x, 0) for x in []])
idle_pre, idle_loop, pairs = 0.0, 0.0, {}
last_end, prev = t0, "-"
for e in ev:
    s, f = e.time_range.start, e.time_range.end
    if s > last_end:
        g = s - last_end
        if s < first_loop:
            idle_pre += g
        else:
            idle_loop += g
            key = prev[:40] + " -> " + e.name[:40]
            a = pairs.setdefault(key, [0, 0.0])
            a[0] += 1
            a[1] += g
    prev = e.name
    last_end = max(last_end, f)
print(f"idle before loop {idle_pre / 1e3:.2f} ms, in loop {idle_loop / 1e3:.2f} ms "
      f"(loop span {(t1 - first_loop) / 1e3:.2f} ms)")
for key, (cnt, tot) in sorted(pairs.items(), key=lambda x: -x[1][1])[:25]:
    print(f"  {tot:8.1f} us  x{cnt:3d}  {key}")
print("pre-loop gaps > 8 us in order (t_ms, gap_us, prev -> next):")
last_end, prev = t0, "-"
for e in ev:
    s, f = e.time_range.start, e.time_range.end
    if s >= first_loop:
        break
    if s - last_end > 8:
        print(f"  {(s - t0) / 1e3:7.3f} {s - last_end:7.1f}  {prev[:50]} -> {e.name[:50]}")
    prev = e.name
    last_end = max(last_end, f)
