"""Kernel timeline of the host-driven wide discretisation at n x k:
python tools/disc_wide_profile.py [n] [k]."""
import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2408_05459_b200 import engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2449029
k = int(sys.argv[2]) if len(sys.argv) > 2 else 47
g = torch.Generator(device="cuda").manual_seed(0)
lab0 = torch.randint(0, k, (n,), device="cuda", generator=g)
q = torch.zeros((n, 48 if k + 1 <= 48 else k + 1), dtype=torch.float32, device="cuda")
q[:, 0] = n ** -0.5
q[torch.arange(n, device="cuda"), lab0 + 1] = 1.0
q[:, 1:k + 1] += 0.3 * torch.randn((n, k), device="cuda", generator=g)
engine.WIDE_DISCRETIZE_K = 16
lab = torch.empty(n, dtype=torch.int32, device="cuda")
info = torch.zeros(8 + 200 + 2 * k * k, dtype=torch.float64, device="cuda")
engine._discretize_device(q, 1, k, 100, 1e-10, lab, info)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    engine._discretize_device(q, 1, k, 100, 1e-10, lab, info)
    torch.cuda.synchronize()
wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
agg = {}
for e in ev:
    a = agg.setdefault(e.name[:60], [0, 0.0])
    a[0] += 1
    a[1] += e.time_range.end - e.time_range.start
print(f"wall {wall * 1e3:.1f} ms, rounds {info[6].item():.0f}+{info[7].item():.0f}")
for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:10]:
    print(f"{t / 1e3:8.2f} ms x{c:4d} {name}")
