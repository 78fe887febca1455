"""Wall time of one device discretisation call on a planted n x k block
(k <= 64: cooperative kernel; 64 < k <= 192: device-driven wide rounds):
python tools/disc_dev_time.py [n] [k] [reps]"""
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
warnings.simplefilter("ignore")
import torch  # noqa: E402

from paper_2408_05459_b200 import engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2449029
k = int(sys.argv[2]) if len(sys.argv) > 2 else 172
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = torch.Generator(device="cuda").manual_seed(0)
lab0 = torch.randint(0, k, (n,), device="cuda", generator=g)
q = torch.zeros((n, (k + 1 + 3) // 4 * 4), dtype=torch.float32, device="cuda")
q[:, 0] = n ** -0.5
q[torch.arange(n, device="cuda"), lab0 + 1] = 1.0
q[:, 1:k + 1] += 0.15 * torch.randn((n, k), device="cuda", generator=g)
lab = torch.empty(n, dtype=torch.int32, device="cuda")
info = torch.zeros(8 + 200 + 2 * k * k + 16, dtype=torch.float64, device="cuda")
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    engine._discretize_device(q, 1, k, 100, 1e-10, lab, info)
    torch.cuda.synchronize()
    print(f"{(time.perf_counter() - t0) * 1e3:.1f} ms  rounds {info[6].item():.0f}+{info[7].item():.0f} "
          f"obj {info[0].item():.6f}", flush=True)
