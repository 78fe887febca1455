"""CholQR pieces at an n x c f32 block (Amazon2M: 2449029 x 48):
python tools/qr_time.py [n] [c] -- gram, factor, apply and the whole QR."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2408_05459_b200 import _lib  # noqa: E402
from paper_2408_05459_b200._device import ld_for  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2449029
c = int(sys.argv[2]) if len(sys.argv) > 2 else 48
ld = ld_for(c, torch.float32)
g = torch.Generator(device="cuda").manual_seed(0)
Z = torch.randn((n, ld), dtype=torch.float32, device="cuda", generator=g)
Z[:, c:] = 0
Q = torch.empty_like(Z)
Qp = torch.randn_like(Z)
G = torch.empty(c * (c + 1) // 2, dtype=torch.float64, device="cuda")
stats = torch.tensor([0.0, 1.0] + [0.0] * 14, dtype=torch.float64, device="cuda")
lib = _lib.load()
ws = torch.empty(lib.ancka_orth_workspace_size(None, c), dtype=torch.uint8, device="cuda")
st = _lib.stream


def gram():
    _lib.call("ancka_gram_f32", Z.data_ptr(), n, ld, c, G.data_ptr(), ws.data_ptr(), ws.numel(), st())


def apply():
    _lib.call("ancka_cholqr_apply_f32", Z.data_ptr(), Qp.data_ptr(), Q.data_ptr(), n, ld, c,
              G.data_ptr(), stats.data_ptr(), ws.data_ptr(), ws.numel(), st())


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


tg = timed(gram)
ta = timed(apply)
tq = timed(lambda: (gram(), apply()))
Qd = Q[:, :c].double()
err = torch.linalg.norm(Qd.T @ Qd - torch.eye(c, dtype=torch.float64, device="cuda")).item()
print(f"n={n} c={c}: gram {tg * 1e3:.0f} us, factor+apply {ta * 1e3:.0f} us, QR {tq * 1e3:.0f} us "
      f"({12 * n * c / (tq * 1e-3) / 1e9:.0f} GB/s on 12nc), ||Q^T Q - I||_F {err:.2e}")
