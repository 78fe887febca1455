"""Measured tensor-pipe peaks (tcgen05.mma M=128 N=256, operands in smem):
fp8 (kind::f8f6f4) and bf16 (kind::f16).  Writes profiles/r02/tc_peak.json.

    python tools/tc_peak.py
"""
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2408_05459_b200 import _lib  # noqa: E402

_lib.require_device()
cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
out = {}
for fmt, name in ((0, "fp8_e4m3"), (1, "bf16")):
    best = None
    for iters in (2000, 20000, 20000, 20000):
        f, ms = ctypes.c_double(), ctypes.c_double()
        _lib.call("ancka_tc_peak", fmt, iters, ctypes.byref(f), ctypes.byref(ms), cyc.data_ptr(),
                  _lib.stream())
        tf = f.value / (ms.value * 1e-3) / 1e12
        if iters == 20000:
            best = max(best or 0.0, tf)
    c = cyc.cpu().numpy()
    out[name] = {"tflops": round(best, 1), "sm_cycles_median": int(sorted(c)[74]),
                 "per_sm_flop_per_clk": round(2 * 128 * 256 * (32 if fmt == 0 else 16) * 4 *
                                              20000 / float(sorted(c)[74]), 1)}
# L2 read bandwidth (ld.global.cg, L1 bypassed): 12.6 MB of 192-byte rows (an
# Amazon2M cluster's rows of Q at c = 48), sequential and hashed-row gathers
rows, rf = 65536, 48
tab = torch.randn(rows * rf, device="cuda")
sink = torch.zeros(1, device="cuda")
for gather, name in ((0, "l2_read_seq"), (1, "l2_read_gather192")):
    best = 0.0
    for _ in range(3):
        b, ms = ctypes.c_double(), ctypes.c_double()
        _lib.call("ancka_l2_read", tab.data_ptr(), rows, rf, 200, gather, sink.data_ptr(),
                  ctypes.byref(b), ctypes.byref(ms), _lib.stream())
        best = max(best, b.value / (ms.value * 1e-3) / 1e12)
    out[name] = {"tb_per_s": round(best, 2), "table_mb": round(rows * rf * 4 / 1e6, 1)}
print(json.dumps(out))
(ROOT / "profiles" / "r02" / "tc_peak.json").write_text(json.dumps(out, indent=1) + "\n")
