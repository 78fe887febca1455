#!/usr/bin/env python
"""Benchmark: end-to-end ANCKA clustering of a DBLP-shaped attributed
hypergraph (BASELINE.json configs[1]) on B200, beside the CPU reference path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one full `run_ancka` pipeline (exact KNN -> KNN graph -> operator
-> greedy init -> orthogonal iterations with discretisation and MHC until the
reference's stop rules fire) on a synthetic n=41,302 / m=22,363 / d=1,425
binary-attribute hypergraph with k=6, K=10.

`value` = seconds per clustering with attributes and structural factors
already resident in HBM (CUDA events on the launching stream, max over
ranks, L2 flushed before every timed step); `e2e` = the same through the
public API `run_ancka(net, params)` from host numpy/scipy inputs (validation,
host->device copies and the label read-back inside the timed region).
Multi-GPU runs are independent replicas (DBLP fits one GPU).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time
import warnings
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
warnings.simplefilter("ignore")

METRIC = "end-to-end clustering seconds + KNN build s; SpMM HBM GB/s at 1/2/4/8 B200 vs CPU"
SHAPE = "dblp"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_instance(seed):
    from paper_2408_05459_b200 import synth
    return synth.make(SHAPE, seed=seed)


def workload_config(inst, K):
    return {"workload": f"synthetic {SHAPE.upper()}-shaped attributed hypergraph",
            "n": int(inst.structure.shape[1]), "m": int(inst.structure.shape[0]),
            "d": int(inst.X.shape[1]), "attributes": "binary bag-of-words (CSR)",
            "k": int(inst.k), "knn_k": K, "alpha": 0.2, "beta": 0.5, "gamma": 3, "tau": 5,
            "t_a": 1000, "knn_mode": "exact", "l2": "flushed (256 MiB write) before each timed step"}


# ------------------------------------------------------------------ clocks --
_SAMPLER = r"""
import sys, time
try:
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
    bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
            nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
    mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
    print("ready", flush=True)
    while True:
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        print(",".join([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits]),
              flush=True)
        time.sleep(0.05)
except Exception as exc:
    print("ready", flush=True)
    print("error", exc, flush=True)
"""


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled by NVML in a
    separate process during the timed region: no thread of the benchmark
    process competes for its interpreter lock while kernels are enqueued."""

    def __init__(self, index=0):
        self.index, self.samples, self._p = index, [], None

    def __enter__(self):
        self._p = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.index)],
                                   stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self._p.stdout.readline()            # wait until NVML is initialised
        return self

    def __exit__(self, *exc):
        self._p.terminate()                  # this exact child process
        out, _ = self._p.communicate(timeout=10)
        for line in out.splitlines():
            v = [x.strip() for x in line.split(",")]
            if len(v) == 6:
                self.samples.append(v)

    def summary(self):
        import numpy as np
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


# --------------------------------------------------------------- CPU side --
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_run(inst, seed):
    from threadpoolctl import threadpool_limits

    from oracle import ancka_cpu as oc
    with threadpool_limits(limits=cpu_threads()):
        t0 = time.perf_counter()
        res = oc.run({"kind": inst.kind, "S": inst.structure, "X": inst.X}, inst.k, knn_k=10,
                     seed=seed)
        return time.perf_counter() - t0, res


def per_call(tm, calls):
    """Per-kernel timings: one orthogonal step (apply + QR),
    one discretisation, one MHC."""
    return {"ortho_step": round(tm["ortho_ms"] / max(calls["ortho"], 1), 4),
            "discretize": round(tm["discretize_ms"] / max(calls["discretize"], 1), 4),
            "mhc": round(tm["mhc_ms"] / max(calls["mhc"], 1), 4)}


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port) on the host."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    inst = make_instance(args.seed)
    oracle_run(make_small(), 0)                     # warm-up: imports, page-in
    steps = max(1, min(args.steps, 2))          # ~100 s per full CPU clustering
    times = [oracle_run(inst, args.seed)[0] for _ in range(steps)]
    v = sum(times) / len(times)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "s",
            "n_gpus": args.gpus, "steps": steps, "warmup": 1, "ms_per_step": round(v * 1e3, 2),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(inst, 10),
            "cpu_baseline": {"value": round(v, 4), "unit": "s", "cores": cpu_threads(),
                             "kind": "port",
                             "sample": f"full {SHAPE}-shaped clustering with the numpy/scipy "
                                       f"restatement of the reference (oracle/ancka_cpu.py), "
                                       f"{steps} timed run(s), BLAS threads = all host cores"},
            "e2e": {"value": round(v, 4), "unit": "s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def make_small():
    from paper_2408_05459_b200 import synth
    return synth.make(SHAPE, seed=1, n=1500)


# -------------------------------------------------------------- GPU side --
def spmm_gbytes_model(op, c, nnz_k):
    """SURVEY.md §8(d) hypergraph gather model (bytes per operator apply)."""
    n, m = op.n, op.m
    nnz_h = op._f["p_e"].nnz
    return (4 * nnz_h + 12 * m + 4 * c * nnz_h + 4 * m * c) + \
           (4 * nnz_h + 8 * nnz_k + 16 * n + 8 * n + 4 * c * (nnz_h + nnz_k) + 4 * n * c)


def time_kernel(fn, reps):
    import torch
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2408_05459_b200 as ancka
    from paper_2408_05459_b200 import _lib
    from paper_2408_05459_b200._device import padded
    from paper_2408_05459_b200.knn import knn_search_exact_device

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.require_device()

    inst = make_instance(args.seed + rank)
    net = ancka.AttributedNetwork.hypergraph(inst.structure, inst.X)
    params = ancka.ClusterParams(k=inst.k, knn_k=10, seed=args.seed + rank,
                                 knn_mode=ancka.KnnMode.EXACT)
    prep = ancka.prepare_network(net, params)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        res = ancka.run_prepared(prep, params)
    barrier()
    step_ms, launches, results = [], 0, []
    with ClockSampler(local) as clocks:
        barrier()
        gc.disable()                          # no collector pauses inside timed steps
        for _ in range(args.steps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            res = ancka.run_prepared(prep, params)
            b.record()
            b.synchronize()
            step_ms.append(a.elapsed_time(b))
            launches += res.gpu_launches
            results = [res]                   # keep one: retained device buffers would
                                              # force fresh allocations inside timed steps
        gc.enable()
        barrier()
    t_step = float(np.mean(step_ms))
    if ws > 1:
        tt = torch.tensor([t_step], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    value = t_step / 1e3 / ws          # seconds per clustering across the job

    # ---- per-kernel rooflines (live, CUDA events on the launching stream)
    hbm, bf16, src = peaks()
    res = results[-1]
    n, d = inst.X.shape
    K = prep.K
    knn_ms = time_kernel(lambda: knn_search_exact_device(prep.x_dev, K, integer=prep.x_level), 3)
    knn_flops = 2.0 * n * n * d
    fp8 = prep.x_level == 2
    tc_peak = 4500.0 if fp8 else bf16
    tc_peak_src = ("nominal fp8 dense, B200_PROFILING.md (no measured fp8 peak)" if fp8
                   else f"{src} bf16 burst, MEASURED_PEAKS.json")
    op = res.operator
    c = inst.k + 1
    q = padded(torch.randn(n, c, dtype=torch.float64), torch.float32)
    z = torch.empty_like(q)
    scr = op.scratch(c, torch.float32)
    s32 = op.struct(_lib.F32)

    def apply():
        _lib.call("ancka_op_apply", s32, q.data_ptr(), q.stride(0), c, z.data_ptr(),
                  z.stride(0), scr.data_ptr(), _lib.stream())
    spmm_ms = time_kernel(apply, 50)
    spmm_bytes = spmm_gbytes_model(op, c, op.p_k_dev.nnz)
    phases = {k: round(v, 3) for k, v in res.timings_ms.items()}
    gpu_calls = {"ortho": res.iterations, "discretize": res.iterations // 5,
                 "mhc": res.iterations // 5 + 1}
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("knn_tc_kernel_dram_bytes")
    roofline = {"kernel": "knn_tc_kernel (tcgen05 exact KNN, fp8 e4m3)" if fp8 else "knn",
                "bound": "tensor", "achieved": round(knn_flops / (knn_ms * 1e-3) / 1e12, 2),
                "peak": tc_peak, "unit": "TFLOP/s",
                "frac": round(knn_flops / (knn_ms * 1e-3) / 1e12 / tc_peak, 4),
                "traffic": traffic, "peak_source": tc_peak_src,
                "algorithmic": f"2*n^2*d = {knn_flops:.3e} FLOP per launch",
                "duration_ms": round(knn_ms, 3)}
    spmm = {"kernel": "spmm_kernel<float> (hypergraph P_E then P_V+P_K stage)", "bound": "hbm",
            "achieved": round(spmm_bytes / (spmm_ms * 1e-3) / 1e9, 1), "peak": hbm,
            "unit": "GB/s", "frac": round(spmm_bytes / (spmm_ms * 1e-3) / 1e9 / hbm, 4),
            "algorithmic": f"gather model {spmm_bytes} B per apply (SURVEY.md §8(d))",
            "duration_ms": round(spmm_ms, 4), "peak_source": f"{src} HBM copy"}

    # fused orthogonal block (tau = 5 steps per launch): SpMM gather model +
    # CholQR 12 n c bytes per step
    from paper_2408_05459_b200 import engine as eng
    loop = eng._Loop(op, c, inst.k, 5, True, True)
    loop.Q[0][:, :c] = torch.randn(n, c, device="cuda")
    orth_ms = time_kernel(lambda: loop.run(5), 5)
    orth_bytes = 5 * (spmm_bytes + 12 * n * c)
    orth_traffic = None
    if tf.exists():
        per_step = json.loads(tf.read_text()).get("orth_fused_kernel_dram_bytes_per_step")
        orth_traffic = None if per_step is None else 5 * per_step
    orth = {"kernel": "orth_fused_kernel (cooperative: 5 x [SpMM + Gram + Cholesky + R^-1 apply])",
            "bound": "hbm", "achieved": round(orth_bytes / (orth_ms * 1e-3) / 1e9, 1),
            "peak": hbm, "unit": "GB/s",
            "frac": round(orth_bytes / (orth_ms * 1e-3) / 1e9 / hbm, 4), "traffic": orth_traffic,
            "algorithmic": f"5 x (gather model {spmm_bytes} B + 12nc = {12 * n * c} B) per launch",
            "duration_ms": round(orth_ms, 4), "peak_source": f"{src} HBM copy",
            "note": "grid-barrier / latency bound at this size: the working set sits in L2"}
    # the headline roofline is the kernel family with the largest share of the step
    share = {"ortho_ms": orth, "knn_ms": roofline}
    dom = max(share, key=lambda k2: phases.get(k2, 0.0))
    rooflines = {"orth_fused": orth, "knn_tc": roofline, "spmm": spmm}
    roofline_main = share[dom] | {"share_of_step": round(phases.get(dom, 0.0) / t_step, 3)}

    # ---- end-to-end through the public API from host inputs
    e2e = None
    if not args.no_e2e:
        e2e_t = []
        ancka.run_ancka(net, params)          # untimed warm-up of the host path
        for _ in range(5):
            barrier()
            gc.collect()
            t0 = time.perf_counter()
            r2 = ancka.run_ancka(net, params)
            lab = r2.y.assignment  # host labels
            torch.cuda.synchronize()
            e2e_t.append(time.perf_counter() - t0)
        te = float(np.median(e2e_t))
        if ws > 1:
            tt = torch.tensor([te], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        if os.environ.get("ANCKA_BENCH_DEBUG"):
            print("e2e runs (s):", [round(x, 4) for x in e2e_t], "last timings:", r2.timings_ms,
                  file=sys.stderr)
        e2e = {"value": round(te / ws, 4), "unit": "s",
               "h2d_bytes_per_step": prep.h2d_bytes(inst.X),
               "d2h_bytes_per_step": int(lab.size * 4 + 8 * 4 * (r2.iterations // 5 + 2)),
               "runs_s": [round(x, 4) for x in e2e_t],
               "note": "median of 5 host wall-clock runs of run_ancka(net, params) incl. host "
                       "validation, pageable H2D uploads and the label read-back"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        t_cpu, ref = oracle_run(inst, args.seed)
        from sklearn.metrics import adjusted_rand_score
        cpu = {"value": round(t_cpu, 3), "unit": "s", "cores": cpu_threads(), "kind": "port",
               "sample": f"one full {SHAPE}-shaped clustering with the numpy/scipy restatement "
                         f"of the reference (oracle/ancka_cpu.py), same instance",
               "ari_vs_gpu": round(float(adjusted_rand_score(ref["labels"], res.y.assignment)), 4),
               "iterations": ref["iterations"],
               "phases_ms": {k2: round(v, 1) for k2, v in ref["timings_ms"].items()},
               "per_call_ms": per_call(ref["timings_ms"], ref["calls"]),
               "gpu_per_call_ms": per_call(phases, gpu_calls)}
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 5), "unit": "s", "n_gpus": ws,
                "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": round(t_step, 3), "step_ms": [round(x, 3) for x in step_ms],
                "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": workload_config(inst, K) | {"parallelism": f"replicas x{ws}"},
                "knn_build_s": round(res.timings_ms["knn_ms"] / 1e3, 5),
                "spmm_hbm_gbs": spmm["achieved"], "roofline": roofline_main,
                "rooflines": rooflines,
                "phases_ms": phases, "iterations": res.iterations, "stop_reason": res.stop_reason,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
