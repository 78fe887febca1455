"""Run-config and command-line driver over the binary network format
(SURVEY.md §8(f) row f3).

Mirrors the reference's `ancka run | gen | oracle` (cli.py:86-181) and its
`RunConfig` / `load_network_from_config` / `result_document` /
`emit_result` (io.py:426-517), with the text loaders (io.py:66-202)
replaced by `io_binary` directories: memory-mapped CSR and attribute
arrays validated in place, so a 1e8-node input loads in seconds.  The
clustering itself is `engine.run_ancka` on the device.

    python -m paper_2408_05459_b200 gen --shape amazon2m --out /data/amz
    python -m paper_2408_05459_b200 run --net-dir /data/amz -k 47 --knn-k 10 -o result.json

Exit codes as in the reference: 0 success, 2 validation error, 3 runtime
failure.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .network import ClusterParams, KnnMode, NetworkError

EXIT_OK = 0
EXIT_VALIDATION = 2
EXIT_RUNTIME = 3


@dataclass
class RunConfig:
    """io.py:426-465 with `net_paths`/`attr_path`/`labels_path` folded into
    one binary directory (`io_binary.save_network` layout)."""

    net_dir: str
    params: ClusterParams
    output_path: str | None = None
    metrics: tuple = ("ari", "nmi")
    knn_cache_dir: str | None = None
    mmap: bool = True
    extra: dict = field(default_factory=dict)

    def __post_init__(self):
        if not (Path(self.net_dir) / "meta.json").exists():
            raise NetworkError(f"file not found: {Path(self.net_dir) / 'meta.json'}")

    def to_dict(self) -> dict:
        p = self.params
        return {
            "net_dir": str(self.net_dir),
            "k": p.k, "alpha": p.alpha, "beta": p.beta, "gamma": p.gamma,
            "knn_k": p.knn_k, "eps_q": p.eps_q, "t_a": p.t_a, "t_i": p.t_i,
            "tau": p.tau, "seed": p.seed, "knn_mode": p.knn_mode.value,
            "metrics": list(self.metrics),
        }


def load_network_from_config(config: RunConfig):
    """io.py:468-485 for the binary layout: (AttributedNetwork, labels | None)."""
    from . import io_binary
    return io_binary.load_network(config.net_dir, mmap=config.mmap)


def score(labels_true, labels_pred, names) -> dict:
    """The reference's metrics.score_all subset used by `run` (sklearn's
    definitions; host-side, O(n))."""
    from sklearn import metrics as skm
    fns = {"ari": skm.adjusted_rand_score, "nmi": skm.normalized_mutual_info_score}
    return {k: float(fns[k](labels_true, labels_pred)) for k in names if k in fns}


def result_document(result, config: RunConfig, metrics: dict | None, total_ms: float,
                    load_ms: float | None = None) -> dict:
    """io.py:488-510 (same keys), plus `load_ms` for the binary load."""
    from . import __version__
    doc = {
        "version": __version__,
        "k": result.y.k,
        "assignment": result.y.assignment.tolist(),
        "mhc": result.mhc,
        "iterations": result.iterations,
        "timings_ms": {key: round(val, 3) for key, val in result.timings_ms.items()},
        "total_ms": round(total_ms, 3),
        "converged": result.converged,
        "stop_reason": result.stop_reason,
        "config": config.to_dict(),
    }
    if load_ms is not None:
        doc["load_ms"] = round(load_ms, 3)
    if metrics is not None:
        doc["metrics"] = metrics
    if result.warnings:
        doc["warnings"] = result.warnings
    if result.error:
        doc["error"] = result.error
    return doc


def emit_result(doc: dict, path) -> None:
    """io.py:513-517."""
    try:
        with open(path, "w") as fh:
            json.dump(doc, fh, indent=2)
            fh.write("\n")
    except OSError as exc:
        raise NetworkError(f"cannot write result to {path}: {exc}") from exc


def run_config(config: RunConfig):
    """The `run` command's body (cli.py:86-128): load, cluster, score, emit.
    Returns (ClusterResult, document)."""
    from . import engine
    t0 = time.perf_counter()
    net, labels = load_network_from_config(config)
    load_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    result = engine.run_ancka(net, config.params, knn_cache_dir=config.knn_cache_dir)
    total_ms = (time.perf_counter() - t0) * 1e3
    scored = score(labels, result.y.assignment, config.metrics) if labels is not None else None
    doc = result_document(result, config, scored, total_ms, load_ms)
    if config.output_path:
        emit_result(doc, config.output_path)
    return result, doc


def _params_from(args) -> ClusterParams:
    return ClusterParams(k=args.k, alpha=args.alpha, beta=args.beta, gamma=args.gamma,
                         knn_k=args.knn_k, eps_q=args.eps_q, t_a=args.t_a, t_i=args.t_i,
                         tau=args.tau, seed=args.seed, knn_mode=KnnMode(args.knn_mode))


def _add_param_args(p: argparse.ArgumentParser) -> None:
    """cli.py:29-43 (same flags and defaults)."""
    p.add_argument("-k", type=int, required=True, help="number of clusters")
    p.add_argument("--knn-k", type=int, default=None)
    p.add_argument("--alpha", type=float, default=0.2)
    p.add_argument("--beta", type=float, default=0.5)
    p.add_argument("--gamma", type=int, default=3)
    p.add_argument("--eps-q", type=float, default=0.005)
    p.add_argument("--t-a", type=int, default=1000)
    p.add_argument("--t-i", type=int, default=25)
    p.add_argument("--tau", type=int, default=5)
    p.add_argument("--knn-mode", choices=["auto", "exact", "approx"], default="auto")
    p.add_argument("--seed", type=int, default=0)


def _cmd_run(args) -> int:
    config = RunConfig(net_dir=args.net_dir, params=_params_from(args),
                       output_path=args.output, knn_cache_dir=args.knn_cache,
                       mmap=not args.no_mmap)
    result, doc = run_config(config)
    for w in result.warnings:
        print(f"warning: {w}", file=sys.stderr)
    line = (f"mhc={result.mhc:.6f} iterations={result.iterations} stop={result.stop_reason} "
            f"load_ms={doc['load_ms']:.1f} total_ms={doc['total_ms']:.1f}")
    if doc.get("metrics"):
        line += " " + " ".join(f"{k}={v:.4f}" for k, v in doc["metrics"].items())
    print(line)
    print(f"result: {config.output_path}")
    if result.error:
        print(f"error: {result.error}", file=sys.stderr)
        return EXIT_RUNTIME
    return EXIT_OK


def _cmd_gen(args) -> int:
    """Synthetic instance of a named BASELINE shape (`synth.make`) written in
    the binary layout (the reference's `gen`, cli.py:131-143, writes text)."""
    from . import io_binary, synth
    from .network import AttributedNetwork
    inst = synth.make(args.shape, seed=args.seed, n=args.n,
                      scale=1.0 if args.scale is None else args.scale)
    if inst.kind == "hypergraph":
        net = AttributedNetwork.hypergraph(inst.structure, inst.X)
    else:
        net = AttributedNetwork.graph(inst.structure, inst.X)
    files = io_binary.save_network(args.out, net, labels=inst.labels)
    files["k"] = inst.k
    print(json.dumps(files, indent=1))
    return EXIT_OK


def _cmd_oracle(args) -> int:
    """cli.py:146-181: score a given assignment with the dense brute-force
    conductance beside the iterative one (small inputs only)."""
    from . import engine, walk
    from .network import BcmMatrix
    config = RunConfig(net_dir=args.net_dir, params=_params_from(args), output_path=args.output)
    net, labels = load_network_from_config(config)
    if labels is None:
        raise NetworkError("oracle mode needs labels.npy with the assignment to score")
    _, compact = np.unique(labels, return_inverse=True)
    y = BcmMatrix(assignment=compact, k=int(compact.max()) + 1)
    op, _, _ = engine.build_pipeline(net, config.params)
    dense_value = walk.brute_mhc_oracle(op, y)
    iterative_value = engine.calc_mhc(op, y)
    doc = {"n": net.n, "k": y.k, "mhc_oracle": dense_value, "mhc_iterative": iterative_value,
           "abs_diff": abs(dense_value - iterative_value)}
    if config.output_path:
        emit_result(doc, config.output_path)
    print(json.dumps(doc, indent=2))
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="ancka-b200", description=__doc__.splitlines()[0])
    sub = parser.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="cluster an attributed network (binary directory)")
    run.add_argument("--net-dir", required=True)
    _add_param_args(run)
    run.add_argument("-o", "--output", required=True, help="result JSON path")
    run.add_argument("--knn-cache", default=None, help="neighbour-list cache directory")
    run.add_argument("--no-mmap", action="store_true", help="read the arrays instead of mapping")
    gen = sub.add_parser("gen", help="write a synthetic instance of a named shape")
    gen.add_argument("--shape", required=True)
    gen.add_argument("--n", type=int, default=None)
    gen.add_argument("--scale", type=float, default=None)
    gen.add_argument("--seed", type=int, default=0)
    gen.add_argument("--out", required=True)
    oracle = sub.add_parser("oracle", help="dense brute-force conductance check")
    oracle.add_argument("--net-dir", required=True)
    _add_param_args(oracle)
    oracle.add_argument("-o", "--output", default=None)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    handlers = {"run": _cmd_run, "gen": _cmd_gen, "oracle": _cmd_oracle}
    try:
        return handlers[args.command](args)
    except (NetworkError, FileNotFoundError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION
    except Exception as exc:  # noqa: BLE001 -- CLI boundary
        print(f"runtime failure: {exc}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
