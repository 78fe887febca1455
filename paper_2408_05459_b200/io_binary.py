"""Binary network format for large inputs.

The reference reads hyperedge-per-line / edge-list / TSV text
(`io.py:66-202`), which cannot feed 1e8-node inputs in reasonable time.
This module stores the same content as raw arrays in a directory:

    meta.json                  kind, n, directed, n_layers, attribute layout
    structure_{indptr,indices,data}.npy     (graph / hypergraph)
    layer{i}_{indptr,indices,data}.npy      (multiplex)
    attributes.npy | attributes_{indptr,indices,data}.npy
    labels.npy                 (optional)

`load_network` memory-maps the arrays (no parse step) and validates them in
place: a canonical CSR (what `save_network` writes) is checked with one read
of its arrays and never copied; anything else is canonicalised exactly as
for any other input.  `cli.py` is the RunConfig / command-line driver on
top (reference cli.py:86-128, io.py:426-517).  `save_network` mirrors the reference's
`io.save_network(out_dir, net, labels)` (`io.py:384-418`).
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import scipy.sparse as sp

from .network import AttributedNetwork, NetworkError, NetworkKind

FORMAT = "ancka-b200-binary/1"


def _save_csr(out: Path, stem: str, m: sp.csr_matrix) -> None:
    m = sp.csr_matrix(m)
    np.save(out / f"{stem}_indptr.npy", m.indptr.astype(np.int64))
    np.save(out / f"{stem}_indices.npy", m.indices.astype(np.int32))
    np.save(out / f"{stem}_data.npy", m.data.astype(np.float64))


def _load_csr(src: Path, stem: str, shape, mmap: bool) -> sp.csr_matrix:
    mode = "r" if mmap else None
    ip = np.load(src / f"{stem}_indptr.npy", mmap_mode=mode)
    ix = np.load(src / f"{stem}_indices.npy", mmap_mode=mode)
    dv = np.load(src / f"{stem}_data.npy", mmap_mode=mode)
    return sp.csr_matrix((dv, ix, ip), shape=tuple(shape), copy=False)


def save_network(out_dir, net: AttributedNetwork, labels=None) -> dict:
    """Write `net` (and optional labels) in the binary layout; returns the file map."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    meta = {"format": FORMAT, "kind": net.kind.value, "n": int(net.n),
            "directed": bool(net.directed)}
    if net.kind is NetworkKind.HYPERGRAPH:
        _save_csr(out, "structure", net.incidence)
        meta["structure_shape"] = list(net.incidence.shape)
    elif net.kind is NetworkKind.GRAPH:
        _save_csr(out, "structure", net.adjacency)
        meta["structure_shape"] = list(net.adjacency.shape)
    else:
        for i, a in enumerate(net.layers):
            _save_csr(out, f"layer{i}", a)
        meta["n_layers"] = len(net.layers)
    x = net.attributes
    if sp.issparse(x):
        _save_csr(out, "attributes", x)
        meta["attributes"] = {"layout": "csr", "shape": list(x.shape)}
    else:
        np.save(out / "attributes.npy", np.ascontiguousarray(x, dtype=np.float64))
        meta["attributes"] = {"layout": "dense", "shape": list(np.shape(x))}
    if labels is not None:
        np.save(out / "labels.npy", np.asarray(labels, dtype=np.int64))
        meta["labels"] = True
    (out / "meta.json").write_text(json.dumps(meta, indent=1))
    return {"dir": str(out), **meta}


def load_network(src_dir, mmap: bool = True):
    """Read a network written by `save_network`: (AttributedNetwork, labels | None)."""
    src = Path(src_dir)
    try:
        meta = json.loads((src / "meta.json").read_text())
    except FileNotFoundError as exc:
        raise NetworkError(f"{src}: no meta.json (not a binary network directory)") from exc
    if meta.get("format") != FORMAT:
        raise NetworkError(f"{src}: unsupported format {meta.get('format')!r}")
    n = int(meta["n"])
    a = meta["attributes"]
    if a["layout"] == "csr":
        x = _load_csr(src, "attributes", a["shape"], mmap)
    else:
        x = np.load(src / "attributes.npy", mmap_mode="r" if mmap else None)
    kind = NetworkKind(meta["kind"])
    if kind is NetworkKind.HYPERGRAPH:
        net = AttributedNetwork.hypergraph(_load_csr(src, "structure", meta["structure_shape"],
                                                     mmap), x, copy=False)
    elif kind is NetworkKind.GRAPH:
        net = AttributedNetwork.graph(_load_csr(src, "structure", meta["structure_shape"], mmap),
                                      x, directed=bool(meta["directed"]), copy=False)
    else:
        layers = [_load_csr(src, f"layer{i}", (n, n), mmap) for i in range(int(meta["n_layers"]))]
        net = AttributedNetwork.multiplex(layers, x, copy=False)
    labels = np.load(src / "labels.npy") if meta.get("labels") else None
    return net, labels
