"""Seeded synthetic attributed networks of the shapes named in BASELINE.json.

SURVEY.md §8(d): planted-partition structure with a random node-id
permutation (no locality), binary bag-of-words attributes for the
Cora/Citeseer/DBLP/MAG-PM shapes and |N(mu_block, I)| continuous attributes
for the Amazon2M/Papers100M shapes.  Everything is vectorised numpy so the
multi-million-node shapes generate in seconds.

The reference's own generator (ancka/io.py:304-343) cannot produce these
shapes (fixed 3n size-3 hyperedges, O(n^2) pair sampling), hence this module.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

# name -> (kind, n, m, d, k, attrs, words)
SHAPES = {
    "cora": ("graph", 2708, 5429, 1433, 7, "binary", 18),
    "citeseer": ("hypergraph", 3312, 1079, 3703, 6, "binary", 32),
    "dblp": ("hypergraph", 41302, 22363, 1425, 6, "binary", 20),
    "magpm": ("hypergraph", 2353996, 1082711, 1000, 22, "binary", 20),
    "amazon2m": ("graph", 2449029, 61859140, 100, 47, "continuous", 0),
    "papers100m": ("graph", 111059956, 1615685872, 128, 172, "continuous", 0),
}


@dataclass
class Synthetic:
    kind: str
    structure: sp.csr_matrix       # A (n x n) or H (m x n)
    X: object                      # csr (binary) or ndarray (continuous)
    labels: np.ndarray             # planted partition, int64[n]
    k: int
    name: str = ""


def _planted(rng, n, k):
    lab = rng.integers(0, k, size=n)
    lab[:k] = np.arange(k)
    return lab[rng.permutation(n)].astype(np.int64)


def _members(lab, k):
    order = np.argsort(lab, kind="stable")
    bounds = np.searchsorted(lab[order], np.arange(k + 1))
    return order, bounds


def _draw_in_block(rng, lab, order, bounds, blocks, count):
    """`count` uniform members of each given block (vectorised)."""
    lo = bounds[blocks]
    size = bounds[blocks + 1] - lo
    off = (rng.random((blocks.size, count)) * size[:, None]).astype(np.int64)
    return order[lo[:, None] + off]


def graph_structure(rng, lab, k, m_edges, p_in=0.8):
    n = lab.size
    order, bounds = _members(lab, k)
    intra = rng.random(m_edges) < p_in
    u = rng.integers(0, n, size=m_edges)
    v = rng.integers(0, n, size=m_edges)
    if intra.any():
        v[intra] = _draw_in_block(rng, lab, order, bounds, lab[u[intra]], 1)[:, 0]
    keep = u != v
    u, v = u[keep], v[keep]
    a = sp.csr_matrix((np.ones(u.size), (u, v)), shape=(n, n))
    a = ((a + a.T) > 0).astype(np.float64).tocsr()
    a.sort_indices()
    return a


def hypergraph_structure(rng, lab, k, m_edges, mean_size=4.0, p_in=0.8):
    n = lab.size
    order, bounds = _members(lab, k)
    sizes = 2 + rng.poisson(mean_size - 2.0, size=m_edges)
    smax = int(sizes.max())
    seed_nodes = rng.integers(0, n, size=m_edges)
    inside = rng.random(m_edges) < p_in
    cand = rng.integers(0, n, size=(m_edges, smax))
    if inside.any():
        cand[inside] = _draw_in_block(rng, lab, order, bounds, lab[seed_nodes[inside]], smax)
    cand[:, 0] = seed_nodes
    valid = np.arange(smax)[None, :] < sizes[:, None]
    rows = np.repeat(np.arange(m_edges), valid.sum(axis=1))
    h = sp.csr_matrix((np.ones(rows.size), (rows, cand[valid])), shape=(m_edges, n))
    h.data[:] = 1.0                  # duplicates inside an edge collapse to one
    h.sort_indices()
    return h


def binary_bag_of_words(rng, lab, k, d, words):
    """Half the words from a block-specific vocabulary, half global; Zipf."""
    n = lab.size
    per = max(words, 2)
    vocab = max(d // (2 * k), 4)
    ranks = np.arange(1, d + 1, dtype=np.float64)
    zipf = 1.0 / ranks
    zipf /= zipf.sum()
    glob = rng.choice(d, size=(n, per // 2), p=zipf)
    local_rank = rng.choice(vocab, size=(n, per - per // 2), p=zipf[:vocab] / zipf[:vocab].sum())
    block_base = (lab * vocab) % max(d - vocab, 1)
    local = (block_base[:, None] + local_rank) % d
    cols = np.concatenate([glob, local], axis=1)
    rows = np.repeat(np.arange(n), cols.shape[1])
    x = sp.csr_matrix((np.ones(rows.size), (rows, cols.ravel())), shape=(n, d))
    x.data[:] = 1.0
    x.sort_indices()
    return x


def continuous_attributes(rng, lab, k, d, spread=1.0):
    mu = rng.normal(0.0, 2.0, size=(k, d))
    x = np.abs(mu[lab] + spread * rng.standard_normal((lab.size, d)))
    return x


def make(name, seed=0, n=None, scale=1.0, p_in=0.8, words=None):
    """Synthetic instance of a named shape (optionally rescaled to n nodes)."""
    kind, n0, m0, d, k, attrs, w0 = SHAPES[name]
    if n is None:
        n = int(round(n0 * scale))
    m = max(2, int(round(m0 * n / n0)))
    rng = np.random.default_rng(seed)
    lab = _planted(rng, n, k)
    if kind == "graph":
        s = graph_structure(rng, lab, k, m, p_in=p_in)
    else:
        s = hypergraph_structure(rng, lab, k, m, p_in=p_in)
    if attrs == "binary":
        x = binary_bag_of_words(rng, lab, k, d, words if words is not None else w0)
    else:
        x = continuous_attributes(rng, lab, k, d)
    return Synthetic(kind=kind, structure=s, X=x, labels=lab, k=k, name=name)
