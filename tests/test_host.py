"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; host-side boundary logic mirrors the oracle."""
from __future__ import annotations

import ctypes
import re
import warnings
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, load_csr, oracle_net, random_seeds
from oracle import ancka_cpu as oc

warnings.simplefilter("ignore")


def _header_symbols():
    text = (ROOT / "include" / "ancka_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|int64_t|size_t|void)\s+(ancka_\w+)\(", text, re.M)))


def test_library_builds_and_exports():
    from paper_2408_05459_b200 import _lib
    from paper_2408_05459_b200.build import build
    build()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = _header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.exported_symbols())
    lib.ancka_abi_version.restype = ctypes.c_int
    assert lib.ancka_abi_version() == 1


def test_no_gpu_raises_loudly():
    import torch
    from paper_2408_05459_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        _lib.require_device()


def test_validate_and_degrees_match_oracle(golden_random):
    import paper_2408_05459_b200 as ancka
    z = golden_random
    for s in random_seeds(z):
        p = f"s{s}_"
        if bool(z[p + "skip"]):
            continue
        on = oc.clean_network(oracle_net(z, p))
        kind = str(z[p + "kind"])
        if kind == "multiplex":
            net = ancka.AttributedNetwork.multiplex(on["layers"], on["X"])
        elif kind == "hypergraph":
            net = ancka.AttributedNetwork.hypergraph(load_csr(z, p + "S"), on["X"])
        else:
            net = ancka.AttributedNetwork.graph(load_csr(z, p + "S"), on["X"],
                                                directed=bool(z[p + "directed"]))
        net, _ = ancka.validate_network(net)
        np.testing.assert_array_equal(ancka.node_degrees(net), oc.structural_degree(on))


def test_centers_match_reference_rule():
    from paper_2408_05459_b200.engine import _centers
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(5, 60))
        deg = rng.integers(0, 5, size=n).astype(float)
        k = int(rng.integers(1, n + 1))
        ref_order = np.lexsort((np.arange(n), -deg))
        nz = int((deg > 0).sum())
        if k > nz:
            chosen = list(ref_order[:nz])
            rest = [i for i in range(n) if i not in set(chosen)]
            ref = np.sort(np.array(chosen + rest[: k - nz]))
        else:
            ref = np.sort(ref_order[:k])
        assert np.array_equal(_centers(deg, k), ref)


def test_cache_roundtrip(tmp_path):
    from paper_2408_05459_b200 import knn
    ids = np.array([[1, -1], [0, 2], [1, 0]])
    sc = np.array([[0.5, 0], [0.5, 0.25], [0.25, 0.125]])
    nl = knn.NeighborLists.from_host(ids, sc)
    f = tmp_path / "x.aknn"
    knn.save_neighbor_cache(f, nl, knn.KnnMode.EXACT)
    back, mode = knn.load_neighbor_cache(f)
    assert np.array_equal(back.ids, ids) and np.allclose(back.scores, sc)


def test_integer_exact_detection():
    import scipy.sparse as sp
    from paper_2408_05459_b200.knn import integer_exact
    assert integer_exact(sp.csr_matrix(np.eye(4))) == 2
    assert integer_exact(np.array([[100.0, 1.0]])) == 1
    assert integer_exact(np.array([[0.5, 1.0]])) == 0
    assert integer_exact(np.array([[300.0, 1.0]])) == 0
