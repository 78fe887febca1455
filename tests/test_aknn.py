"""`.aknn` neighbour-cache wire format (SURVEY.md §8(f) row f1,
knn.py:327-382 of the reference) against files and keys written by the
reference itself (tests/golden/make_golden.py `aknn_cache`)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from conftest import load_x
from oracle import ancka_cpu as oc

ancka = pytest.importorskip("paper_2408_05459_b200")
from paper_2408_05459_b200 import knn  # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "aknn.json").read_text())
Z = np.load(GOLD / "aknn.npz")


@pytest.mark.parametrize("name", sorted(META))
def test_cache_key_matches_reference(name):
    x = load_x(Z, name)
    m = META[name]
    assert knn.cache_key(x, m["K"], knn.KnnMode.EXACT) == m["key_exact"]
    assert knn.cache_key(x, m["K"], knn.KnnMode.APPROX) == m["key_approx"]


@pytest.mark.parametrize("name", sorted(META))
def test_reader_writer_byte_identical(name, tmp_path):
    src = GOLD / META[name]["file"]
    nl, mode = knn.load_neighbor_cache(src)
    assert mode is knn.KnnMode.EXACT and nl.ids.shape[1] == META[name]["K"]
    out = tmp_path / "x.aknn"
    knn.save_neighbor_cache(out, nl, mode)
    assert out.read_bytes() == src.read_bytes()


def test_reference_file_matches_oracle_lists():
    """Continuous attributes (no exact ties): the reference's cached lists are
    the oracle's exact lists, scores rounded to f32."""
    x = load_x(Z, "dense")
    nl, _ = knn.load_neighbor_cache(GOLD / META["dense"]["file"])
    ids, sc = oc.knn_exact(x, META["dense"]["K"])
    assert np.array_equal(nl.ids, ids)
    np.testing.assert_array_equal(nl.scores, sc.astype(np.float32).astype(np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(META))
def test_device_knn_written_cache_matches_reference(name, tmp_path):
    """The device KNN's lists written through the cache equal the reference's
    file: ids exact (binary X: up to exact ties at the K-th value), f32 scores
    within one f32 rounding."""
    from test_gpu_parity import knn_sets_match
    x = load_x(Z, name)
    K = META[name]["K"]
    nl = knn.knn_search_exact(x, K)
    f = tmp_path / f"{knn.cache_key(x, K, knn.KnnMode.EXACT)}.aknn"
    knn.save_neighbor_cache(f, nl, knn.KnnMode.EXACT)
    assert f.stem == META[name]["key_exact"]
    ours, _ = knn.load_neighbor_cache(f)
    ref, _ = knn.load_neighbor_cache(GOLD / META[name]["file"])
    if name == "dense":
        assert np.array_equal(ours.ids, ref.ids)
    else:
        assert knn_sets_match(ours.ids, ref.ids, x, K) == 0
    np.testing.assert_allclose(np.sort(ours.scores, axis=1), np.sort(ref.scores, axis=1),
                               rtol=2 ** -23, atol=0)
