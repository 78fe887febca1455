"""Shared test helpers.  `-m gpu` tests need a B200; everything else runs on CPU."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_csr(z, prefix):
    shape = tuple(int(v) for v in z[prefix + "_shape"])
    return sp.csr_matrix((z[prefix + "_data"], z[prefix + "_indices"], z[prefix + "_indptr"]),
                         shape=shape)


def load_x(z, prefix):
    if prefix + "_dense" in z:
        return z[prefix + "_dense"]
    return load_csr(z, prefix + "_csr")


@pytest.fixture(scope="session")
def golden_random():
    return np.load(GOLDEN / "random_instances.npz")


@pytest.fixture(scope="session")
def golden_spec():
    return np.load(GOLDEN / "spec_examples.npz")


@pytest.fixture(scope="session")
def golden_runs():
    z = np.load(GOLDEN / "end_to_end.npz")
    meta = json.loads((GOLDEN / "end_to_end.json").read_text())
    return z, meta


def random_seeds(z):
    return sorted({int(k[1:].split("_")[0]) for k in z.files if k.startswith("s")})


def load_layers(z, p):
    return [load_csr(z, p + f"L{i}") for i in range(int(z[p + "n_layers"]))]


def oracle_net(z, p):
    kind = str(z[p + "kind"])
    if kind == "multiplex":
        return {"kind": kind, "layers": load_layers(z, p), "directed": False,
                "X": load_x(z, p + "X")}
    return {"kind": kind, "S": load_csr(z, p + "S"), "directed": bool(z[p + "directed"]),
            "X": load_x(z, p + "X")}


@pytest.fixture(scope="session")
def golden_multiplex():
    z = np.load(GOLDEN / "multiplex.npz")
    meta = json.loads((GOLDEN / "multiplex.json").read_text())
    return z, meta


@pytest.fixture(scope="session")
def golden_approx():
    z = np.load(GOLDEN / "approx.npz")
    meta = json.loads((GOLDEN / "approx.json").read_text())
    return z, meta
