"""Binary network format round trips -- CPU only."""
import numpy as np
import scipy.sparse as sp

from paper_2408_05459_b200 import io_binary, synth
from paper_2408_05459_b200.network import AttributedNetwork


def _same(a, b):
    return (sp.csr_matrix(a) != sp.csr_matrix(b)).nnz == 0


def test_roundtrip_hypergraph_graph_multiplex(tmp_path):
    hg = synth.make("dblp", seed=1, n=300)
    net = AttributedNetwork.hypergraph(hg.structure, hg.X)
    io_binary.save_network(tmp_path / "hg", net, labels=hg.labels)
    back, lab = io_binary.load_network(tmp_path / "hg")
    assert back.kind is net.kind and back.n == net.n
    assert _same(back.incidence, net.incidence) and _same(back.attributes, net.attributes)
    assert np.array_equal(lab, hg.labels)

    g = synth.make("amazon2m", seed=2, n=250)
    net = AttributedNetwork.graph(g.structure, g.X, directed=True)
    io_binary.save_network(tmp_path / "g", net)
    back, lab = io_binary.load_network(tmp_path / "g", mmap=False)
    assert back.directed and lab is None
    assert _same(back.adjacency, net.adjacency)
    np.testing.assert_array_equal(np.asarray(back.attributes), net.attributes)

    layers = [sp.csr_matrix(g.structure), sp.csr_matrix(g.structure.T)]
    net = AttributedNetwork.multiplex(layers, g.X)
    io_binary.save_network(tmp_path / "m", net)
    back, _ = io_binary.load_network(tmp_path / "m")
    assert len(back.layers) == 2 and all(_same(a, b) for a, b in zip(back.layers, net.layers))


def test_load_validates_in_place_and_canonicalises_otherwise(tmp_path):
    """A canonical file is mapped, not copied; a non-canonical one (unsorted
    indices, explicit zeros, duplicates) is canonicalised as the reference's
    check_sparse_nonneg does (network.py:43-63)."""
    g = synth.make("amazon2m", seed=3, n=400)
    net = AttributedNetwork.graph(g.structure, g.X)
    io_binary.save_network(tmp_path / "c", net)
    back, _ = io_binary.load_network(tmp_path / "c")
    assert isinstance(back.adjacency.data, np.memmap) or back.adjacency.data.base is not None
    assert not back.adjacency.data.flags.writeable          # still the mapped file
    assert _same(back.adjacency, net.adjacency)

    a = sp.csr_matrix(net.adjacency, copy=True)
    # reverse each row's column order and store one explicit zero
    for r in range(a.shape[0]):
        s, e = a.indptr[r], a.indptr[r + 1]
        a.indices[s:e] = a.indices[s:e][::-1].copy()
        a.data[s:e] = a.data[s:e][::-1].copy()
    a.data[0] = 0.0
    a.has_sorted_indices = False
    io_binary._save_csr(tmp_path / "c", "structure", a)
    back, _ = io_binary.load_network(tmp_path / "c")
    ref = sp.csr_matrix(net.adjacency, copy=True)
    ref.data[ref.indptr[0]:ref.indptr[1]][-1] = 0.0       # the same stored zero
    ref.eliminate_zeros()
    assert back.adjacency.has_canonical_format
    assert _same(back.adjacency, ref)


def test_cli_gen_and_config(tmp_path):
    import json

    from paper_2408_05459_b200 import cli
    from paper_2408_05459_b200.network import ClusterParams, NetworkError

    rc = cli.main(["gen", "--shape", "citeseer", "--n", "300", "--out", str(tmp_path / "cs")])
    assert rc == cli.EXIT_OK
    meta = json.loads((tmp_path / "cs" / "meta.json").read_text())
    assert meta["kind"] == "hypergraph" and meta["n"] == 300 and meta["labels"]
    cfg = cli.RunConfig(net_dir=str(tmp_path / "cs"), params=ClusterParams(k=6))
    net, lab = cli.load_network_from_config(cfg)
    assert net.n == 300 and lab.shape == (300,)
    assert cfg.to_dict()["k"] == 6 and cfg.to_dict()["knn_mode"] == "auto"
    try:
        cli.RunConfig(net_dir=str(tmp_path / "missing"), params=ClusterParams(k=2))
        raise AssertionError("missing directory accepted")
    except NetworkError:
        pass
    rc = cli.main(["run", "--net-dir", str(tmp_path / "missing"), "-k", "2", "-o",
                   str(tmp_path / "r.json")])
    assert rc == cli.EXIT_VALIDATION
