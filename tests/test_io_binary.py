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
