"""Binary-format load time at scale.

    python tools/load_scale.py papers100m 0.125 /tmp/p100m8

Writes the synthetic instance with io_binary.save_network, then times
io_binary.load_network (mapped arrays, in-place validation) and the host
validation run_ancka performs (validate_network).  The files are in the page
cache after the write, so this is the warm-cache load."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2408_05459_b200 import io_binary, synth  # noqa: E402
from paper_2408_05459_b200.network import AttributedNetwork, validate_network  # noqa: E402

name, scale, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
t0 = time.perf_counter()
inst = synth.make(name, seed=0, scale=scale)
t_gen = time.perf_counter() - t0
t0 = time.perf_counter()
net = (AttributedNetwork.hypergraph if inst.kind == "hypergraph" else AttributedNetwork.graph)(
    inst.structure, inst.X)
t_ctor = time.perf_counter() - t0
t0 = time.perf_counter()
io_binary.save_network(out, net, labels=inst.labels)
t_save = time.perf_counter() - t0
del net, inst
t0 = time.perf_counter()
back, lab = io_binary.load_network(out)
t_load = time.perf_counter() - t0
t0 = time.perf_counter()
validate_network(back)
t_val = time.perf_counter() - t0
s = back.incidence if back.incidence is not None else back.adjacency
size = sum(p.stat().st_size for p in Path(out).iterdir())
print(json.dumps({"shape": name, "scale": scale, "n": back.n, "nnz": int(s.nnz),
                  "bytes_on_disk": size, "gen_s": round(t_gen, 2),
                  "in_memory_ctor_s": round(t_ctor, 2), "save_s": round(t_save, 2),
                  "load_s": round(t_load, 2), "validate_network_s": round(t_val, 2)}))
