"""Subsystem 2: the joint-walk operator on the B200 (reference: ancka/walk.py).

Structural factors are built on the device from the uploaded structure
(`ancka_csr_row_normalize` / `ancka_csr_transpose` / `ancka_csr_col_scale`,
bit-identical to the reference's scipy normalisation); the KNN factor P_K is
produced on the device by `ancka_knn_graph`.  `apply_joint_transition` and
`apply_structure_rowvec` run `ancka_op_apply` / `ancka_op_apply_struct_t`;
in f64 they are bit-identical to scipy's csr_matvecs.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from ._device import WORKSPACE, DeviceCSR, csr_struct, dev, ld_for, padded
from .network import AttributedNetwork, NetworkError, NetworkKind, node_degrees, symmetrize_union


def _row_normalize(a: sp.csr_matrix) -> sp.csr_matrix:
    """D^-1 A, zero rows stay zero (walk.py:38-44)."""
    rs = np.asarray(a.sum(axis=1)).ravel()
    inv = np.divide(1.0, rs, out=np.zeros_like(rs), where=rs > 0)
    p = (sp.diags(inv) @ a).tocsr()
    p.sort_indices()
    return p


def beta_vector(net: AttributedNetwork, knn_zero_rows, beta: float) -> np.ndarray:
    """beta_i per Eq. (2) (walk.py:47-57)."""
    deg = node_degrees(net)
    b = np.full(net.n, float(beta))
    b[deg == 0] = 1.0
    b[np.asarray(knn_zero_rows, dtype=bool)] = 0.0
    return b


def hypergraph_factors(net: AttributedNetwork):
    """P_V = D_V^-1 H^T, P_E = D_E^-1 H (walk.py:60-71)."""
    if net.kind is not NetworkKind.HYPERGRAPH:
        raise NetworkError("hypergraph_factors requires a hypergraph")
    return _row_normalize(net.incidence.T.tocsr()), _row_normalize(net.incidence)


def graph_transition(net: AttributedNetwork) -> sp.csr_matrix:
    """P_N = D^-1 A, symmetrised for directed input (walk.py:74-79)."""
    if net.kind is not NetworkKind.GRAPH:
        raise NetworkError("graph_transition requires a graph")
    return _row_normalize(symmetrize_union(net.adjacency) if net.directed else net.adjacency)


def multiplex_transition(net: AttributedNetwork):
    """Per-layer transitions P_l = D_l^-1 A_l (walk.py:82-86), host scipy."""
    if net.kind is not NetworkKind.MULTIPLEX:
        raise NetworkError("multiplex_transition requires a multiplex network")
    return [_row_normalize(a) for a in net.layers]


def _upload(m: sp.csr_matrix) -> DeviceCSR:
    d = dev()
    rp = torch.from_numpy(np.ascontiguousarray(m.indptr, dtype=np.int64)).to(d)
    ci = torch.from_numpy(np.ascontiguousarray(m.indices, dtype=np.int32)).to(d)
    v = torch.from_numpy(np.ascontiguousarray(m.data, dtype=np.float64)).to(d)
    return DeviceCSR(m.shape[0], m.shape[1], rp, ci, v, None)


def _with_values(a: DeviceCSR, vals: torch.Tensor) -> DeviceCSR:
    return DeviceCSR(a.rows, a.cols, a.rowptr, a.colidx, vals, vals.to(torch.float32))


def _row_normalize_dev(a: DeviceCSR, want_inv: bool = False):
    out = torch.empty_like(a.val64)
    inv = torch.empty(a.rows, dtype=torch.float64, device=out.device) if want_inv else None
    _lib.call("ancka_csr_row_normalize", a.struct(_lib.F64), out.data_ptr(),
              None if inv is None else inv.data_ptr(), _lib.stream())
    return _with_values(a, out), inv


def _transpose_dev(a: DeviceCSR) -> DeviceCSR:
    d = a.colidx.device
    rp = torch.empty(a.cols + 1, dtype=torch.int64, device=d)
    ci = torch.empty(a.nnz, dtype=torch.int32, device=d)
    v = torch.empty(a.nnz, dtype=torch.float64, device=d)
    wsb = _lib.load().ancka_csr_transpose_workspace_size(a.rows, a.cols, a.nnz)
    ws = WORKSPACE.get("csr_transpose", wsb)
    _lib.call("ancka_csr_transpose", a.struct(_lib.F64), rp.data_ptr(), ci.data_ptr(),
              v.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
    return DeviceCSR(a.cols, a.rows, rp, ci, v, v.to(torch.float32))


class StructureFactors:
    """Structural factors (walk.py:60-79), the init transposes (walk.py:163-165)
    and the pattern degrees, built on the device from one upload of the
    structure.  Host scipy views (`host_view`) are materialised on access."""

    def __init__(self, net: AttributedNetwork, degrees=None):
        self.kind, self.n = net.kind, net.n
        self.degrees = node_degrees(net) if degrees is None else degrees
        self.host, self.dev = {}, {}
        if net.kind is NetworkKind.HYPERGRAPH:
            h = _upload(net.incidence)                      # H  (m x n)
            ht = _transpose_dev(h)                          # H^T (n x m)
            p_e, _ = _row_normalize_dev(h)                  # P_E = D_E^-1 H
            p_v, inv_v = _row_normalize_dev(ht, True)       # P_V = D_V^-1 H^T
            t_a = torch.empty_like(h.val64)                 # P_V^T = H D_V^-1
            _lib.call("ancka_csr_col_scale", h.struct(_lib.F64), inv_v.data_ptr(),
                      t_a.data_ptr(), _lib.stream())
            self.dev.update(p_v=p_v, p_e=p_e, t_a=_with_values(h, t_a), t_b=_transpose_dev(p_e))
            self.m = h.rows
            self._up = h.rowptr.numel() * 8 + h.colidx.numel() * 4 + h.val64.numel() * 8
        elif net.kind is NetworkKind.MULTIPLEX:
            if len(net.layers) > _lib.MAX_LAYERS:
                raise NetworkError(f"multiplex networks support at most {_lib.MAX_LAYERS} layers")
            layers, layers_t, self._up = [], [], 0
            for a in net.layers:                       # P_l = D_l^-1 A_l (walk.py:82-86)
                A = _upload(a)
                p_l, _ = _row_normalize_dev(A)
                layers.append(p_l)
                layers_t.append(_transpose_dev(p_l))
                self._up += A.rowptr.numel() * 8 + A.colidx.numel() * 4 + A.val64.numel() * 8
            self.dev.update(layers=layers, layers_t=layers_t)
            self.m = 0
        else:
            a = symmetrize_union(net.adjacency) if net.directed else net.adjacency
            A = _upload(a)
            p_n, _ = _row_normalize_dev(A)
            self.dev.update(p_n=p_n, t_a=_transpose_dev(p_n))
            self.m = 0
            self._up = A.rowptr.numel() * 8 + A.colidx.numel() * 4 + A.val64.numel() * 8
        self.degrees_dev = torch.from_numpy(self.degrees).to(dev())

    def host_view(self, name: str):
        """scipy CSR of a device factor (p_n, p_v, p_e), materialised once."""
        if name not in self.host and name in self.dev and name in ("p_n", "p_v", "p_e"):
            self.host[name] = self.dev[name].to_scipy()
        return self.host.get(name)

    def h2d_bytes(self) -> int:
        return int(self._up + self.degrees.nbytes)


class WalkOperator:
    """Device-resident joint-walk factors (walk.py:89-104).  The scipy
    attributes of the reference (`p_k`, `p_n`, `p_v`, `p_e`, `beta`,
    `selfloop`) are host views materialised on access."""

    def __init__(self, factors: StructureFactors, p_k_dev: DeviceCSR, beta_vecs, alpha, gamma):
        self.kind, self.n, self.m = factors.kind, factors.n, factors.m
        self.alpha, self.gamma = float(alpha), int(gamma)
        self.degrees = factors.degrees
        self._fac = factors
        self._f = factors.dev
        self.p_k_dev = p_k_dev
        # (beta f64, beta f32, self-loop flags) from beta_device
        self.beta64, self.beta32, self.selfloop_dev = beta_vecs
        self._structs = {}
        self._beta_host = None

    @property
    def beta(self) -> np.ndarray:
        if self._beta_host is None:
            self._beta_host = self.beta64.cpu().numpy()
        return self._beta_host

    @property
    def selfloop(self) -> np.ndarray:
        return np.flatnonzero(self.selfloop_dev.cpu().numpy())

    @property
    def p_k(self):
        return self.p_k_dev.to_scipy()

    @property
    def p_n(self):
        return self._fac.host_view("p_n")

    @property
    def p_v(self):
        return self._fac.host_view("p_v")

    @property
    def p_e(self):
        return self._fac.host_view("p_e")

    @property
    def layer_p(self):
        """multiplex: per-layer P_l (walk.py:100), host views."""
        if self.kind is not NetworkKind.MULTIPLEX:
            return None
        return tuple(m.to_scipy() for m in self._f["layers"])

    def struct(self, dtype: int) -> _lib.Operator:
        """ctypes ancka_operator for f32 (`_lib.F32`) or f64 values."""
        s = self._structs.get(dtype)
        if s is None:
            f = self._f
            kind = {NetworkKind.HYPERGRAPH: _lib.HYPERGRAPH, NetworkKind.GRAPH: _lib.GRAPH,
                    NetworkKind.MULTIPLEX: _lib.MULTIPLEX}[self.kind]
            nl, lay, lay_t = 0, None, None
            if self.kind is NetworkKind.MULTIPLEX:
                nl = len(f["layers"])
                lay = (_lib.CSR * nl)(*[m.struct(dtype) for m in f["layers"]])
                lay_t = (_lib.CSR * nl)(*[m.struct(dtype) for m in f["layers_t"]])
                self._keep = getattr(self, "_keep", []) + [lay, lay_t]   # ctypes arrays stay alive
            split = (self._split_plan() if dtype == _lib.F32 and self.kind is not NetworkKind.MULTIPLEX
                     else _lib.RowSplit())
            s = _lib.Operator(
                kind, dtype, self.n, self.m,
                csr_struct(f.get("p_n"), dtype), csr_struct(f.get("p_e"), dtype),
                csr_struct(f.get("p_v"), dtype), csr_struct(self.p_k_dev, dtype),
                csr_struct(f.get("t_a"), dtype), csr_struct(f.get("t_b"), dtype),
                (self.beta64 if dtype == _lib.F64 else self.beta32).data_ptr(),
                self.selfloop_dev.data_ptr(), split, nl,
                ctypes.cast(lay, ctypes.c_void_p) if lay is not None else None,
                ctypes.cast(lay_t, ctypes.c_void_p) if lay_t is not None else None)
            self._structs[dtype] = s
        return s

    # rows costing more than max(LONG_ROW, HUB_FACTOR x the mean row) nonzeros
    # (hubs) get a whole warp; ordinary rows stay one thread (group)
    LONG_ROW, HUB_FACTOR = 64, 4

    def _split_plan(self) -> _lib.RowSplit:
        """Load-balancing plan of the f32 n-row pass (KNN hubs, graph hubs):
        cost order and long rows, built on the device by plan.cu."""
        sf = self._f["p_v" if self.kind is NetworkKind.HYPERGRAPH else "p_n"]
        srp, krp = sf.rowptr, self.p_k_dev.rowptr
        d, n = srp.device, self.n
        # mean row cost = (structural + KNN nonzeros) / n, known on the host
        mean = (sf.nnz + self.p_k_dev.nnz) / n if n else 0.0
        thr = max(self.LONG_ROW, self.HUB_FACTOR * mean)
        lib = _lib.load()
        ws = WORKSPACE.get("row_split", lib.ancka_row_split_workspace_size(n))
        self._order = torch.empty(n, dtype=torch.int32, device=d)
        is_long = torch.empty(n, dtype=torch.uint8, device=d)
        long_rows = torch.empty(n, dtype=torch.int32, device=d)
        n_long_dev = torch.zeros(1, dtype=torch.int64, device=d)
        _lib.call("ancka_row_split_plan", srp.data_ptr(), krp.data_ptr(), n, float(thr),
                  self._order.data_ptr(), is_long.data_ptr(), long_rows.data_ptr(),
                  n_long_dev.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream())
        n_long = int(n_long_dev.item())
        self._plan = {"is_long": is_long, "long_rows": long_rows}
        if n_long == 0:
            return _lib.RowSplit(0, None, None, self._order.data_ptr())
        return _lib.RowSplit(n_long, is_long.data_ptr(), long_rows.data_ptr(),
                             self._order.data_ptr())

    def set_locality(self, labels: torch.Tensor, k: int) -> None:
        """Process the rows of the f32 graph apply grouped by cluster label
        (ancka_locality_order): the rows in flight then gather mostly their
        own cluster's rows of the block, which stay in L2.  Performance only:
        every row's sum is computed exactly as before."""
        if self.kind is not NetworkKind.GRAPH or os.environ.get("ANCKA_NO_LOCALITY"):
            return
        s = self.struct(_lib.F32)
        order = getattr(self, "_locality", None)
        if order is None:
            order = torch.empty(self.n, dtype=torch.int32, device=labels.device)
        lib = _lib.load()
        ws = WORKSPACE.get("locality", lib.ancka_locality_order_workspace_size(self.n))
        _lib.call("ancka_locality_order", labels.data_ptr(), self.n, int(k), order.data_ptr(),
                  ws.data_ptr(), ws.numel(), _lib.stream())
        self._locality = order
        s.split.locality_order = order.data_ptr()

    def scratch(self, c: int, dtype: torch.dtype, key: str = "op_scratch") -> torch.Tensor:
        rows = max(self.m, 1)
        return WORKSPACE.get(f"{key}_{dtype}", rows * ld_for(c, dtype) * (4 if dtype == torch.float32 else 8))


def beta_device(factors: StructureFactors, knn_zero_rows, beta: float):
    """beta_vector (walk.py:47-57) on the device: (beta f64, beta f32,
    self-loop flags of walk.py:123), one kernel."""
    z = knn_zero_rows if isinstance(knn_zero_rows, torch.Tensor) else \
        torch.from_numpy(np.asarray(knn_zero_rows, dtype=bool)).to(dev())
    z = z.to(torch.uint8) if z.dtype != torch.uint8 else z
    n = factors.n
    b64 = torch.empty(n, dtype=torch.float64, device=dev())
    b32 = torch.empty(n, dtype=torch.float32, device=dev())
    loops = torch.empty(n, dtype=torch.uint8, device=dev())
    _lib.call("ancka_beta_vector", factors.degrees_dev.data_ptr(), z.data_ptr(), n, float(beta),
              b64.data_ptr(), b32.data_ptr(), loops.data_ptr(), _lib.stream())
    return b64, b32, loops


def build_walk_operator(net: AttributedNetwork, p_k, knn_zero_rows, alpha: float, beta: float,
                        gamma: int, factors: StructureFactors | None = None) -> WalkOperator:
    """walk.py:107-132.  `p_k` may be a device `DeviceCSR` (engine path) or a
    scipy CSR (API callers); `knn_zero_rows` a bool array or device tensor;
    `factors` reuses already-uploaded structural factors."""
    _lib.require_device()
    if factors is None:
        factors = StructureFactors(net)
    if not isinstance(p_k, DeviceCSR):
        p_k = DeviceCSR.from_scipy(p_k)
    return WalkOperator(factors, p_k, beta_device(factors, knn_zero_rows, beta), alpha, gamma)


def _apply(op: WalkOperator, m, transposed: bool):
    _lib.require_device()
    host = not isinstance(m, torch.Tensor)
    t = torch.as_tensor(m)
    squeeze = t.ndim == 1
    if squeeze:
        t = t[:, None]
    if t.shape[0] != op.n:
        raise NetworkError(f"block has {t.shape[0]} rows, operator expects {op.n}")
    c = t.shape[1]
    q = padded(t, torch.float64)
    z = torch.empty_like(q)
    scr = op.scratch(c, torch.float64)
    fn = "ancka_op_apply_struct_t" if transposed else "ancka_op_apply"
    _lib.call(fn, op.struct(_lib.F64), q.data_ptr(), q.stride(0), c, z.data_ptr(), z.stride(0),
              scr.data_ptr(), _lib.stream())
    out = z[:, :c]
    if squeeze:
        out = out[:, 0]
    return out.cpu().numpy() if host else out


def apply_joint_transition(op: WalkOperator, m):
    """(I-B) P_N M + B P_K M on the device in f64 (walk.py:177-190)."""
    return _apply(op, m, transposed=False)


def apply_structure_rowvec(op: WalkOperator, m):
    """c x n row block times the structural transition (walk.py:153-174)."""
    if m.shape[1] != op.n:
        raise NetworkError(f"block has {m.shape[1]} columns, operator expects {op.n}")
    mt = m.T if isinstance(m, torch.Tensor) else np.ascontiguousarray(np.asarray(m).T)
    out = _apply(op, mt, transposed=True)
    return out.T if isinstance(out, torch.Tensor) else np.ascontiguousarray(out.T)


def apply_structure(op: WalkOperator, m):
    """Structural transition times a block (walk.py:135-150): P_N M (graph),
    P_V (P_E M) (hypergraph) or the layer average (multiplex), plus M on the
    self-loop rows.  Runs the same device apply as apply_joint_transition on
    a view of the operator whose beta is zero, so (1 - 0) struct + 0 attr is
    exactly the structural product."""
    return _apply(_structure_view(op), m, transposed=False)


def _structure_view(op: WalkOperator) -> WalkOperator:
    view = op.__dict__.get("_structure_only")
    if view is None:
        import copy
        view = copy.copy(op)
        view.beta64 = torch.zeros_like(op.beta64)
        view.beta32 = torch.zeros_like(op.beta32)
        view._structs, view._beta_host = {}, None
        op.__dict__["_structure_only"] = view
    return view


#: the reference's dense-oracle size limit (walk.py DENSE_ORACLE_MAX_N)
DENSE_ORACLE_MAX_N = 2000


def _check_dense(op: WalkOperator) -> None:
    if op.n > DENSE_ORACLE_MAX_N:
        raise NetworkError(f"dense oracle is limited to n <= {DENSE_ORACLE_MAX_N}, got {op.n}")


def dense_transition(op: WalkOperator) -> np.ndarray:
    """Materialised joint transition (walk.py:193-208): the device apply of
    the identity block, P = apply(op, I_n), in f64."""
    _check_dense(op)
    eye = torch.eye(op.n, dtype=torch.float64, device=dev())
    return apply_joint_transition(op, eye).cpu().numpy()


def dense_walk_scores(op: WalkOperator) -> np.ndarray:
    """alpha * sum_{s=0..gamma} (1 - alpha)^s P^s (walk.py:211-225); each power
    is one device apply of the previous one (P^s = P P^(s-1))."""
    _check_dense(op)
    power = torch.eye(op.n, dtype=torch.float64, device=dev())
    s = op.alpha * power.clone()
    for step in range(1, op.gamma + 1):
        power = apply_joint_transition(op, power)
        s += op.alpha * (1.0 - op.alpha) ** step * power
    return s.cpu().numpy()


def brute_mhc_oracle(op: WalkOperator, y) -> float:
    """Multi-hop conductance from the dense walk scores (walk.py:228-242):
    1 - tr(Yhat^T S Yhat) / k, independent of the iterative calc_mhc."""
    if y.n != op.n:
        raise NetworkError("membership length does not match operator size")
    empty = y.empty_clusters()
    if empty.size:
        raise NetworkError(f"empty cluster(s) {empty.tolist()}: conductance undefined")
    s = dense_walk_scores(op)
    sizes = y.cluster_sizes().astype(np.float64)
    yhat = y.to_onehot() / np.sqrt(sizes)[y.assignment][:, None]
    return float(1.0 - np.trace(yhat.T @ s @ yhat) / y.k)
