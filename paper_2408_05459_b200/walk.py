"""Subsystem 2: the joint-walk operator on the B200 (reference: ancka/walk.py).

Structural factors are normalised on the host with the same scipy calls as
the reference (O(nnz), once per network) and uploaded; the KNN factor P_K is
produced on the device by `ancka_knn_graph`.  `apply_joint_transition` and
`apply_structure_rowvec` run `ancka_op_apply` / `ancka_op_apply_struct_t`;
in f64 they are bit-identical to scipy's csr_matvecs.
"""
from __future__ import annotations

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
    raise NetworkError("multiplex networks are outside the B200 hot path (SURVEY.md §8f)")


class StructureFactors:
    """Host-normalised structural factors uploaded once (walk.py:60-79), plus
    the init transposes (walk.py:163-165) and the pattern degrees."""

    def __init__(self, net: AttributedNetwork):
        if net.kind is NetworkKind.MULTIPLEX:
            multiplex_transition(net)
        self.kind, self.n = net.kind, net.n
        self.degrees = node_degrees(net)
        self.host, self.dev = {}, {}
        if net.kind is NetworkKind.HYPERGRAPH:
            p_v, p_e = hypergraph_factors(net)
            self.host.update(p_v=p_v, p_e=p_e)
            self.dev["p_v"], self.dev["p_e"] = DeviceCSR.from_scipy(p_v), DeviceCSR.from_scipy(p_e)
            # init_bcm transposes: (p_e^T @ (p_v^T @ m)), walk.py:163
            self.dev["t_a"] = DeviceCSR.from_scipy(p_v.T.tocsr())
            self.dev["t_b"] = DeviceCSR.from_scipy(p_e.T.tocsr())
            self.m = p_e.shape[0]
        else:
            p_n = graph_transition(net)
            self.host["p_n"] = p_n
            self.dev["p_n"] = DeviceCSR.from_scipy(p_n)
            self.dev["t_a"] = DeviceCSR.from_scipy(p_n.T.tocsr())
            self.m = 0
        self.degrees_dev = torch.from_numpy(self.degrees).to(dev())

    def h2d_bytes(self) -> int:
        return int(sum(m.rowptr.numel() * 8 + m.colidx.numel() * 4 + m.val64.numel() * 8
                       for m in self.dev.values()) + self.degrees.nbytes)


class WalkOperator:
    """Device-resident joint-walk factors (walk.py:89-104).  The scipy
    attributes of the reference (`p_k`, `p_n`, `p_v`, `p_e`, `beta`,
    `selfloop`) are host views materialised on access."""

    def __init__(self, factors: StructureFactors, p_k_dev: DeviceCSR, beta_dev, alpha, gamma):
        self.kind, self.n, self.m = factors.kind, factors.n, factors.m
        self.alpha, self.gamma = float(alpha), int(gamma)
        self.degrees = factors.degrees
        self._fac = factors
        self._f = factors.dev
        self.p_k_dev = p_k_dev
        self.beta64 = beta_dev
        self.beta32 = beta_dev.to(torch.float32)
        self.selfloop_dev = ((factors.degrees_dev == 0) & (beta_dev == 0)).to(torch.uint8)
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
        return self._fac.host.get("p_n")

    @property
    def p_v(self):
        return self._fac.host.get("p_v")

    @property
    def p_e(self):
        return self._fac.host.get("p_e")

    layer_p = None

    def struct(self, dtype: int) -> _lib.Operator:
        """ctypes ancka_operator for f32 (`_lib.F32`) or f64 values."""
        s = self._structs.get(dtype)
        if s is None:
            f = self._f
            s = _lib.Operator(
                _lib.HYPERGRAPH if self.kind is NetworkKind.HYPERGRAPH else _lib.GRAPH, dtype,
                self.n, self.m,
                csr_struct(f.get("p_n"), dtype), csr_struct(f.get("p_e"), dtype),
                csr_struct(f.get("p_v"), dtype), csr_struct(self.p_k_dev, dtype),
                csr_struct(f.get("t_a"), dtype), csr_struct(f.get("t_b"), dtype),
                (self.beta64 if dtype == _lib.F64 else self.beta32).data_ptr(),
                self.selfloop_dev.data_ptr(),
                self._split_plan() if dtype == _lib.F32 else _lib.RowSplit())
            self._structs[dtype] = s
        return s

    # rows costing more than max(LONG_ROW, HUB_FACTOR x the mean row) nonzeros
    # (hubs) are cut into PIECE-long pieces; ordinary rows stay one thread group
    LONG_ROW, HUB_FACTOR, PIECE, MAX_LD = 64, 4, 32, 256

    def _split_plan(self) -> _lib.RowSplit:
        """Load-balancing plan of the f32 n-row pass (KNN hubs, graph hubs)."""
        srp = self._f["p_v" if self.kind is NetworkKind.HYPERGRAPH else "p_n"].rowptr.cpu().numpy()
        krp = self.p_k_dev.rowptr.cpu().numpy()
        ls, lk = np.diff(srp), np.diff(krp)
        cost = ls + lk
        thr = max(self.LONG_ROW, self.HUB_FACTOR * float(cost.mean()) if cost.size else 0.0)
        long_rows = np.flatnonzero(cost > thr).astype(np.int32)
        if long_rows.size == 0:
            return _lib.RowSplit()
        P = self.PIECE
        ns = -(-ls[long_rows] // P)                   # structural pieces per long row
        nk = -(-lk[long_rows] // P)                   # KNN pieces per long row
        per = ns + nk
        ptr = np.concatenate([[0], np.cumsum(per)])
        # within-row piece ordinal q and its segment (structural pieces first)
        q = np.arange(ptr[-1]) - np.repeat(ptr[:-1], per)
        rrep = np.repeat(long_rows, per)
        is_k = q >= np.repeat(ns, per)
        qq = np.where(is_k, q - np.repeat(ns, per), q)
        rb = np.where(is_k, krp[rrep], srp[rrep])
        re = np.where(is_k, krp[rrep + 1], srp[rrep + 1])
        begins = rb + qq * P
        ends = np.minimum(re, begins + P)
        segs = is_k.astype(np.int32)
        d = dev()
        mask = np.zeros(self.n, dtype=np.uint8)
        mask[long_rows] = 1
        self._plan = {
            "is_long": torch.from_numpy(mask).to(d),
            "long_rows": torch.from_numpy(long_rows).to(d),
            "piece_ptr": torch.from_numpy(ptr.astype(np.int64)).to(d),
            "piece_seg": torch.from_numpy(segs).to(d),
            "piece_begin": torch.from_numpy(begins.astype(np.int64)).to(d),
            "piece_end": torch.from_numpy(ends.astype(np.int64)).to(d),
            "partial": torch.empty(len(segs) * self.MAX_LD, dtype=torch.float32, device=d),
        }
        p = self._plan
        return _lib.RowSplit(long_rows.size, len(segs), p["is_long"].data_ptr(),
                             p["long_rows"].data_ptr(), p["piece_ptr"].data_ptr(),
                             p["piece_seg"].data_ptr(), p["piece_begin"].data_ptr(),
                             p["piece_end"].data_ptr(), p["partial"].data_ptr(), self.MAX_LD)

    def scratch(self, c: int, dtype: torch.dtype, key: str = "op_scratch") -> torch.Tensor:
        rows = max(self.m, 1)
        return WORKSPACE.get(f"{key}_{dtype}", rows * ld_for(c, dtype) * (4 if dtype == torch.float32 else 8))


def beta_device(factors: StructureFactors, knn_zero_rows, beta: float) -> torch.Tensor:
    """beta_vector (walk.py:47-57) on the device."""
    z = knn_zero_rows if isinstance(knn_zero_rows, torch.Tensor) else \
        torch.from_numpy(np.asarray(knn_zero_rows, dtype=bool)).to(dev())
    b = torch.full((factors.n,), float(beta), dtype=torch.float64, device=dev())
    b = torch.where(factors.degrees_dev == 0, torch.ones_like(b), b)
    return torch.where(z.bool(), torch.zeros_like(b), b)


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
    """Structural transition times a block (walk.py:135-150): the joint apply
    with beta = 0 is not exposed separately on the device; provided for API
    completeness via a beta-free operator view."""
    raise NetworkError("apply_structure is internal to the fused device operator; "
                       "use apply_joint_transition")
