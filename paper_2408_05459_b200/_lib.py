"""ctypes binding of libancka_b200.so (include/ancka_b200.h).

The shared library is the product: there is no Python or CPU fallback.  If it
is missing, or no sm_100 device is present when a compute entry point is
used, the call raises.
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int32, c_int64, c_size_t, c_void_p
from pathlib import Path

from .network import NetworkError

LIB_PATH = Path(__file__).resolve().parent / "libancka_b200.so"

ANCKA_OK, ANCKA_ERR_ARG, ANCKA_ERR_CUDA, ANCKA_ERR_NETWORK, ANCKA_ERR_UNSUPPORTED = range(5)
F32, F64 = 0, 1
GRAPH, HYPERGRAPH, MULTIPLEX = 0, 1, 2
MAX_LAYERS = 8


class CSR(ctypes.Structure):
    _fields_ = [("rows", c_int64), ("cols", c_int64), ("nnz", c_int64),
                ("rowptr", c_void_p), ("colidx", c_void_p), ("values", c_void_p)]


class RowSplit(ctypes.Structure):
    _fields_ = [("n_long", c_int64), ("is_long", c_void_p), ("long_rows", c_void_p),
                ("row_order", c_void_p), ("locality_order", c_void_p)]


class Operator(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("dtype", c_int32), ("n", c_int64), ("m", c_int64),
                ("p_n", CSR), ("p_e", CSR), ("p_v", CSR), ("p_k", CSR), ("t_a", CSR),
                ("t_b", CSR), ("beta", c_void_p), ("selfloop", c_void_p), ("split", RowSplit),
                ("n_layers", c_int32), ("layers", c_void_p), ("layers_t", c_void_p)]


_OP = POINTER(Operator)
# name -> (restype, argtypes)
_SIGS = {
    "ancka_last_error": (ctypes.c_char_p, []),
    "ancka_abi_version": (c_int32, []),
    "ancka_device_check": (c_int32, []),
    "ancka_launch_count": (c_int64, []),
    "ancka_knn_workspace_size": (c_size_t, [c_int64, c_int64, c_int32, c_int32]),
    "ancka_knn_exact": (c_int32, [c_void_p, c_int64, c_int64, c_int64, c_int32, c_int32,
                                  c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_size_t,
                                  c_void_p]),
    "ancka_knn_fallback_rows": (c_int32, [c_void_p, c_size_t, c_int64, c_int64, c_int32, c_int64,
                                          c_int64, c_void_p]),
    "ancka_knn_fallback_rows_async": (c_int32, [c_void_p, c_size_t, c_int64, c_int64, c_int32,
                                                c_int64, c_int64, c_void_p, c_void_p]),
    "ancka_knn_exact_csr": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int32,
                                      c_int32, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                      c_size_t, c_void_p]),
    "ancka_spmm2": (c_int32, [c_int32, c_int64, c_int32, POINTER(CSR), c_void_p, c_int64,
                              POINTER(CSR), c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                              c_int64, c_int64, c_void_p, c_void_p, c_double, c_void_p, c_int64,
                              c_void_p, c_void_p]),
    "ancka_gram_f32": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p,
                                 c_size_t, c_void_p]),
    "ancka_cholqr_apply_f32": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int32,
                                         c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ancka_knn_exact_keys": (c_int32, [c_void_p, c_int64, c_int64, c_int64, c_int32, c_int32,
                                       c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                       c_void_p, c_size_t, c_void_p]),
    "ancka_knn_exact_csr_keys": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                           c_int32, c_int32, c_int64, c_int64, c_int64, c_int64,
                                           c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ancka_ivf_normalize": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
                                      c_int64, c_void_p, c_int64, c_void_p]),
    "ancka_ivf_gemm": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int32,
                                 c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "ancka_ivf_argmax_finish": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "ancka_ivf_topsel": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_int32, c_void_p,
                                   c_void_p]),
    "ancka_ivf_bucket_workspace_size": (c_size_t, [c_int32]),
    "ancka_ivf_bucket": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_int32,
                                   c_void_p, c_void_p, c_size_t, c_void_p]),
    "ancka_ivf_search": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_int32, c_int32, c_int64, c_int32,
                                   ctypes.c_float, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ancka_ivf_merge": (c_int32, [c_void_p, c_int64, c_int64, c_int64, c_int32, c_int32, c_int32,
                                  c_void_p, c_void_p, ctypes.c_float, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ancka_ivf_half_prep": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                      c_void_p, c_void_p]),
    "ancka_ivf_split_probes": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_int32, c_void_p,
                                         c_void_p, c_void_p]),
    "ancka_ivf_search_tc": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32,
                                      c_int64, c_int32, ctypes.c_float, c_void_p, c_void_p,
                                      c_void_p, c_void_p]),
    "ancka_ivf_rows_exact": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                       c_int32, c_int64, c_void_p, c_void_p, c_int32, c_void_p,
                                       c_void_p, c_int32, c_void_p]),
    "ancka_ivf_kmeans_update": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                          c_int32, c_int64, c_void_p, c_void_p, c_void_p,
                                          c_int64, c_void_p, c_void_p]),
    "ancka_discw_dist_workspace_size": (c_size_t, [c_int64, c_int32]),
    "ancka_discw_dist_init": (c_int32, [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64,
                                        c_int32, c_int32, c_double, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ancka_discw_dist_op": (c_int32, [c_void_p, c_int32, c_int64, c_int64, c_void_p, c_void_p]),
    "ancka_l2_read": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p,
                                ctypes.POINTER(c_double), ctypes.POINTER(c_double), c_void_p]),
    "ancka_tc_peak": (c_int32, [c_int32, c_int32, ctypes.POINTER(c_double),
                                ctypes.POINTER(c_double), c_void_p, c_void_p]),
    "ancka_knn_merge_lists": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                        c_void_p]),
    "ancka_knn_graph_coo_workspace_size": (c_size_t, [c_int64]),
    "ancka_knn_graph_coo": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_size_t, c_void_p]),
    "ancka_locality_order_workspace_size": (c_size_t, [c_int64]),
    "ancka_locality_order": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_size_t,
                                       c_void_p]),
    "ancka_knn_graph_workspace_size": (c_size_t, [c_int64, c_int32]),
    "ancka_knn_graph": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_size_t, c_void_p]),
    "ancka_csr_row_normalize": (c_int32, [POINTER(CSR), c_void_p, c_void_p, c_void_p]),
    "ancka_csr_col_scale": (c_int32, [POINTER(CSR), c_void_p, c_void_p, c_void_p]),
    "ancka_csr_transpose_workspace_size": (c_size_t, [c_int64, c_int64, c_int64]),
    "ancka_csr_transpose": (c_int32, [POINTER(CSR), c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_size_t, c_void_p]),
    "ancka_attr_check": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p,
                                   c_void_p]),
    "ancka_op_apply": (c_int32, [_OP, c_void_p, c_int64, c_int32, c_void_p, c_int64, c_void_p,
                                 c_void_p]),
    "ancka_op_apply_struct_t": (c_int32, [_OP, c_void_p, c_int64, c_int32, c_void_p, c_int64,
                                          c_void_p, c_void_p]),
    "ancka_init_workspace_size": (c_size_t, [_OP, c_int32]),
    "ancka_init_bcm": (c_int32, [_OP, c_void_p, c_int32, c_int32, c_double, c_void_p, c_void_p,
                                 c_size_t, c_void_p]),
    "ancka_orth_workspace_size": (c_size_t, [_OP, c_int32]),
    "ancka_orth_step_f32": (c_int32, [_OP, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                      c_void_p, c_void_p, c_size_t, c_void_p]),
    "ancka_orth_block_workspace_size": (c_size_t, [_OP]),
    "ancka_orth_block_f32": (c_int32, [_OP, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                       c_int32, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ancka_qr_f64_workspace_size": (c_size_t, [c_int64, c_int32]),
    "ancka_qr_f64": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p, c_size_t,
                               c_void_p]),
    "ancka_discretize_workspace_size": (c_size_t, [c_int64, c_int32, c_int32]),
    "ancka_discretize": (c_int32, [c_void_p, c_int64, c_int64, c_int64, c_int32, c_int32,
                                   c_double, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ancka_disc_normalize": (c_int32, [c_void_p, c_int64, c_int64, c_int64, c_int32, c_void_p,
                                       c_int64, c_void_p, c_void_p]),
    "ancka_disc_score": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_int64,
                                   c_void_p, c_void_p, c_void_p]),
    "ancka_disc_accumulate": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_double,
                                        c_void_p, c_void_p, c_void_p]),
    "ancka_disc_proto_pass": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p,
                                        c_void_p]),
    "ancka_mhc_workspace_size": (c_size_t, [_OP, c_int32]),
    "ancka_mhc": (c_int32, [_OP, c_void_p, c_int32, c_double, c_int32, c_void_p, c_void_p,
                            c_void_p, c_size_t, c_void_p]),
    "ancka_mhc_timing": (None, [c_void_p, c_int32]),
    "ancka_same_partition": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p,
                                       c_void_p]),
    "ancka_cluster_sizes": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    "ancka_row_split_workspace_size": (c_size_t, [c_int64]),
    "ancka_beta_vector": (c_int32, [c_void_p, c_void_p, c_int64, c_double, c_void_p, c_void_p,
                                    c_void_p, c_void_p]),
    "ancka_bcm_block": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_double, c_void_p,
                                  c_int64, c_void_p]),
    "ancka_row_split_plan": (c_int32, [c_void_p, c_void_p, c_int64, c_double, c_void_p,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                       c_void_p]),
}

_lib = None


def load():
    """Load the library and bind every exported entry point (raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH.name} is not built; run `python -m paper_2408_05459_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return sorted(_SIGS)


def check(status: int) -> None:
    if status == ANCKA_OK:
        return
    msg = load().ancka_last_error().decode(errors="replace")
    if status == ANCKA_ERR_NETWORK:
        raise NetworkError(msg)
    if status == ANCKA_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"ancka_b200 (status {status}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


_device_ok = False


def require_device():
    """Raise unless a B200-class (sm_100) CUDA device is usable."""
    global _device_ok
    if _device_ok:
        return
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2408_05459_b200 needs a CUDA device (sm_100a); none is visible")
    torch.cuda.init()
    check(load().ancka_device_check())
    _device_ok = True


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream
