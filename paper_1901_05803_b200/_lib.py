"""ctypes binding of libralpb200.so (the C ABI declared in include/ralpb.h).

The library is the only compute path: if it is missing or fails to load this
module raises, there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("RALPB_LIB", _PKG / "libralpb200.so"))

_lib = None

c_ll = C.c_longlong
c_vp = C.c_void_p
c_i = C.c_int
c_f = C.c_float
c_fp = C.c_void_p  # float*
c_cp = C.c_char_p

# name -> (restype, argtypes); mirrors include/ralpb.h
SIGNATURES: dict[str, tuple] = {
    "ralpb_last_error": (c_cp, []),
    "ralpb_version": (c_i, []),
    "ralpb_gemm_bf16": (c_i, [c_vp, c_ll, c_ll, c_ll, c_i, c_vp, c_ll, c_ll, c_ll, c_i, c_i, c_i, c_ll,
                              c_vp, c_i, c_ll, c_ll, c_fp, c_i, c_vp, c_ll, c_i, c_i, c_vp]),
    "ralpb_conv_fwd": (c_i, [c_vp, c_vp, c_fp, c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_vp]),
    "ralpb_conv_first_fwd": (c_i, [c_vp, c_i, c_i, c_i, c_vp, c_vp, c_i, c_vp]),
    "ralpb_conv_first_wgrad": (c_i, [c_vp, c_i, c_i, c_i, c_vp, c_i, c_vp, c_vp]),
    "ralpb_conv_fwd_pool": (c_i, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i, c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i,
                                  c_vp]),
    "ralpb_maxpool_fwd_idx": (c_i, [c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_vp, c_i, c_vp, c_vp]),
    "ralpb_maxpool_bwd_gather": (c_i, [c_vp, c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_vp, c_vp, c_vp]),
    "ralpb_maxpool_bwd_idx": (c_i, [c_vp, c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_vp, c_vp, c_vp]),
    "ralpb_conv_dgrad": (c_i, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_vp]),
    "ralpb_conv_wgrad": (c_i, [c_vp, c_vp, c_fp, c_fp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_vp]),
    "ralpb_pack_input": (c_i, [c_fp, c_i, c_i, c_i, c_i, c_vp, c_i, c_i, c_vp]),
    "ralpb_pack_im2col": (c_i, [c_fp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_vp, c_vp]),
    "ralpb_maxpool_fwd": (c_i, [c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_vp, c_i, c_vp]),
    "ralpb_maxpool_bwd": (c_i, [c_vp, c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_vp, c_vp, c_vp]),
    "ralpb_softmax_xent": (c_i, [c_fp, c_i, c_i, c_ll, c_vp, c_f, c_fp, c_vp, c_ll, c_vp]),
    "ralpb_sgd_momentum": (c_i, [c_fp, c_fp, c_fp, c_ll, c_f, c_f, c_f, c_vp]),
    "ralpb_colsum_bf16": (c_i, [c_vp, c_ll, c_i, c_ll, c_fp, c_vp]),
    "ralpb_conv_weight_prep": (c_i, [c_fp, c_i, c_i, c_i, c_vp, c_vp, c_vp]),
    "ralpb_cast_bf16": (c_i, [c_fp, c_ll, c_vp, c_vp]),
    "ralpb_model_create": (c_i, [c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, C.POINTER(c_vp)]),
    "ralpb_model_create_graph": (c_i, [c_vp, c_i, c_vp, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i, c_i,
                                       C.POINTER(c_vp)]),
    "ralpb_model_destroy": (None, [c_vp]),
    "ralpb_model_ipc_handle": (c_i, [c_vp, c_vp]),
    "ralpb_model_ipc_open": (c_i, [c_vp, c_vp]),
    "ralpb_model_set_params": (c_i, [c_vp, c_i, c_vp, c_vp, c_i]),
    "ralpb_model_get_params": (c_i, [c_vp, c_i, c_vp, c_vp, c_i]),
    "ralpb_model_get_grads": (c_i, [c_vp, c_i, c_vp, c_vp]),
    "ralpb_model_step": (c_i, [c_vp, c_vp, c_vp, c_i, c_f, c_f]),
    "ralpb_model_stats": (c_i, [c_vp, c_vp]),
    "ralpb_model_read_loss": (c_i, [c_vp, c_i, c_vp]),
    "ralpb_model_timed_launches": (c_i, [c_vp, c_vp, c_i]),
    "ralpb_model_grad_buffer": (c_i, [c_vp, c_vp, c_vp]),
    "ralpb_model_apply": (c_i, [c_vp, c_f, c_f]),
    "ralpb_model_stream": (c_vp, [c_vp]),
    "ralpb_model_set_profiling": (c_i, [c_vp, c_i]),
    "ralpb_model_debug_buffer": (c_ll, [c_vp, c_i, c_i, c_vp]),
}


class LayerDesc(C.Structure):
    """ralpb_layer_desc (include/ralpb.h)."""
    _fields_ = [("kind", c_i), ("k", c_i), ("stride", c_i), ("pad", c_i), ("h", c_i), ("w", c_i),
                ("cin", c_i), ("cout", c_i), ("relu", c_i), ("bn", c_i), ("width", c_i), ("downsample", c_i),
                ("node_begin", c_i), ("node_count", c_i)]


class NodeDesc(C.Structure):
    """ralpb_node_desc (include/ralpb.h): one node of a MODULE layer."""
    _fields_ = [("op", c_i), ("input", c_i), ("kh", c_i), ("kw", c_i), ("stride", c_i), ("pad_h", c_i),
                ("pad_w", c_i), ("cout", c_i), ("bn", c_i), ("output", c_i)]


class LaunchRec(C.Structure):
    """ralpb_launch_rec (include/ralpb.h)."""
    _fields_ = [("kind", C.c_int), ("ms", C.c_float), ("flops", C.c_double), ("bytes", C.c_double),
                ("t0", C.c_float), ("stream", C.c_int)]


LAUNCH_KINDS = ["conv_fwd", "conv_fwd_pair", "conv_wgrad_pair", "conv_wgrad", "first_conv_fwd", "first_conv_wgrad",
                "gemm", "push", "shard_update", "maxpool_bwd", "sgd"]
TENSOR_KINDS = LAUNCH_KINDS[:7]


class StepStats(C.Structure):
    """ralpb_step_stats (include/ralpb.h)."""
    _fields_ = [("loss", C.c_double), ("logical_bytes", c_ll), ("physical_bytes", c_ll), ("launches", c_i),
                ("ms_step", c_f), ("ms_front_fwd", c_f), ("ms_back", c_f), ("ms_front_bwd", c_f),
                ("ms_sync", c_f), ("ms_gemm", c_f), ("gemm_launches", c_i), ("nvlink_out_bytes", c_ll),
                ("nvlink_in_bytes", c_ll)]


RALPB_CONV, RALPB_POOL, RALPB_FC, RALPB_BLOCK, RALPB_APOOL, RALPB_MODULE = 0, 1, 2, 3, 4, 5
RALPB_NODE_CONV, RALPB_NODE_MAXPOOL, RALPB_NODE_AVGPOOL = 0, 1, 2
RALPB_STRATEGY_BASELINE, RALPB_STRATEGY_RALP, RALPB_STRATEGY_RING, RALPB_STRATEGY_RING_EXTERNAL = 0, 1, 2, 3
RALPB_STRATEGY_RALP_MPS = 4
RALPB_STRATEGY_BASELINE_LAYER_SHARDS = 5
RALPB_PRECISION_BF16, RALPB_PRECISION_FP32 = 0, 1
PRECISIONS = {"bf16": RALPB_PRECISION_BF16, "fp32": RALPB_PRECISION_FP32}
# ralpb_model_debug_buffer selectors (include/ralpb.h)
(DBG_ACT, DBG_ACT_GRAD, DBG_LOGITS, DBG_FC_OUT, DBG_MPS_PARTIAL, DBG_FC_WEIGHT, DBG_DLOGITS, DBG_FC_OUT_GRAD,
 DBG_CUT_ROWS, DBG_CUT_GRAD_ROWS, DBG_CUT_GRAD, DBG_FC_IN, DBG_FC_IN_GRAD) = range(13)


class BackendError(RuntimeError):
    """A call into libralpb200.so failed."""


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise BackendError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1901_05803_b200.build` "
                "(there is no CPU fallback)")
        handle = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
        # RALPB_LIB_LENIENT=1 tolerates entry points an older build lacks (A/B timing of builds)
        lenient = os.environ.get("RALPB_LIB_LENIENT") == "1"
        for name, (res, args) in SIGNATURES.items():
            if lenient and not hasattr(handle, name):
                continue
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def call(name: str, *args) -> None:
    fn = getattr(lib(), name)
    rc = fn(*args)
    if rc != 0:
        msg = lib().ralpb_last_error().decode(errors="replace")
        raise BackendError(f"{name} failed ({rc}): {msg}")


def call_count(name: str, *args) -> int:
    """Entry points that return a count (>= 0) or -1 on error."""
    fn = getattr(lib(), name)
    rc = fn(*args)
    if rc < 0:
        msg = lib().ralpb_last_error().decode(errors="replace")
        raise BackendError(f"{name} failed ({rc}): {msg}")
    return rc
