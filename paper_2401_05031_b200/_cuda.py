"""ctypes binding of libtokadapt_cuda.so (include/tokadapt_cuda.h).

This is the only way the Python layer reaches the GPU path.  There is no fallback: if the
library is missing or the device is not sm_100, every call raises.  Status codes map onto
the reference's exception types (pkg/src/tokadapt/errors.py) — see ``check``.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

from .errors import ConfigError, ProfileGapError

__all__ = ["lib", "check", "LIB_PATH", "ModelDesc", "LayerWeights", "Weights", "TAError",
           "StageRecord", "STAGES", "ABI_VERSION", "DTYPE_BF16", "DTYPE_F32", "PROMPT_ACCUMULATE",
           "PROMPT_REPLACE", "EXPORTED_SYMBOLS"]

LIB_PATH = os.environ.get("TA_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtokadapt_cuda.so")

TA_OK, TA_ERR_INVALID, TA_ERR_SHAPE, TA_ERR_CONFIG, TA_ERR_NO_PROMPT = 0, -1, -2, -3, -4
TA_ERR_NO_WEIGHTS, TA_ERR_WORKSPACE, TA_ERR_CUDA, TA_ERR_ARCH = -5, -6, -7, -8
ABI_VERSION = 3
DTYPE_BF16, DTYPE_F32 = 0, 1
# TA_STAGE_* order of include/tokadapt_cuda.h
STAGES = ("patchify", "patch_gemm", "insert_rows", "ln1", "qkv", "attention", "proj", "match",
          "merge", "ln2", "fc1", "fc2", "head")
PROMPT_ACCUMULATE, PROMPT_REPLACE = 0, 1

# Every symbol include/tokadapt_cuda.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "ta_abi_version", "ta_strerror", "ta_last_cuda_error", "ta_model_create", "ta_model_destroy",
    "ta_model_set_weights", "ta_model_set_head", "ta_model_set_prompts", "ta_token_schedule",
    "ta_merge_trace_len", "ta_workspace_size", "ta_forward", "ta_forward_host", "ta_match",
    "ta_match_qkv", "ta_merge", "ta_attention", "ta_gemm", "ta_layernorm", "ta_stage_name",
    "ta_profile_stages", "ta_stage_records",
)


class TAError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ModelDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "dim", "depth", "heads", "mlp_dim", "patch", "img", "n_tasks", "max_classes",
        "prompt_mode", "dtype")]


class LayerWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "ln1_w", "ln1_b", "qkv_w", "qkv_b", "proj_w", "proj_b", "ln2_w", "ln2_b",
        "fc1_w", "fc1_b", "fc2_w", "fc2_b",
        "qkv_w_ln", "qkv_c1", "qkv_c2", "fc1_w_ln", "fc1_c1", "fc1_c2")]


class StageRecord(ctypes.Structure):
    _fields_ = [("stage", ctypes.c_int), ("layer", ctypes.c_int), ("us", ctypes.c_float)]


class Weights(ctypes.Structure):
    _fields_ = [("patch_w", ctypes.c_void_p), ("patch_b", ctypes.c_void_p),
                ("cls", ctypes.c_void_p), ("pos", ctypes.c_void_p),
                ("norm_w", ctypes.c_void_p), ("norm_b", ctypes.c_void_p),
                ("layers", ctypes.POINTER(LayerWeights))]


_lib: Optional[ctypes.CDLL] = None


def _declare(l: ctypes.CDLL) -> None:
    vp, i, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    ip = ctypes.POINTER(ctypes.c_int)
    sig = {
        "ta_abi_version": ([], i),
        "ta_strerror": ([i], ctypes.c_char_p),
        "ta_last_cuda_error": ([], i),
        "ta_model_create": ([i, ctypes.POINTER(ModelDesc), ctypes.POINTER(vp)], i),
        "ta_model_destroy": ([vp], None),
        "ta_model_set_weights": ([vp, ctypes.POINTER(Weights)], i),
        "ta_model_set_head": ([vp, i, vp, vp, i], i),
        "ta_model_set_prompts": ([vp, i, i, vp], i),
        "ta_token_schedule": ([vp, i, ip, ip], i),
        "ta_merge_trace_len": ([vp, i, i, ctypes.POINTER(sz)], i),
        "ta_workspace_size": ([vp, i, i, ctypes.POINTER(sz)], i),
        "ta_forward": ([vp, vp, vp, i, i, vp, vp, vp, vp, sz, vp], i),
        "ta_forward_host": ([vp, vp, vp, i, i, vp, vp], i),
        "ta_match": ([vp, i, i, i, i, vp, vp, vp, vp], i),
        "ta_match_qkv": ([vp, i, i, i, i, i, i, vp, vp, vp, vp], i),
        "ta_stage_name": ([i], ctypes.c_char_p),
        "ta_profile_stages": ([vp, i], i),
        "ta_stage_records": ([vp, ctypes.POINTER(StageRecord), i, ip], i),
        "ta_merge": ([vp, vp, i, i, i, i, vp, vp, vp, vp, vp, vp, vp, vp, i, vp], i),
        "ta_attention": ([vp, vp, i, i, i, i, vp, i, vp], i),
        "ta_gemm": ([vp, vp, vp, vp, vp, i, i, i, i, i, i, vp], i),
        "ta_layernorm": ([vp, vp, vp, vp, i, i, i, vp], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(l, name)
        fn.argtypes = args
        fn.restype = res


def lib() -> ctypes.CDLL:
    """Load (once) and return the CUDA library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not found: build it with `python __graft_entry__.py build` "
                "(make -C paper_2401_05031_b200/csrc); there is no CPU fallback")
        l = ctypes.CDLL(LIB_PATH)
        _declare(l)
        _lib = l
    return _lib


def check(code: int, *, task: Optional[str] = None, gamma: Optional[int] = None) -> None:
    """Raise the reference-convention exception for a non-zero status."""
    if code == TA_OK:
        return
    l = lib()
    msg = l.ta_strerror(code).decode()
    if code == TA_ERR_NO_PROMPT:
        raise ProfileGapError(task if task is not None else "?", gamma if gamma is not None else 0,
                              "prompt")
    if code in (TA_ERR_INVALID, TA_ERR_SHAPE):
        raise ValueError(f"tokadapt_cuda: {msg}")
    if code == TA_ERR_CONFIG:
        raise ConfigError(f"tokadapt_cuda: {msg}")
    if code == TA_ERR_CUDA:
        raise TAError(code, f"tokadapt_cuda: {msg} (cudaError {l.ta_last_cuda_error()})")
    raise TAError(code, f"tokadapt_cuda: {msg}")
