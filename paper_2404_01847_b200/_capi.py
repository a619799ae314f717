"""ctypes binding of the C ABI (include/sparse24_b200.h) -> libs24b200.so.

The library is the only compute path: if it is missing this module raises on
first use (no CPU fallback).  Status codes map to the reference's exception
types (matrix.py:11-16): S24_ERR_SHAPE -> ShapeError, S24_ERR_FORMAT ->
FormatError, everything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .matrix import FormatError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
# S24_LIB_PATH: load a differently-built variant of the same library (build experiments)
LIB_PATH = os.environ.get("S24_LIB_PATH") or os.path.join(_HERE, "libs24b200.so")

S24_OK, S24_ERR_SHAPE, S24_ERR_FORMAT, S24_ERR_UNSUPPORTED, S24_ERR_CUDA, S24_ERR_ARG = range(6)
S24_BF16, S24_F32, S24_F64 = 0, 1, 2
ACT_RELU, ACT_GELU, ACT_GEGLU, ACT_SWIGLU = 0, 1, 2, 3
GEMM_WORKSPACE_BYTES, GEMM_WS_TIMEOUTS_WORD = 8448, 2  # S24_GEMM_WORKSPACE_BYTES (header)
EPI_STORE, EPI_GELU_AUX, EPI_GELU_GRAD, EPI_DGELU, EPI_GEGLU_GRAD, EPI_SWIGLU_GRAD, EPI_DGATED, EPI_STORE_ADD = range(8)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_F = ctypes.c_float

# name -> argtypes (every entry point returns int status)
SIGNATURES = {
    "s24_abi_version": [],
    "s24_device_check": [],
    "s24_transposable_search": [_P, _I, _I64, _I64, _P, _P],
    "s24_search_compress": [_P, _I, _I64, _I64, _P, _P, _P, _P, _P, _I64, _P],
    "s24_search_compress_pair": [_P, _P, _I, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                 _I64, _I64, _P],
    "s24_prune_compress": [_P, _I, _I64, _I64, _P, _P, _P, _P, _P, _I64, _P],
    "s24_idx_to_bits": [_P, _I64, _I64, _P, _P],
    "s24_bits_to_idx": [_P, _I64, _I64, _P, _P, _P],
    "s24_meta_flat": [_P, _I64, _I64, _P, _P, _P],
    "s24_e_to_flat": [_P, _I64, _I64, _P, _P],
    "s24_spmm": [_P, _P, _I64, _I64, _P, _I, _I64, _I64, _P, _I64, _P, _I, _P, _I64, _P, _P, _I, _I64, _P, _I, _P],
    "s24_gemm_dw": [_P, _I, _I64, _P, _I, _I64, _I64, _I64, _I64, _P, _I64, _P, _I, _P, _F, _I64, _I, _P, _I, _P],
    "s24_gemm_act": [_P, _I, _I64, _I64, _I64, _I64, _P, _I64, _I64, _P, _I64, _P, _I, _P, _P, _P, _I64, _P, _I,
                     _P],
    "s24_mvue_compress": [_P, _I64, _I64, _I64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                          ctypes.c_uint64, _I64, _P, _P, _P, _I, _P],
    "s24_mvue_compress_ragged": [_P, _I64, _I64, _I64, _I64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_uint64, _I64, _P, _P, _P, _I, _P],
    "s24_spmm_dw": [_P, _P, _I64, _I64, _P, _I, _I64, _I64, _P, _I64, _P, _I, _P, _F, _I64, _I, _P, _I, _P],
    "s24_act_fwd": [_P, _I64, _I64, _I64, _I, _P, _I64, _P],
    "s24_act_bwd": [_P, _I64, _P, _I64, _I64, _I64, _I, _P, _I64, _P, _P],
    "s24_transpose_bf16": [_P, _I64, _I64, _I64, _P, _I64, _P],
    "s24_masked_decay": [_P, _P, _I, _P, _I64, _I64, _F, _P],
    "s24_masked_decay_bits": [_P, _P, _I, _P, _I64, _F, _P],
    "s24_split_bf16": [_P, _I64, _P, _P, _P],
    "s24_act_fwd_f32": [_P, _I64, _P, _I64, _I64, _I, _P, _I64, _P, _P, _P],
    "s24_act_bwd_f32": [_P, _I64, _P, _I64, _I64, _I64, _I, _P, _I64, _P, _P, _P, _P],
    "s24_adam_step": [_P, _P, _P, _I, _P, _I, _I64, _I64, _P] + [ctypes.c_double] * 10 + [_I, _P],
    "s24_adam_compress": [_P, _P, _P, _P, _I64, _I64, _P] + [ctypes.c_double] * 10 + [_I, _P, _P, _I64, _P],
    "s24_mask_flips": [_P, _P, _I64, _P, _P, _P],
    "s24_greedy_search": [_P, _I, _I64, _I64, _P, _P, _P],
    "s24_prune_compress_pair": [_P, _P, _I, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _I64, _I64, _P],
    "s24_prune_2of4": [_P, _I, _I64, _I64, _I, _P, _P],
    "s24_block_gaps": [_P, _I, _I64, _I64, _P, _P],
    "s24_pack24": [_P, _I, _P, _I64, _I64, _I, _P, _P, _P, _P],
    "s24_unpack24": [_P, _I, _P, _I64, _I64, _I, _P, _P, _P, _P],
    "s24_flat_to_e": [_P, _I64, _I64, _P, _P],
    "s24_mvue_prune": [_P, _I, _I64, _I64, _I, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                       _P, _P, _P],
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"sparse24 B200 library not built ({path}); run `python -m paper_2404_01847_b200.build` "
                "or __graft_entry__.build().  There is no CPU fallback."
            )
        lib = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        lib.s24_last_error_string.argtypes = []
        lib.s24_last_error_string.restype = ctypes.c_char_p
        lib.s24_gemm_workspace_bytes.argtypes = []
        lib.s24_gemm_workspace_bytes.restype = ctypes.c_int64
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == S24_OK:
        return
    msg = _lib.s24_last_error_string().decode(errors="replace")
    if rc == S24_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == S24_ERR_FORMAT:
        raise FormatError(msg)
    raise RuntimeError(f"sparse24 B200 kernel error {rc}: {msg}")


def call(name: str, *args) -> None:
    lib = _lib or load()
    check(getattr(lib, name)(*args))


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_of(t: torch.Tensor | None = None) -> int:
    dev = t.device if t is not None else torch.device("cuda")
    return torch.cuda.current_stream(dev).cuda_stream


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return S24_BF16
    if t.dtype == torch.float32:
        return S24_F32
    if t.dtype == torch.float64:
        return S24_F64
    raise RuntimeError(f"unsupported dtype {t.dtype} (bf16 / fp32 / fp64 weights)")


def require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("the B200 path takes CUDA tensors only (no CPU fallback)")
