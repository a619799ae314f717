"""Shared helpers for the -m gpu tests (test infrastructure)."""
import numpy as np
import pytest
import torch

from oracle import s24_oracle as o


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2404_01847_b200._capi as C
    C.load()
    C.call("s24_device_check")


def to_dev_bf16(x: np.ndarray) -> torch.Tensor:
    """float64 array of bf16-representable values -> CUDA bf16 (bit-exact)."""
    bits = o.bf16_bits(x).astype(np.int16)
    return torch.from_numpy(bits).cuda().view(torch.bfloat16)


def bf16_bits_of(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def normwise_rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
