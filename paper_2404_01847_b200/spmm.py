"""Packed 2:4 storage and the packed-route products on the B200 (spmm.py:38-190).

The reference keeps this route as its correctness tool: a Compressed24 holds the kept
values in group order plus one metadata nibble i0 | i1 << 2 per group of four (one per
uint8), row-wise groups row-major and column-wise groups column-major, and spmm /
spmm_right multiply through it.  Here the buffers live on the GPU, compress / decompress /
mask_of run as kernels (s24_pack24 / s24_unpack24) and the products run on the 2:4 tensor
cores: a row-wise Compressed24's value order is exactly the sparse GEMM's operand order,
so only its nibbles are rearranged into E tiles (s24_flat_to_e).  Products take bf16
operands (other value dtypes are rounded to bf16) and accumulate in fp32, so they match
the reference's float64 dense_matmul within a bf16 tolerance, not bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _capi as C
from .matrix import Direction, FormatError, ShapeError
from .sparsity import Mask24, SparseEstimate

__all__ = [
    "Compressed24",
    "compress",
    "compress_masked",
    "decompress",
    "mask_of",
    "transpose_view",
    "spmm",
    "spmm_right",
    "dense_matmul",
    "dense_matmul_flops",
    "sparse_matmul_flops",
]


@dataclass
class Compressed24:
    """Packed 2:4 sparse storage (spmm.py:38-89): `values` (rows*cols/2, any of bf16 /
    fp32 / fp64) and `meta` (rows*cols/4 uint8 nibbles) on one CUDA device."""

    rows: int
    cols: int
    direction: Direction
    values: torch.Tensor
    meta: torch.Tensor

    def __post_init__(self) -> None:
        self.values = self.values.reshape(-1)
        self.meta = self.meta.reshape(-1)
        if self.meta.dtype != torch.uint8:
            raise FormatError("metadata must be uint8 nibbles")
        n = self.rows * self.cols
        if self.values.numel() != n // 2 or self.meta.numel() != n // 4:
            raise FormatError("compressed buffer sizes do not match the dense shape")

    @property
    def colwise(self) -> bool:
        return self.direction is Direction.COL_WISE

    def _unpack(self, out: torch.Tensor | None, bits: torch.Tensor | None) -> None:
        bad = torch.zeros(1, dtype=torch.int32, device=self.meta.device)
        vals = self.values.contiguous()
        C.call("s24_unpack24", vals.data_ptr(), C.dtype_code(vals), self.meta.contiguous().data_ptr(), self.rows,
               self.cols, int(self.colwise), C.ptr(out), C.ptr(bits), bad.data_ptr(), C.stream_of(self.meta))
        if int(bad.item()):
            raise FormatError("metadata indices must be distinct and ascending")

    def kept_indices(self) -> tuple[torch.Tensor, torch.Tensor]:
        """Per-group kept indices (i0, i1), each in 0..3, i0 < i1 (spmm.py:56-63)."""
        self._unpack(None, None)
        return (self.meta & 3).to(torch.int64), ((self.meta >> 2) & 3).to(torch.int64)


def _check_groups(rows: int, cols: int, direction: Direction) -> None:
    if direction is Direction.ROW_WISE and cols % 4:
        raise ShapeError(f"cols={cols} not divisible by 4 for row-wise groups")
    if direction is Direction.COL_WISE and rows % 4:
        raise ShapeError(f"rows={rows} not divisible by 4 for column-wise groups")


def compress(s: SparseEstimate) -> Compressed24:
    """Pack a pruned matrix (spmm.py:92-106): per group the first and last kept index, the
    two values copied verbatim.  FormatError unless the mask is a valid 2:4 mask."""
    w, bits, direction = s.values, s.mask.bits, s.mask.direction
    if w.dim() != 2:
        raise ShapeError(f"expected a 2-D operand, got ndim={w.dim()}")
    C.require_cuda(w, bits)
    rows, cols = w.shape
    _check_groups(rows, cols, direction)
    w, b = w.contiguous(), bits.contiguous()
    vals = torch.empty(rows * cols // 2, dtype=w.dtype, device=w.device)
    meta = torch.empty(rows * cols // 4, dtype=torch.uint8, device=w.device)
    bad = torch.zeros(1, dtype=torch.int32, device=w.device)
    C.call("s24_pack24", w.data_ptr(), C.dtype_code(w), b.data_ptr(), rows, cols,
           int(direction is Direction.COL_WISE), vals.data_ptr(), meta.data_ptr(), bad.data_ptr(), C.stream_of(w))
    if int(bad.item()):
        raise FormatError("every group of 4 must contain exactly 2 ones")
    return Compressed24(rows, cols, direction, vals, meta)


def compress_masked(w: torch.Tensor, mask: Mask24) -> Compressed24:
    """compress(apply_mask(w, mask)) (spmm.py:109-114); the kernel reads only kept entries,
    so the masked estimate is never materialised."""
    if tuple(w.shape) != tuple(mask.bits.shape):
        raise ShapeError("weight and mask shapes differ")
    return compress(SparseEstimate(w, mask))


def decompress(c: Compressed24) -> torch.Tensor:
    """Dense matrix with the kept values at their metadata positions (spmm.py:117-129);
    a column-wise operand comes back with column-major strides, like the reference's
    Matrix.col_major."""
    out = torch.empty((c.rows, c.cols), dtype=c.values.dtype, device=c.values.device)
    c._unpack(out, None)
    if c.colwise:
        return out.t().contiguous().t()
    return out


def mask_of(c: Compressed24) -> Mask24:
    """The 0/1 mask encoded by the metadata (spmm.py:132-139)."""
    bits = torch.empty((c.rows, c.cols), dtype=torch.uint8, device=c.meta.device)
    c._unpack(None, bits)
    return Mask24(bits, c.direction)


def transpose_view(c: Compressed24) -> Compressed24:
    """Transpose without copying (spmm.py:142-148): row-wise (m, k) becomes column-wise
    (k, m) over the same buffers."""
    d = Direction.COL_WISE if c.direction is Direction.ROW_WISE else Direction.ROW_WISE
    return Compressed24(c.cols, c.rows, d, c.values, c.meta)


# ---------------------------------------------------------------------------
# products on the tensor cores


def _ceil(x: int, q: int) -> int:
    return (x + q - 1) // q * q


def _bf16_2d(x: torch.Tensor, name: str) -> torch.Tensor:
    if x.dim() != 2:
        raise ShapeError(f"expected a 2-D {name}, got ndim={x.dim()}")
    C.require_cuda(x)
    return x if x.dtype == torch.bfloat16 else x.to(torch.bfloat16)


def _sparse_product(vals: torch.Tensor, meta: torch.Tensor, m: int, k: int, b_nk: torch.Tensor,
                    out_nm: bool) -> torch.Tensor:
    """D[m, n] = A~[m, k] B[n, k]^T with A~ row-wise 2:4 (values m x k/2, nibbles m x k/4),
    B given n x k.  Pads to the kernel's tile multiples (pad groups keep (0, 1) with zero
    values).  out_nm: return the (n, m) token-major result instead of (m, n)."""
    n = b_nk.shape[0]
    dev = vals.device
    M, K, N = _ceil(max(m, 1), 128), _ceil(max(k, 1), 128), _ceil(max(n, 1), 32)
    v = torch.zeros((M, K // 2), dtype=torch.bfloat16, device=dev)
    v[:m, :k // 2] = vals.reshape(m, k // 2)
    mt = torch.full((M, K // 4), 4, dtype=torch.uint8, device=dev)
    mt[:m, :k // 4] = meta.reshape(m, k // 4)
    e = torch.empty(M * K // 8, dtype=torch.uint8, device=dev)
    C.call("s24_flat_to_e", mt.data_ptr(), M, K, e.data_ptr(), C.stream_of(mt))
    b = torch.zeros((N, K), dtype=torch.bfloat16, device=dev)
    b[:n, :k] = b_nk
    if out_nm:
        d = torch.empty((N, M), dtype=torch.bfloat16, device=dev)
    else:
        d = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    C.call("s24_spmm", v.data_ptr(), e.data_ptr(), M, K, b.data_ptr(), 0, K, N, d.data_ptr(), d.stride(0), None,
           C.EPI_STORE, None, 0, None, None, int(out_nm), 0, None, 0, C.stream_of(d))
    return d[:n, :m] if out_nm else d[:m, :n]


def spmm(a: Compressed24, b: torch.Tensor) -> torch.Tensor:
    """C = A @ B with A row-wise 2:4 compressed (spmm.py:165-178), on the 2:4 tensor cores
    (bf16 operands, fp32 accumulation, bf16 result)."""
    if a.direction is not Direction.ROW_WISE:
        raise FormatError("left operand must be row-wise compressed")
    b = _bf16_2d(b, "operand")
    if a.cols != b.shape[0]:
        raise ShapeError(f"inner dims differ: ({a.rows},{a.cols}) x {tuple(b.shape)}")
    a.kept_indices()  # FormatError on malformed metadata, like the reference
    return _sparse_product(a.values, a.meta, a.rows, a.cols, b.t(), out_nm=False)


def spmm_right(a: torch.Tensor, b: Compressed24) -> torch.Tensor:
    """C = A @ B with B column-wise 2:4 compressed (spmm.py:181-190): C^T = B^T A^T with
    B^T the row-wise view of the same buffers; the result has column-major strides, like
    the reference's."""
    if b.direction is not Direction.COL_WISE:
        raise FormatError("right operand must be column-wise compressed")
    a = _bf16_2d(a, "operand")
    if a.shape[1] != b.rows:
        raise ShapeError(f"inner dims differ: {tuple(a.shape)} x ({b.rows},{b.cols})")
    b.kept_indices()
    bt = transpose_view(b)  # row-wise (cols x rows)
    return _sparse_product(bt.values, bt.meta, bt.rows, bt.cols, a, out_nm=False).t()


def dense_matmul(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """A @ B on the dense tcgen05 GEMM (spmm.py:154-162): bf16 operands, fp32 result."""
    a, b = _bf16_2d(a, "operand"), _bf16_2d(b, "operand")
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"inner dims differ: {tuple(a.shape)} x {tuple(b.shape)}")
    m, k = a.shape
    n = b.shape[1]
    M, K, N = _ceil(max(m, 1), 128), _ceil(max(k, 1), 64), _ceil(max(n, 1), 128)
    ap = torch.zeros((M, K), dtype=torch.bfloat16, device=a.device)
    ap[:m, :k] = a
    bp = torch.zeros((K, N), dtype=torch.bfloat16, device=a.device)
    bp[:k, :n] = b
    d = torch.empty((M, N), dtype=torch.float32, device=a.device)
    C.call("s24_gemm_dw", ap.data_ptr(), 0, K, bp.data_ptr(), 1, N, M, N, K, d.data_ptr(), N, None, 0, None, 0.0,
           0, 0, None, 0, C.stream_of(d))
    return d[:m, :n]


def dense_matmul_flops(m: int, k: int, n: int) -> int:
    return 2 * m * k * n


def sparse_matmul_flops(m: int, k: int, n: int) -> int:
    """Half the dense count: two of every four contraction terms are skipped."""
    return m * k * n
