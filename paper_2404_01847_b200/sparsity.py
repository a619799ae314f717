"""Transposable 2:4 masks on the B200: pattern table, mask type and the
mask search (K1).  Mirrors sparse24.sparsity (sparsity.py:111-271).

A mask is held as its per-block canonical pattern index (`idx`, uint8,
rows/4 x cols/4, 1 byte per 16 weights) -- the full 0/1 `bits` matrix of the
reference is produced on demand by a kernel.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _capi as C
from .matrix import FormatError, ShapeError


@dataclass(frozen=True)
class PatternTable:
    """The 90 4x4 blocks with row and column sums 2, in lexicographic order of
    their row-major bits (sparsity.py:165-217)."""

    patterns: np.ndarray  # (90, 4, 4) uint8
    positions: np.ndarray  # (90, 8) int32

    def __len__(self) -> int:
        return len(self.patterns)

    @property
    def count(self) -> int:
        return len(self.patterns)

    def to_text(self) -> str:
        return "".join("".join(str(int(b)) for b in p.reshape(16)) + "\n" for p in self.patterns)

    def index_of(self, block) -> int:
        flat = np.asarray(block, dtype=np.uint8).reshape(16)
        hits = np.nonzero((self.patterns.reshape(-1, 16) == flat).all(axis=1))[0]
        if len(hits) == 0:
            raise KeyError("block is not a transposable pattern")
        return int(hits[0])


@lru_cache(maxsize=1)
def enumerate_patterns() -> PatternTable:
    rows = [r for r in itertools.product((0, 1), repeat=4) if sum(r) == 2]
    pats = sorted(
        sum(combo, ())
        for combo in itertools.product(rows, repeat=4)
        if all(sum(r[j] for r in combo) == 2 for j in range(4))
    )
    arr = np.array(pats, dtype=np.uint8).reshape(-1, 4, 4)
    pos = np.array([np.flatnonzero(p.reshape(16)) for p in arr], dtype=np.int32)
    return PatternTable(arr, pos)


@lru_cache(maxsize=None)
def _transpose_map(device: str) -> torch.Tensor:
    """pattern index -> index of its transpose (the table is transpose-closed); indices
    outside the table (invalid blocks) map to 255, so a lookup can never leave the table."""
    t = enumerate_patterns()
    lut = [t.index_of(p.T) for p in t.patterns] + [255] * (256 - len(t.patterns))
    return torch.tensor(lut, dtype=torch.uint8, device=device)


def _check_blocks(rows: int, cols: int) -> None:
    if rows % 4 or cols % 4:
        raise ShapeError(f"shape ({rows}, {cols}) not divisible into 4x4 blocks")


class TransposableMask:
    """Mask whose aligned 4x4 blocks hold two ones per block row and column
    (sparsity.py:111-145), stored as per-block pattern indices on the GPU.

    Built from a 0/1 `bits` matrix the mask also keeps those raw bits, as the
    reference does: an invalid mask (a block that is none of the 90 patterns)
    still reports, transposes and scores its own bits, and fails only in
    `validate()` (FormatError) -- which every consumer of the pattern indices
    (FFNMasks.plans, compress) runs first."""

    def __init__(self, idx: torch.Tensor | None = None, shape: tuple[int, int] | None = None,
                 bits: torch.Tensor | None = None):
        self._bad = None
        self._raw = None
        if bits is not None:
            C.require_cuda(bits)
            if bits.dim() != 2:
                raise FormatError("mask must be 2-D")
            rows, cols = bits.shape
            _check_blocks(rows, cols)
            b = bits.to(torch.uint8).contiguous()
            idx = torch.empty((rows // 4, cols // 4), dtype=torch.uint8, device=b.device)
            bad = torch.zeros(1, dtype=torch.int32, device=b.device)
            C.call("s24_bits_to_idx", b.data_ptr(), rows, cols, idx.data_ptr(), bad.data_ptr(), C.stream_of(b))
            self._bad = bad
            self._raw = b
            shape = (rows, cols)
        if idx is None or shape is None:
            raise ValueError("TransposableMask needs idx + shape, or bits")
        self.idx = idx
        self._shape = (int(shape[0]), int(shape[1]))

    @property
    def shape(self) -> tuple[int, int]:
        return self._shape

    @property
    def device(self):
        return self.idx.device

    def validate(self) -> None:
        """FormatError unless every block is one of the 90 patterns (sparsity.py:122-131)."""
        if self._bad is not None and int(self._bad.item()) != 0:
            raise FormatError("every 4x4 block must hold exactly two ones per block row and column")
        if self.idx.numel() and int(self.idx.max().item()) > 89:
            raise FormatError("invalid pattern index")

    @property
    def bits(self) -> torch.Tensor:
        if self._raw is not None:
            return self._raw
        rows, cols = self._shape
        out = torch.empty((rows, cols), dtype=torch.uint8, device=self.idx.device)
        C.call("s24_idx_to_bits", self.idx.data_ptr(), rows, cols, out.data_ptr(), C.stream_of(self.idx))
        return out

    def transpose(self) -> "TransposableMask":
        if self._raw is not None:  # sparsity.py:137-138: any 0/1 matrix transposes
            return TransposableMask(bits=self._raw.t().contiguous())
        lut = _transpose_map(str(self.idx.device))
        idx_t = lut[self.idx.t().long()].contiguous()
        return TransposableMask(idx_t, (self._shape[1], self._shape[0]))

    def to_mask24(self, direction) -> "Mask24":
        return Mask24(self.bits, direction)

    def retained_l1(self, w: torch.Tensor) -> float:
        return float((w.abs().double() * self.bits.double()).sum().item())

    def meta(self) -> tuple[torch.Tensor, torch.Tensor]:
        """Reference-layout metadata nibbles (Compressed24.meta, spmm.py:98-104)
        for the row-wise groups of W (rows x cols/4) and of W^T (cols x rows/4)."""
        rows, cols = self._shape
        f = torch.empty((rows, cols // 4), dtype=torch.uint8, device=self.idx.device)
        b = torch.empty((cols, rows // 4), dtype=torch.uint8, device=self.idx.device)
        C.call("s24_meta_flat", self.idx.data_ptr(), rows, cols, f.data_ptr(), b.data_ptr(), C.stream_of(self.idx))
        return f, b


def transposable_search_conv(w: torch.Tensor, table: PatternTable | None = None) -> TransposableMask:
    """Exhaustive per-block pattern search (sparsity.py:258-271), K1 on the GPU.

    Bit-exact with the reference: the selected pattern maximizes the retained
    |w| sum accumulated in float64 ascending order; ties go to the lowest
    canonical index.  `table` is accepted for signature compatibility (only the
    canonical table is supported)."""
    if w.dim() != 2:
        raise ShapeError(f"expected a 2-D operand, got ndim={w.dim()}")
    C.require_cuda(w)
    rows, cols = w.shape
    _check_blocks(rows, cols)
    w = w.contiguous()
    idx = torch.empty((rows // 4, cols // 4), dtype=torch.uint8, device=w.device)
    C.call("s24_transposable_search", w.data_ptr(), C.dtype_code(w), rows, cols, idx.data_ptr(), C.stream_of(w))
    return TransposableMask(idx, (rows, cols))


def transposable_search_greedy(w: torch.Tensor) -> TransposableMask:
    """2-approximation comparator (sparsity.py:229-238 -> kernels.greedy_masks, _core.pyx:139-219)
    on the GPU, bit-exact: per block, cells by descending |w| (lowest flat index on ties) are
    picked while their block row and column hold fewer than two picks, and a stranded block
    is completed by the single best swap.  Raises RuntimeError when a block cannot be
    completed, like the reference."""
    if w.dim() != 2:
        raise ShapeError(f"expected a 2-D operand, got ndim={w.dim()}")
    C.require_cuda(w)
    rows, cols = w.shape
    _check_blocks(rows, cols)
    w = w.contiguous()
    idx = torch.empty((rows // 4, cols // 4), dtype=torch.uint8, device=w.device)
    bad = torch.zeros(1, dtype=torch.int32, device=w.device)
    C.call("s24_greedy_search", w.data_ptr(), C.dtype_code(w), rows, cols, idx.data_ptr(), bad.data_ptr(),
           C.stream_of(w))
    if int(bad.item()):
        raise RuntimeError("greedy mask completion failed")
    return TransposableMask(idx, (rows, cols))


class Mask24:
    """0/1 mask with exactly two ones per aligned group of four along `direction`
    (sparsity.py:85-108): row-wise groups run along rows, column-wise down columns."""

    def __init__(self, bits: torch.Tensor, direction=None):
        from .matrix import Direction

        self.bits = bits if bits.dtype == torch.uint8 else bits.to(torch.uint8)
        self.direction = direction or Direction.ROW_WISE

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self.bits.shape)

    def validate(self) -> None:
        """FormatError unless every group holds exactly two 0/1 ones (sparsity.py:98-105),
        checked by the pack kernel in validation-only mode."""
        from .matrix import Direction

        if self.bits.dim() != 2:
            raise FormatError("mask must be 2-D")
        rows, cols = self.bits.shape
        colwise = self.direction is Direction.COL_WISE
        if colwise and rows % 4:
            raise ShapeError(f"rows={rows} not divisible by 4 for column-wise groups")
        if not colwise and cols % 4:
            raise ShapeError(f"cols={cols} not divisible by 4 for row-wise groups")
        C.require_cuda(self.bits)
        b = self.bits.contiguous()
        bad = torch.zeros(1, dtype=torch.int32, device=b.device)
        C.call("s24_pack24", None, C.S24_BF16, b.data_ptr(), rows, cols, int(colwise), None, None, bad.data_ptr(),
               C.stream_of(b))
        if int(bad.item()):
            raise FormatError("every group of 4 must contain exactly 2 ones")


class SparseEstimate:
    """A pruned matrix (zeros at dropped positions) with its Mask24 (sparsity.py:148-158).
    `bits` / `direction` are shorthands for the mask's."""

    def __init__(self, values: torch.Tensor, mask: Mask24):
        if tuple(values.shape) != tuple(mask.bits.shape):
            raise ShapeError("values and mask shapes differ")
        self.values = values
        self.mask = mask

    @property
    def bits(self) -> torch.Tensor:
        return self.mask.bits

    @property
    def direction(self):
        return self.mask.direction


def apply_mask(w: torch.Tensor, mask) -> torch.Tensor:
    """Elementwise product of a matrix with a binary mask (sparsity.py:241-251)."""
    bits = mask.bits if isinstance(mask, (Mask24, TransposableMask)) else mask
    if tuple(w.shape) != tuple(bits.shape):
        raise ShapeError(f"mask shape {tuple(bits.shape)} != matrix shape {tuple(w.shape)}")
    return w * bits.to(w.dtype)


def prune_2of4(m: torch.Tensor, direction=None) -> SparseEstimate:
    """Keep the two largest |m| of every aligned group of four along `direction`
    (sparsity.py:274-279 -> kernels.prune_2of4_keep, _core.pyx:113-136); ties keep the
    lowest indices.  Bit-exact on the GPU."""
    from .matrix import Direction

    direction = direction or Direction.ROW_WISE
    if m.dim() != 2:
        raise ShapeError(f"expected a 2-D operand, got ndim={m.dim()}")
    C.require_cuda(m)
    rows, cols = m.shape
    m = m.contiguous()
    bits = torch.empty((rows, cols), dtype=torch.uint8, device=m.device)
    C.call("s24_prune_2of4", m.data_ptr(), C.dtype_code(m), rows, cols, int(direction is Direction.COL_WISE),
           bits.data_ptr(), C.stream_of(m))
    return SparseEstimate(m * bits.to(m.dtype), Mask24(bits, direction))


# kept index pairs of a group, lexicographic (sparsity.py:283-285)
MVUE_PAIRS = np.array([(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], dtype=np.int64)


def mvue_prune(g: torch.Tensor, direction=None, rng_seed: int = 0) -> SparseEstimate:
    """Unbiased stochastic 2-of-4 sparsifier (sparsity.py:379-398) on the GPU: per group the
    water-filled inclusion probabilities, the greedy pair distribution, one uniform of numpy's
    default_rng(rng_seed) stream per group (group order of to_groups) and the kept values
    g / pi, all in float64 -- bit-exact with the reference.  Values come back float64."""
    from .engine import pcg64_state
    from .matrix import Direction

    direction = direction or Direction.ROW_WISE
    if g.dim() != 2:
        raise ShapeError(f"expected a 2-D operand, got ndim={g.dim()}")
    C.require_cuda(g)
    rows, cols = g.shape
    colwise = direction is Direction.COL_WISE
    if colwise and rows % 4:
        raise ShapeError(f"rows={rows} not divisible by 4 for column-wise groups")
    if not colwise and cols % 4:
        raise ShapeError(f"cols={cols} not divisible by 4 for row-wise groups")
    g = g.contiguous()
    out = torch.empty((rows, cols), dtype=torch.float64, device=g.device)
    bits = torch.empty((rows, cols), dtype=torch.uint8, device=g.device)
    sh, sl, ih, il = pcg64_state(rng_seed)
    C.call("s24_mvue_prune", g.data_ptr(), C.dtype_code(g), rows, cols, int(colwise), sh, sl, ih, il,
           out.data_ptr(), bits.data_ptr(), C.stream_of(g))
    return SparseEstimate(out, Mask24(bits, direction))
