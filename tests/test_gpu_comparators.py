"""GPU greedy transposable search and directional prune_2of4, bit-exact
against reference-generated goldens (tests/golden/comparators_golden.npz)."""
import os

import numpy as np
import pytest
import torch

from oracle import s24_oracle as o
from gpu_util import need_gpu
from make_golden import mask_corpora

pytestmark = pytest.mark.gpu
GD = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "comparators_golden.npz")))
NAMES = ["gauss_f64", "gauss_bf16", "int_ties", "kats"]


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _dev(w, tag):
    t = torch.from_numpy(w).cuda()
    return t if tag == "f64" else t.to(torch.bfloat16 if tag == "bf16" else torch.float32)


@pytest.mark.parametrize("name", NAMES)
def test_greedy_search_bit_exact(name):
    import paper_2404_01847_b200 as P

    w, tag = mask_corpora()[name]
    m = P.transposable_search_greedy(_dev(w, tag))
    assert np.array_equal(m.idx.cpu().numpy(), GD[f"{name}.greedy_idx"])
    m.validate()


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("col", [False, True])
def test_prune_2of4_bit_exact(name, col):
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.matrix import Direction

    w, tag = mask_corpora()[name]
    est = P.prune_2of4(_dev(w, tag), Direction.COL_WISE if col else Direction.ROW_WISE)
    assert np.array_equal(est.bits.cpu().numpy(), GD[f"{name}.prune_{'col' if col else 'row'}"])
    wd = _dev(w, tag)
    assert torch.equal(est.values, wd * est.bits.to(wd.dtype))


def test_greedy_never_beats_exhaustive_and_is_2_approx():
    """Bound chain of test_acceptance.py:153-166: greedy >= 0.5 optimum, exhaustive >= greedy."""
    import paper_2404_01847_b200 as P

    w = torch.from_numpy(o.det_normal((256, 256), 33)).cuda()
    a = w.abs()
    g = (a * P.transposable_search_greedy(w).bits.double()).reshape(64, 4, 64, 4).sum((1, 3))
    c = (a * P.transposable_search_conv(w).bits.double()).reshape(64, 4, 64, 4).sum((1, 3))
    assert bool((g >= 0.5 * c - 1e-12).all()) and bool((c >= g - 1e-12).all())


def test_prune_2of4_shape_errors():
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.matrix import Direction, ShapeError

    with pytest.raises(ShapeError):
        P.prune_2of4(torch.zeros(8, 6, device="cuda"))
    with pytest.raises(ShapeError):
        P.prune_2of4(torch.zeros(6, 8, device="cuda"), Direction.COL_WISE)
    with pytest.raises(ShapeError):
        P.transposable_search_greedy(torch.zeros(6, 8, device="cuda"))
