"""The reference's CPU FFN training step, for the CPU-baseline / reference
arm of bench.py -- TEST/BENCH INFRASTRUCTURE ONLY (never product code).

One step = what run_training does for one FFN block per iteration
(trainer.py:418-447) with mvue=False: per-step gather of the kept weights
(gated_ffn.py:159-162), fst_forward (gated_ffn.py:273-301), fst_backward
(gated_ffn.py:304-364), masked_decay_gradient (optim.py:105-114), and every
`refresh` steps a new transposable mask search of both weights + gather plans
(trainer.py:422-432, FFNMasks.plans gated_ffn.py:176-188).

The hot loops run in the reference's own compiled kernels
(oracle/_ref/_core*.so built from /root/reference/pkg/src/sparse24/_core.pyx,
`kind = "reference"`) when present, else in the numpy restatement of them in
s24_oracle (`kind = "port"`).  Cost is linear in tokens, so tokens/s measured
on a bounded token sample is the full-size rate.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import s24_oracle as o


class _PortKernels:
    """numpy restatement of the three kernels on the path (_core_py.py:41-63, 127-144)."""

    BACKEND_NAME = "port"
    pattern_scores = staticmethod(o.pattern_scores)
    spmm_colwise = staticmethod(o.spmm_colwise)

    @staticmethod
    def gate_gelu(z1, z2, row_order):
        return o.gate(z1, z2, "geglu")


def kernels():
    k = o.ref_kernels()
    return (k, "reference") if k is not None else (_PortKernels, "port")


class RefFFNStep:
    def __init__(self, d: int, d_ff: int, act: str, tokens: int, seed: int = 0, lam: float = 6e-5,
                 refresh: int = 40):
        self.k, self.kind = kernels()
        self.act, self.lam, self.refresh_period = act, lam, refresh
        r_in = 2 * d_ff if act in ("geglu", "swiglu") else d_ff
        self.d, self.d_ff, self.r_in = d, d_ff, r_in
        # reference init (trainer.py:180-191), values rounded to bf16 like the GPU inputs
        self.w_in = o.round_bf16(o.det_normal((r_in, d), seed + 1) / np.sqrt(d))
        self.w2 = o.round_bf16(o.det_normal((d, d_ff), seed + 2) / np.sqrt(d_ff))
        self.bias = np.zeros(r_in)
        self.x = o.round_bf16(o.det_normal((tokens, d), seed + 3))
        self.dy = o.round_bf16(o.det_normal((tokens, d), seed + 4) / np.sqrt(tokens * d))
        self.t = 0
        self.search_seconds = 0.0

    # -- mask refresh: search both weights + build the four gather plans
    def _search(self, w):
        _, pos = o.pattern_table()
        pats, _ = o.pattern_table()
        _, best = self.k.pattern_scores(np.abs(o.blocks16(w)), pos)
        return o.unblocks16(pats.reshape(90, 16)[best], w.shape)

    def refresh(self):
        t0 = time.perf_counter()
        self.m_in, self.m_out = self._search(self.w_in), self._search(self.w2)
        self.plans = {
            "in_fwd": o.gather_plan(self.m_in, False),
            "in_bwd": o.gather_plan(np.ascontiguousarray(self.m_in.T), True),
            "out_fwd": o.gather_plan(self.m_out, False),
            "out_bwd": o.gather_plan(np.ascontiguousarray(self.m_out.T), True),
        }
        self.search_seconds = time.perf_counter() - t0

    def _product(self, name, a, w):
        take, pos_t = self.plans[name]
        vals = w.ravel()[take]
        return self.k.spmm_colwise(np.ascontiguousarray(a), np.ascontiguousarray(vals.T), pos_t)

    def _activate(self, z):
        r = self.d_ff
        if self.act == "geglu":
            return self.k.gate_gelu(z[:, :r], z[:, r:], False)
        if self.act == "swiglu":
            return o.gate(z[:, :r], z[:, r:], "swiglu")
        if self.act == "gelu":
            return o.gelu(z)
        return np.maximum(z, 0.0)

    def step(self):
        if self.t % self.refresh_period == 0:
            self.refresh()
        self.t += 1
        z = self._product("in_fwd", self.x, self.w_in)
        z += self.bias
        a = self._activate(z)
        y = self._product("out_fwd", a, self.w2)
        da = self._product("out_bwd", self.dy, self.w2)
        dw2 = self.dy.T @ a
        r = self.d_ff
        if self.act in ("geglu", "swiglu"):
            f, fp = (o.gelu, o.gelu_grad) if self.act == "geglu" else (o.silu, o.silu_grad)
            z1, z2 = z[:, :r], z[:, r:]
            dz = np.concatenate([da * z2 * fp(z1), da * f(z1)], axis=1)
        elif self.act == "gelu":
            dz = da * o.gelu_grad(z)
        else:
            dz = da * (z > 0)
        dbias = dz.sum(axis=0)
        dx = self._product("in_bwd", dz, self.w_in)
        dw_in = dz.T @ self.x
        dw_in = o.masked_decay_gradient(dw_in, self.w_in, self.m_in, self.lam)
        dw2 = o.masked_decay_gradient(dw2, self.w2, self.m_out, self.lam)
        return y, dx, dw_in, dbias, dw2


def ref_slice(d: int, d_ff: int, act: str, target_weights: float = 12.6e6) -> int:
    """Hidden width of the bounded CPU sample: the largest d_ff' <= d_ff (a multiple of 4, d_ff
    divided by an integer) whose first weight has at most ~target_weights elements.  Every term
    of the step -- the four sparse products, the activation, both dW products, the decay and the
    mask search -- is linear in d_ff at fixed d and tokens, so tokens/s at d_ff' divided by
    d_ff / d_ff' is the full-width rate (used at C3 / C4, where one reference step over the full
    weights takes minutes and tens of GB per process)."""
    r_mult = 2 if act in ("geglu", "swiglu") else 1
    f = 1
    while d * r_mult * (d_ff // f) > target_weights and d_ff // (f + 1) >= 4:
        f += 1
    return max(4, (d_ff // f) // 4 * 4)


def time_reference(d, d_ff, act, tokens, steps, warmup=1, refresh=40, budget_s=None, d_ff_sample=None):
    """Seconds per step (mask search amortized over `refresh` steps) on a `tokens` sample,
    scaled to the full hidden width when `d_ff_sample` < d_ff (see ref_slice).  Returns
    (sec_per_step, info)."""
    dfs = d_ff if d_ff_sample is None else int(d_ff_sample)
    st = RefFFNStep(d, dfs, act, tokens, refresh=refresh)
    st.refresh()
    search_s = st.search_seconds
    st.t = 1  # skip the refresh inside the timed steps; add it amortized below
    for _ in range(warmup):
        st.step()
    t0 = time.perf_counter()
    n = 0
    while n < steps:
        st.t = 1  # keep masks: refresh cost is accounted for once, amortized
        st.step()
        n += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    per = ((time.perf_counter() - t0) / n + search_s / refresh) * (d_ff / dfs)
    cores = 1 if st.kind == "reference" else os.cpu_count()
    return per, dict(kind=st.kind, steps=n, search_s=search_s, cores=cores, d_ff_sample=dfs)
