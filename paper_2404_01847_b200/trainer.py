"""End-to-end 2:4 sparse training loop on the GPU: the
reference's `run_training` (trainer.py:387-480) over a residual stack of FFN blocks
(`_FFNStack`, trainer.py:159-262) whose layers are this package's SparseFFN (the hot
path: K1/K2 mask search and compression, 2:4 tcgen05 GEMMs, fused activation epilogues,
dense dW GEMMs with the fused masked decay), updated by the fused Adam kernel
(optim.adam_step).  Same configuration surface and schedule semantics as the reference:

  * lr warm-up + cosine schedule (`_lr_at`, trainer.py:375-384);
  * optional dense pre-training steps and the dense fine-tune switch at
    t_s = ceil(T (1 - f)) (TrainConfig.switch_step / pretrain_steps, trainer.py:111-119);
  * mask refresh every `decay.refresh_period` optimizer steps while sparse, with the flip
    rate of each refresh (trainer.py:422-432);
  * masked decay on the gradients (fused in the dW epilogue) or on the weights (fused in
    the Adam kernel) (trainer.py:438-447);
  * MVUE-sparsified weight gradients with the reference's per-step, per-layer seeds
    (trainer.py:245-247) when `mvue` is set.

The synthetic tasks (teacher-student regression, synthetic classification,
trainer.py:265-343) are generated on the host with the reference's numpy RNG streams,
so a run sees the reference's exact data and initial weights; the arithmetic is the GPU's
(bf16 tensor-core GEMMs, fp32 master weights and Adam state), so loss curves agree with
the reference's float64 CPU run to bf16 tolerance, not bitwise.
"""

from __future__ import annotations

import dataclasses
import json
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import engine as E
from .matrix import ShapeError
from .module import SparseFFN
from .optim import DecayConfig, DecayMode, OptimizerState, adam_step, block_flip_stats, mask_flips
from .sparsity import TransposableMask

_SALT_INIT = 0x12171
_SALT_TASK = 0xDA7A
_SALT_TEACHER = 0x7EAC
_SALT_EVAL = 0xE7A1
_SALT_MVUE = 0x6D76


class TaskKind(Enum):
    TEACHER_STUDENT_REGRESSION = "teacher_student_regression"
    SYNTHETIC_CLASSIFICATION = "synthetic_classification"


_ACTS = {"gelu": "gelu", "geglu": "geglu", "relu": "relu", "swiglu": "swiglu"}


@dataclass
class TrainConfig:
    """trainer.py:73-152 (field names and defaults of the reference; `activation` is the
    reference Activation value string; the reference's Activation enum is accepted and
    coerced to it).  The tensor-core path needs d, d_ff % 128 == 0; the batch is any multiple
    of 4 like the reference's (MVUE groups 4 tokens): it is zero-padded to the 64-token granule
    of the GEMMs (and to 128 for the MVUE operand, the reference's draws for the real tokens)."""

    d: int = 128
    d_ff: int = 256
    depth: int = 2
    batch: int = 128
    steps: int = 2000
    task: TaskKind = TaskKind.TEACHER_STUDENT_REGRESSION
    activation: str = "geglu"
    seed: int = 0
    lr: float = 1e-2
    warmup_fraction: float = 0.05
    lr_floor_fraction: float = 0.0
    dense_ft_fraction: float = 1.0 / 6.0
    dense_pretrain_fraction: float = 0.0
    sparse: bool = True
    decay: DecayConfig = field(default_factory=DecayConfig)
    mvue: bool = True
    proxy_flips: bool = False  # per-step mask search on the current weights (dense-run proxy)
    eval_batches: int = 8
    n_classes: int = 4
    schedule_total_steps: int | None = None
    collect_block_stats: bool = False  # trainer.py:93: weight snapshots at refreshes -> block_flip_stats

    def __post_init__(self) -> None:
        if hasattr(self.activation, "value"):  # the reference's Activation enum (gated_ffn.py:47-50)
            self.activation = self.activation.value
        if self.steps < 1:
            raise ValueError("steps must be >= 1")
        for name in ("d", "d_ff"):
            if getattr(self, name) % 128 != 0:
                raise ShapeError(f"{name} must be divisible by 128 on the tensor-core path")
        if self.batch < 4 or self.batch % 4 != 0:
            raise ShapeError("batch must be a positive multiple of 4 (MVUE groups of 4 tokens)")
        for name in ("dense_ft_fraction", "dense_pretrain_fraction", "warmup_fraction"):
            frac = getattr(self, name)
            if not (0.0 <= frac < 1.0):
                raise ValueError(f"{name} must lie in [0, 1)")
        if self.depth < 1:
            raise ValueError("depth must be >= 1")
        if self.activation not in _ACTS:
            raise ValueError(f"unknown activation {self.activation}")

    @property
    def switch_step(self) -> int:
        """Last sparse step before dense fine-tuning takes over (trainer.py:111-114)."""
        return math.ceil(self.steps * (1.0 - self.dense_ft_fraction))

    @property
    def pretrain_steps(self) -> int:
        """Dense steps at the start (trainer.py:116-119)."""
        return self.steps - math.ceil(self.steps * (1.0 - self.dense_pretrain_fraction))

    def to_dict(self) -> dict:
        out = dataclasses.asdict(self)
        out["task"] = self.task.value
        out["decay"]["mode"] = self.decay.mode.value
        return out

    @classmethod
    def from_dict(cls, data: dict) -> "TrainConfig":
        data = dict(data)
        if "task" in data:
            data["task"] = TaskKind(data["task"])
        if "decay" in data and isinstance(data["decay"], dict):
            dec = dict(data["decay"])
            if "mode" in dec:
                dec["mode"] = DecayMode(dec["mode"])
            data["decay"] = DecayConfig(**dec)
        return cls(**data)

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2)

    @classmethod
    def from_json(cls, text: str) -> "TrainConfig":
        return cls.from_dict(json.loads(text))


# ---------------------------------------------------------------------------
# host-side reference data streams (trainer.py:159-343): parameters and batches


def _rng(seed: int, salt: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([seed & 0xFFFF_FFFF, salt]))


def init_params(d: int, d_ff: int, depth: int, gated: bool, rng: np.random.Generator) -> list[dict]:
    """_FFNStack.init_params (trainer.py:180-191): per block w_in ~ N(0,1)/sqrt(d) then
    w2 ~ N(0,1)/sqrt(d_ff) from one stream, biases zero.  float64 host arrays."""
    r_in = 2 * d_ff if gated else d_ff
    out = []
    for _ in range(depth):
        w_in = rng.standard_normal((r_in, d)) / math.sqrt(d)
        w2 = rng.standard_normal((d, d_ff)) / math.sqrt(d_ff)
        out.append({"w_in": w_in, "bias": np.zeros(r_in), "w2": w2})
    return out


def _np_gelu(x):
    from math import sqrt

    import scipy.special as sp

    return 0.5 * x * (1.0 + sp.erf(x / sqrt(2.0)))


def _np_stack_forward(params: list[dict], x: np.ndarray, act: str, d_ff: int) -> np.ndarray:
    """Dense float64 residual FFN stack (the teacher of the regression task,
    trainer.py:228-236 with masks=None)."""
    h = x
    for p in params:
        z = h @ p["w_in"].T + p["bias"]
        if act in ("geglu", "swiglu"):
            u, v = z[:, :d_ff], z[:, d_ff:]
            a = (_np_gelu(u) if act == "geglu" else u / (1.0 + np.exp(-u))) * v
        elif act == "gelu":
            a = _np_gelu(z)
        else:
            a = np.maximum(z, 0.0)
        h = h + a @ p["w2"].T
    return h


class Task:
    """Deterministic mini-batch stream (trainer.py:268-343) with the reference's RNG
    streams; loss and upstream gradient are computed on the GPU."""

    def __init__(self, cfg: TrainConfig):
        self.cfg = cfg
        self._rng = _rng(cfg.seed, _SALT_TASK)
        rng_t = _rng(cfg.seed, _SALT_TEACHER)
        if cfg.task is TaskKind.TEACHER_STUDENT_REGRESSION:
            self._teacher = init_params(cfg.d, cfg.d_ff, cfg.depth, cfg.activation in ("geglu", "swiglu"), rng_t)
        else:
            self._means = rng_t.standard_normal((cfg.n_classes, cfg.d))

    def _make_batch(self, rng):
        c = self.cfg
        if c.task is TaskKind.TEACHER_STUDENT_REGRESSION:
            x = rng.standard_normal((c.batch, c.d))
            return x, _np_stack_forward(self._teacher, x, c.activation, c.d_ff)
        labels = rng.integers(0, c.n_classes, size=c.batch)
        x = self._means[labels] + 0.5 * rng.standard_normal((c.batch, c.d))
        return x, labels

    def next_batch(self):
        return self._make_batch(self._rng)

    def eval_batches(self, n: int):
        rng = _rng(self.cfg.seed, _SALT_EVAL)
        return [self._make_batch(rng) for _ in range(n)]

    def loss_and_grad(self, out: torch.Tensor, target: torch.Tensor):
        """trainer.py:321-343 on the device (fp32): MSE (2 diff / size) or softmax
        cross-entropy over the first n_classes outputs (mean over the batch)."""
        out = out.float()
        if self.cfg.task is TaskKind.TEACHER_STUDENT_REGRESSION:
            diff = out - target
            return (diff * diff).mean(), 2.0 * diff / diff.numel()
        k = self.cfg.n_classes
        logits = out[:, :k] - out[:, :k].max(dim=1, keepdim=True).values
        p = torch.softmax(logits, dim=1)
        rows = torch.arange(len(target), device=out.device)
        loss = -torch.log(p[rows, target]).mean()
        dl = p.clone()
        dl[rows, target] -= 1.0
        dout = torch.zeros_like(out)
        dout[:, :k] = dl / len(target)
        return loss, dout


# ---------------------------------------------------------------------------
# model and loop


class FFNStack(torch.nn.Module):
    """Residual stack of SparseFFN blocks (the B200 counterpart of _FFNStack)."""

    def __init__(self, cfg: TrainConfig, params: list[dict], device):
        super().__init__()
        self.cfg = cfg
        self.layers = torch.nn.ModuleList()
        for p in params:
            w_in = torch.from_numpy(p["w_in"]).to(device, torch.float32)
            b = torch.from_numpy(p["bias"]).to(device, torch.float32)
            w2 = torch.from_numpy(p["w2"]).to(device, torch.float32)
            self.layers.append(SparseFFN.from_weights(w_in, b, w2, _ACTS[cfg.activation],
                                                      refresh_period=cfg.decay.refresh_period))
        self.size = sum(p.numel() for p in self.parameters())

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        h = x
        for layer in self.layers:
            h = h + layer(h)
        return h

    def set_sparse(self, sparse: bool) -> None:
        for layer in self.layers:
            layer.sparse = sparse

    def masks(self):
        """(weight, TransposableMask) of every sparse weight, block order."""
        out = []
        for layer in self.layers:
            out.append((layer.w_in, TransposableMask(layer.op_in.mask_idx(), tuple(layer.w_in.shape))))
            out.append((layer.w2, TransposableMask(layer.op_out.idx, tuple(layer.w2.shape))))
        return out


@dataclass
class RunArtifacts:
    config: TrainConfig
    losses: np.ndarray  # length T
    flips: np.ndarray  # length T; refresh steps carry the flip rate (the proxy rates of a dense proxy run)
    final_params: list[dict]
    final_eval_loss: float
    mask_search_calls: int
    proxy_rates: np.ndarray | None = None
    block_stats: list | None = None  # [(name, FlipTrace)] when cfg.collect_block_stats (trainer.py:463-468)


def _proxy_masks(stack: "FFNStack") -> list[TransposableMask]:
    from .sparsity import transposable_search_conv

    out = []
    for layer in stack.layers:
        out.append(transposable_search_conv(layer.w_in.detach()))
        out.append(transposable_search_conv(layer.w2.detach()))
    return out


def _flips_between(a: list[TransposableMask], b: list[TransposableMask], size: int) -> float:
    return float(sum(mask_flips(x, y) for x, y in zip(a, b))) / size


def lr_at(t: int, total: int, peak: float, warmup_fraction: float, floor_fraction: float) -> float:
    """trainer.py:375-384: linear warm-up then cosine decay to the floor."""
    warmup = max(1, int(round(warmup_fraction * total)))
    if t <= warmup:
        return peak * t / warmup
    floor = floor_fraction * peak
    frac = (t - warmup) / max(1, total - warmup)
    return floor + (peak - floor) * 0.5 * (1.0 + math.cos(math.pi * min(frac, 1.0)))


def layer_mvue_seed(seed: int, step: int, blk: int) -> int:
    """Per-step, per-layer MVUE seed of _FFNStack.backward (trainer.py:245-247)."""
    return int(np.random.SeedSequence([int(seed) & 0xFFFF_FFFF, _SALT_MVUE, step, blk]).generate_state(1, np.uint64)[0])


def run_training(cfg: TrainConfig, device="cuda") -> RunArtifacts:
    """trainer.py:387-480 on the GPU; deterministic data given cfg.seed."""
    dev = torch.device(device)
    gated = cfg.activation in ("geglu", "swiglu")
    params = init_params(cfg.d, cfg.d_ff, cfg.depth, gated, _rng(cfg.seed, _SALT_INIT))
    stack = FFNStack(cfg, params, dev)
    states = [OptimizerState(w=p.data, u=torch.zeros_like(p.data), v=torch.zeros_like(p.data), lr=cfg.lr)
              for p in stack.parameters()]
    task = Task(cfg)
    T = cfg.steps
    t_switch = cfg.switch_step if cfg.dense_ft_fraction > 0 else T
    t_pre = cfg.pretrain_steps
    sched_total = cfg.schedule_total_steps or T
    lam = cfg.decay.lambda_w
    losses = torch.zeros(T, dtype=torch.float32, device=dev)
    flips = np.zeros(T)
    searches = 0
    have_masks = False
    since_refresh = 0
    proxy = np.zeros(T) if cfg.proxy_flips else None
    snapshots: dict = {}
    prev_proxy = None
    if proxy is not None:
        prev_proxy = _proxy_masks(stack)
        searches += 2 * cfg.depth

    for t in range(1, T + 1):
        lr = lr_at(t, sched_total, cfg.lr, cfg.warmup_fraction, cfg.lr_floor_fraction)
        sparse_now = cfg.sparse and t_pre < t <= t_switch
        stack.set_sparse(sparse_now)
        if sparse_now:
            refresh = (not have_masks) or since_refresh >= cfg.decay.refresh_period
            for layer in stack.layers:
                # SparseFFN.forward refreshes when its counter says so; drive it from here
                layer.steps_since_refresh = None if refresh else 0
            if refresh:
                old = [m.idx.clone() for _, m in stack.masks()] if have_masks else None
        x_np, y_np = task.next_batch()
        x = torch.from_numpy(x_np).to(dev, torch.float32)
        tgt = torch.from_numpy(np.asarray(y_np)).to(dev)
        if tgt.is_floating_point():
            tgt = tgt.float()
        for blk, layer in enumerate(stack.layers):
            layer.mvue = bool(cfg.mvue and sparse_now)
            layer.mvue_seed = layer_mvue_seed(cfg.seed, t, blk)
            layer.decay_lambda = lam if (sparse_now and lam > 0 and cfg.decay.mode is DecayMode.ON_GRADIENTS) else 0.0
        for p in stack.parameters():
            p.grad = None
        out = stack(x)
        if sparse_now and refresh:
            searches += 2 * cfg.depth
            new = [m.idx for _, m in stack.masks()]
            if old is not None:
                # flip_rate(mask_vec, new_vec) over the whole parameter vector (biases never flip)
                shape = lambda i: (4 * i.shape[0], 4 * i.shape[1])  # noqa: E731
                n = sum(mask_flips(TransposableMask(a, shape(a)), TransposableMask(b, shape(b))) for a, b in zip(old, new))
                flips[t - 1] = float(n) / stack.size
            have_masks = True
            since_refresh = 0
            if cfg.collect_block_stats:
                for blk, layer in enumerate(stack.layers):
                    for name, w in (("w_in", layer.w_in), ("w2", layer.w2)):
                        snapshots.setdefault(f"block{blk}.{name}", []).append(w.detach().clone())
        loss, dout = task.loss_and_grad(out, tgt)
        out.backward(dout.to(out.dtype))
        losses[t - 1] = loss.detach()
        mode = cfg.decay.mode if (sparse_now and lam > 0 and cfg.decay.mode is DecayMode.ON_WEIGHTS) else None
        masks = dict((id(w), m) for w, m in stack.masks()) if mode is not None else {}
        # when the next step is sparse and keeps its masks, the sparse weights' Adam updates also
        # write the next forward's compressed operands (s24_adam_compress): no K2 launch there
        fuse = (sparse_now and cfg.sparse and t_pre < t + 1 <= t_switch
                and since_refresh + 1 < cfg.decay.refresh_period)
        ops = {}
        if fuse:
            for layer in stack.layers:
                ops[id(layer.w_in)], ops[id(layer.w2)] = layer.op_in, layer.op_out
        for st, p in zip(states, stack.parameters()):
            st.lr = lr
            m = masks.get(id(p))
            dec = DecayConfig(lambda_w=lam, mode=DecayMode.ON_WEIGHTS) if m is not None else None
            adam_step(st, p.grad, m, dec, compress_into=ops.get(id(p)))
        for layer in stack.layers:
            layer.mark_weights_updated(compressed=fuse)  # adam_step writes p.data: version counters miss it
        since_refresh += 1
        if proxy is not None:
            pm = _proxy_masks(stack)
            searches += 2 * cfg.depth
            proxy[t - 1] = _flips_between(prev_proxy, pm, stack.size)
            prev_proxy = pm

    final_sparse = cfg.sparse and t_pre < T <= t_switch
    stack.set_sparse(final_sparse)
    stack.eval()
    for layer in stack.layers:
        layer.steps_since_refresh = 0  # evaluate with the current masks, no refresh
    ev = []
    with torch.no_grad():
        for xe, ye in task.eval_batches(cfg.eval_batches):
            oe = stack(torch.from_numpy(xe).to(dev, torch.float32))
            te = torch.from_numpy(np.asarray(ye)).to(dev)
            ev.append(float(task.loss_and_grad(oe, te.float() if te.is_floating_point() else te)[0]))
    final = [{k: getattr(layer, n).detach().double().cpu().numpy() for k, n in
              (("w_in", "w_in"), ("bias", "bias_in"), ("w2", "w2"))} for layer in stack.layers]
    rates = proxy if (not cfg.sparse and proxy is not None) else flips
    block_stats = None
    if cfg.collect_block_stats and snapshots:
        block_stats = [(name, block_flip_stats(snaps)) for name, snaps in snapshots.items() if len(snaps) >= 2]
    return RunArtifacts(cfg, losses.cpu().numpy().astype(np.float64), rates, final, float(np.mean(ev)), searches,
                        proxy, block_stats)


def make_warmup_runner(base_cfg: TrainConfig, warmup_steps: int, refresh_period: int = 1):
    """Warm-up handle of the decay-factor search (trainer.py:570-598): None runs the dense
    proxy (per-step flip instrumentation on a dense run), a float the sparse run with that
    ON_GRADIENTS decay factor, refreshing masks every `refresh_period` steps."""

    def runner(lam):
        common = dict(steps=warmup_steps, schedule_total_steps=base_cfg.steps, dense_ft_fraction=0.0,
                      dense_pretrain_fraction=0.0)
        if lam is None:
            cfg = dataclasses.replace(base_cfg, sparse=False, proxy_flips=True, **common)
        else:
            cfg = dataclasses.replace(base_cfg, sparse=True, proxy_flips=False,
                                      decay=DecayConfig(lam, DecayMode.ON_GRADIENTS, refresh_period), **common)
        return run_training(cfg).flips

    return runner
