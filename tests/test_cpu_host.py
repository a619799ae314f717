"""CPU-only tests: the C-ABI library exports every declared symbol, the
host-side logic (pattern table, schedules, metadata tile layout model) and the
data-parallel gradient exchange (gloo, world_size 2) against the oracle."""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from oracle import s24_oracle as o

REPO = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(REPO, "include", "sparse24_b200.h")


def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+(s24_\w+)\(", text, re.M)))


def test_library_builds_and_exports_every_header_symbol():
    from paper_2404_01847_b200 import build

    lib = build.build()
    syms = _declared_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (s24_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # the ctypes binding types exactly the declared compute entry points
    from paper_2404_01847_b200 import _capi

    assert set(_capi.SIGNATURES) | {"s24_last_error_string", "s24_gemm_workspace_bytes"} == set(syms)
    lib_h = _capi.load()
    assert lib_h.s24_abi_version() == 2
    assert lib_h.s24_gemm_workspace_bytes() == _capi.GEMM_WORKSPACE_BYTES


def test_cuda_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2404_01847_b200 import transposable_search_conv

    with pytest.raises(RuntimeError):
        transposable_search_conv(torch.zeros(8, 8))


def test_product_pattern_table_matches_golden():
    from paper_2404_01847_b200 import enumerate_patterns

    t = enumerate_patterns()
    assert t.count == 90
    assert t.to_text() == open(os.path.join(REPO, "tests", "golden", "patterns.txt")).read()
    pats, pos = o.pattern_table()
    np.testing.assert_array_equal(t.patterns, pats)
    np.testing.assert_array_equal(t.positions, pos)


def test_generated_kernel_tables_match_pattern_table():
    import itertools

    hdr = open(os.path.join(REPO, "paper_2404_01847_b200", "csrc", "s24_patterns.h")).read()
    bits = [int(x, 16) for x in re.search(r"S24_PATTERN_BITS \{([^}]*)\}", hdr).group(1).split(",")]
    pats, _ = o.pattern_table()
    assert bits == [int(sum(int(b) << i for i, b in enumerate(p.reshape(16)))) for p in pats]


def _e_tile_model(meta: np.ndarray) -> np.ndarray:
    """Python model of the E-tile layout of include/sparse24_b200.h (the
    sm_100 sparse tensor-core metadata arrangement) from reference nibbles."""
    m, kq = meta.shape
    k = 4 * kq
    out = np.zeros((m // 128) * (k // 128) * 2048, dtype=np.uint8)
    for row in range(m):
        for grp in range(kq):
            tile = (row // 128) * (k // 128) + (4 * grp) // 128
            mm, kk = row % 128, (4 * grp) % 128
            lane = (mm % 8) + 8 * ((kk % 32) // 16) + 16 * (mm // 16)
            c, h, g = kk // 32, (mm // 8) % 2, (kk % 16) // 4
            byte = tile * 2048 + lane * 16 + c * 4 + h * 2 + (g // 2)
            out[byte] |= int(meta[row, grp]) << (4 * (g % 2))
    return out


def test_e_tile_layout_model_roundtrip():
    """The layout is a bijection: every (row, group) nibble has its own slot."""
    rng = np.random.default_rng(0)
    w = rng.standard_normal((256, 256))
    bits = o.transposable_search_conv(w)
    _, meta = o.compress_rowwise(w, bits)
    e = _e_tile_model(meta)
    back = np.zeros_like(meta)
    for row in range(256):
        for grp in range(64):
            tile = (row // 128) * 2 + (4 * grp) // 128
            mm, kk = row % 128, (4 * grp) % 128
            lane = (mm % 8) + 8 * ((kk % 32) // 16) + 16 * (mm // 16)
            byte = tile * 2048 + lane * 16 + (kk // 32) * 4 + ((mm // 8) % 2) * 2 + ((kk % 16) // 4) // 2
            back[row, grp] = (e[byte] >> (4 * (((kk % 16) // 4) % 2))) & 0xF
    np.testing.assert_array_equal(back, meta)


def test_schedule_and_config_semantics():
    from paper_2404_01847_b200.optim import DecayConfig
    from paper_2404_01847_b200 import dp

    assert o.switch_step(60000, 1 / 6) == 50000  # test_trainer.py:68-71
    with pytest.raises(ValueError):
        DecayConfig(lambda_w=-1)
    with pytest.raises(ValueError):
        DecayConfig(refresh_period=0)
    assert DecayConfig().refresh_period == 40
    shards = [dp.shard_rows(10, r, 3) for r in range(3)]
    assert [s.stop - s.start for s in shards] == [4, 3, 3] and shards[-1].stop == 10
    assert dp.decay_share(6e-5, 4) == pytest.approx(1.5e-5)


def _dp_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2404_01847_b200 import dp

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    d, d_ff, n, lam = 16, 32, 24, 0.05
    w_in = rng.standard_normal((d_ff, d)) / 4
    w2 = rng.standard_normal((d, d_ff)) / 4
    b = rng.standard_normal(d_ff) / 8
    x = rng.standard_normal((n, d))
    dy = rng.standard_normal((n, d)) / 8
    layer = o.Layer(w_in, b, w2, "gelu")
    mi, mo = o.transposable_search_conv(w_in), o.transposable_search_conv(w2)
    sl = dp.shard_rows(n, rank, world)
    f = o.fst_forward(layer, x[sl], mi, mo, exact=False)
    g = o.fst_backward(layer, f, dy[sl], mi, mo, exact=False)
    share = dp.decay_share(lam, world)
    bucket = dp.GradBucket([w_in.shape, (d_ff,), w2.shape], "cpu")
    bucket.views[0].copy_(torch.from_numpy(o.masked_decay_gradient(g["dw_in"], w_in, mi, share)))
    bucket.views[1].copy_(torch.from_numpy(g["dbias_in"]))
    bucket.views[2].copy_(torch.from_numpy(o.masked_decay_gradient(g["dw2"], w2, mo, share)))
    bucket.allreduce()
    if rank == 0:
        fr = o.fst_forward(layer, x, mi, mo, exact=False)
        gr = o.fst_backward(layer, fr, dy, mi, mo, exact=False)
        ref = [o.masked_decay_gradient(gr["dw_in"], w_in, mi, lam), gr["dbias_in"],
               o.masked_decay_gradient(gr["dw2"], w2, mo, lam)]
        errs = [float(np.abs(v.numpy() - r).max()) for v, r in zip(bucket.views, ref)]
        q.put(errs)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_data_parallel_gradient_exchange_gloo(world):
    """Linearity oracle: sum over ranks of shard gradients (decay pre-scaled by
    1/world) == full-batch gradient with the decay applied once."""
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    errs = q.get(timeout=120)
    for p in ps:
        p.join(60)
    assert all(p.exitcode == 0 for p in ps)
    assert max(errs) < 1e-5, errs


def test_bench_reference_arm_line():
    """`bench.py --impl reference` (the reference's own CPU path on the host cores) prints the
    contract's JSON line: same metric / unit / workload as our arm, impl, cpu_baseline, e2e."""
    import json

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-tokens", "8"], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "tokens/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["metric"].startswith("2:4 FFN fwd+bwd tokens/s")
    assert "BASELINE.json configs[3]" in line["config"]["workload"]  # the default headline: C4
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"] and cb["value"] == line["value"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_mvue_certificate_bound_below_margin():
    """The certified exact-MVUE kernel decides c_j <= draw in fp32 only with a 2^-14 (1024 ulp(1))
    margin; the worst-case error propagated through the reference's greedy pair fill must stay
    below it (tools/mvue_bound.py, the kernel's constant kMargin)."""
    import importlib.util

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("mvue_bound", os.path.join(root, "tools", "mvue_bound.py"))
    mb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mb)
    assert mb.bound(2.0) < 1024
    src = open(os.path.join(root, "paper_2404_01847_b200", "csrc", "s24_mvue.cu")).read()
    assert "kMargin = 6.103515625e-5f" in src  # 2^-14
