"""Build the sm_100a C-ABI library in-tree: paper_2404_01847_b200/libs24b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, one shared object,
no torch headers (the boundary is plain C).  Cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libs24b200.so")
SOURCES = ["s24_capi.cu", "s24_mask.cu", "s24_act.cu", "s24_gemm.cu", "s24_mvue.cu", "s24_optim.cu", "s24_greedy.cu", "s24_pack.cu", "s24_fp32.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2", "-shared", "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "sparse24_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build the library (default: in-tree LIB).  `out` + `defines` (e.g. ["S24_EPI_WARPS=8"])
    build a variant elsewhere for experiments; load it with S24_LIB_PATH."""
    lib = out or LIB
    if out is None and not defines and not force and not _stale():
        return LIB
    # one nvcc per translation unit in parallel (no cross-TU device symbols), then one link
    from concurrent.futures import ThreadPoolExecutor

    objdir = lib + ".objs"
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]

    def cc(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *cflags, *[f"-D{d}" for d in defines], "-c", "-o", obj, os.path.join(CSRC, src)]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        res = list(ex.map(cc, SOURCES))
    for _, r in res:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libs24b200.so")
        if verbose:
            sys.stderr.write(r.stderr)
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                        "-o", lib + ".tmp", *[o for o, _ in res]], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libs24b200.so")
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out = args[args.index("-o") + 1] if "-o" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, out=out, defines=defs))
