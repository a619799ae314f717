"""One-line summary of bench.py JSON lines: python tools/bench_summary.py file.json [...]"""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unparsable", e)
        continue
    ks = {k: round(v["ms_per_launch"] * 1e3, 1) for k, v in (d.get("kernels") or {}).items()}
    print(p.split("/")[-1], f"{d['value']:.4g} tok/s {d['ms_per_step']:.4f} ms", "best_dense x%.3f" % (d.get("speedup_vs_best_dense") or 0),
          "eager x%.3f" % (d.get("speedup_vs_dense") or 0), "clk", (d.get("clocks") or {}).get("sm_mhz"), ks)
    for sn, sl in (d.get("sub_lines") or {}).items():
        print("   sub", sn, f"{sl['value']:.4g} tok/s {sl['ms_per_step']:.4f} ms best_dense x{sl.get('speedup_vs_best_dense', 0):.3f}")
