"""One-kernel brief from `ncu -i rep --page raw --csv` output: time, clock, issue / warp activity,
instructions, DRAM bytes, pipe utilisation and the top warp-stall reasons (per issue).
python tools/ncu_kernel_brief.py raw.csv [algorithmic_bytes]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))

    def g(k, scale=1.0):
        try:
            return float(d[k]) * scale
        except (KeyError, ValueError):
            return float("nan")

    t_us = g("gpu__time_duration.sum") * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u.get("gpu__time_duration.sum"), 1.0)
    gb = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
    rd = g("dram__bytes_read.sum") * gb.get(u.get("dram__bytes_read.sum"), 1.0)
    wr = g("dram__bytes_write.sum") * gb.get(u.get("dram__bytes_write.sum"), 1.0)
    print(f"{d['Kernel Name'][:70]}")
    print(f"  {t_us:.1f} us at {g('sm__cycles_elapsed.avg.per_second'):.3f} GHz, grid {d.get('launch__grid_size')} x "
          f"{d.get('launch__block_size')} thr, {d.get('launch__registers_per_thread')} regs")
    if alg:
        print(f"  algorithmic {alg / 1e9:.3f} GB -> {alg / (t_us * 1e-6) / 1e9:.0f} GB/s")
    print(f"  DRAM read {rd:.3f} GB + write {wr:.3f} GB; dram% {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}")
    print(f"  issue active {g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}%, warps active "
          f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%, warp-inst {g('smsp__inst_executed.sum') / 1e6:.1f} M")
    print(f"  pipes: alu {g('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%, fma "
          f"{g('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%, fp64 "
          f"{g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%, lsu "
          f"{g('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active'):.1f}%")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("  stalls per issue: " + ", ".join(f"{n} {v:.2f}" for v, n in st[:7] if n != "selected"))
