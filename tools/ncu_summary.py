"""Summarise an ncu --set full report: per kernel, the metrics we judge by."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
keys = [
    ("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("gpc__cycles_elapsed.avg.per_second", "clk"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_on.avg.pct_of_peak_sustained_elapsed", "sp_ops%"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "dn_ops%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "lsu_smem%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit%"),
    ("launch__registers_per_thread", "regs"),
]
idx = [(hdr.index(k) if k in hdr else -1, n) for k, n in keys]
print(" | ".join(n for _, n in idx))
for r in rows[2:]:
    vals = []
    for i, n in idx:
        v = r[i] if i >= 0 else "NA"
        if n == "kernel":
            v = v.split("(")[0].replace("void ", "")[:44]
        vals.append(v)
    print(" | ".join(vals))
print("units:", {n: units[i] for i, n in idx if i >= 0})
