"""Per-kernel HBM traffic of one FFN step from an ncu --set full report (profiles/ evidence
for bench.py's roofline.traffic).

python tools/ncu_traffic.py <report.ncu-rep> <cfg> <out.json> [first_tag_index]

The report must hold consecutive GEMM launches of one step (tools/gpu_profile_round.sh
captures -k regex:gemm_kernel -s 6 -c 6, i.e. exactly the second step), in the engine's
launch order: fwd_in, fwd_out, bwd_out, bwd_in, dW2, dW_in (engine.ffn_forward/backward).
"""
import csv, json, subprocess, sys

ORDER = ["k3_spmm_fwd_in", "k3_spmm_fwd_out", "k4_spmm_bwd_out", "k4_spmm_bwd_in", "k5_gemm_dw2", "k5_gemm_dw_in"]
rep, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
first = int(sys.argv[4]) if len(sys.argv) > 4 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]


def col(name):
    return hdr.index(name)


scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}
res = {}
gemms = [r for r in rows[2:] if "gemm_kernel" in r[col("Kernel Name")]]
for i, r in enumerate(gemms):
    tag = ORDER[(first + i) % len(ORDER)]
    if tag in res:
        continue
    rd = float(r[col("dram__bytes_read.sum")]) * scale[units[col("dram__bytes_read.sum")]]
    wr = float(r[col("dram__bytes_write.sum")]) * scale[units[col("dram__bytes_write.sum")]]
    us = float(r[col("gpu__time_duration.sum")]) * scale[units[col("gpu__time_duration.sum")]]
    clk = r[col("gpc__cycles_elapsed.avg.per_second")]
    res[tag] = {"kernel": r[col("Kernel Name")].split("(")[0].replace("void ", ""), "us": us,
                "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                "gpc_ghz": float(clk) * (1e-9 if units[col("gpc__cycles_elapsed.avg.per_second")] == "hz" else 1.0)}
json.dump({"cfg": cfg, "report": rep.split("/")[-1], "kernels": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
