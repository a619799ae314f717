"""Per-kernel HBM traffic of one FFN step from an ncu --set full report (profiles/ evidence
for bench.py's roofline.traffic).

python tools/ncu_traffic.py <report.ncu-rep> <cfg> <out.json>

The report must hold the six GEMM launches of one step (tools/gpu_profile_round.sh
captures -k regex:gemm_kernel -s 6 -c 6, i.e. exactly the second step).
"""
import csv, json, subprocess, sys



def classify(names):
    """Tag the six GEMMs of one step by template signature: dense = dW (dW2 first, then
    dW_in), sparse epilogue 3/5 = fwd_in (GELU / gated forward), 4/6 = bwd_out (dGELU /
    dgated), plain-store sparse GEMMs = fwd_out before bwd_out, bwd_in after it."""
    tags, dense_seen, bwd_seen = [], 0, False
    for nm in names:
        args = [a.strip() for a in nm.split("<", 1)[1].split(">", 1)[0].split(",")]
        sparse, epi = args[0] in ("1", "true"), int(args[6])
        if not sparse:
            tags.append("k5_gemm_dw2" if dense_seen == 0 else "k5_gemm_dw_in")
            dense_seen += 1
        elif epi in (3, 5):
            tags.append("k3_spmm_fwd_in")
        elif epi in (4, 6):
            tags.append("k4_spmm_bwd_out")
            bwd_seen = True
        else:
            tags.append("k4_spmm_bwd_in" if bwd_seen else "k3_spmm_fwd_out")
    return tags


rep, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]


def col(name):
    return hdr.index(name)


scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}
res = {}
gemms = [r for r in rows[2:] if "gemm_kernel" in r[col("Kernel Name")]]
for tag, r in zip(classify([r[col("Kernel Name")] for r in gemms]), gemms):
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
