"""Per-region warp-stall breakdown of an `ncu --page source --csv --print-source sass` dump.
python tools/ncu_src_stalls.py dump.csv lo hi   (instruction index range, first copy)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
half = len(data) // 2 if len(data) > 1 and data[0][1] == data[len(data) // 2][1] else len(data)
lo, hi = int(sys.argv[2]), int(sys.argv[3])
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ie = hdr.index("Instructions Executed")
tot = {c: 0 for c in cols}
inst = 0
for r in data[lo:hi]:
    for c in cols:
        try:
            tot[c] += int(r[hdr.index(c)])
        except ValueError:
            pass
    try:
        inst += int(r[ie])
    except ValueError:
        pass
s = sum(tot.values())
print(f"region [{lo},{hi}) samples {s} warp-inst {inst}")
for c, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"  {c:24s} {v:6d} {100.0 * v / max(s, 1):5.1f}%")
