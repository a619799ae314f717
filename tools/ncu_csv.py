"""Print an ncu --csv metrics log as one row per launch: id, kernel, metric=value ..."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[h]
ki, mi, vi, ii = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
d = OrderedDict()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    d.setdefault((r[ii], r[ki].split('(')[0].replace('void ', '')[:48]), OrderedDict())[r[mi]] = r[vi]
for (i, k), v in d.items():
    print(i, k, " ".join(f"{m.split('.')[0].replace('__', ':')}={x}" for m, x in v.items()))
