"""Aggregate ncu source-page warp-stall samples per CUDA source line.

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_n = hdr.index("Warp Stall Sampling (Not-issued Samples)")
per_line = collections.Counter()
per_line_ni = collections.Counter()
src = {}
cur = None
for r in rows[hdr_i + 1:]:
    if not r:
        continue
    if r[0]:
        cur = int(r[0]) if r[0].isdigit() else cur
        if r[0].isdigit():
            src[cur] = r[1]
    if len(r) > i_s and r[i_s].isdigit() and cur is not None:
        per_line[cur] += int(r[i_s])
        per_line_ni[cur] += int(r[i_n]) if r[i_n].isdigit() else 0
tot = sum(per_line.values())
print("total samples", tot)
for ln, v in per_line.most_common(top):
    print(f"{v:7d} {100 * v / max(tot, 1):5.1f}% (not-issued {per_line_ni[ln]:6d}) L{ln}: {src.get(ln, '').strip()[:110]}")
