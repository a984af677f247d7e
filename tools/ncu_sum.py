"""Summarise an ncu CSV launch list (gpu__time_duration / dram bytes per kernel launch)."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hdr = rows[hdr_i]
iid, ik, im, iv = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iu = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
SCALE = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
per = collections.defaultdict(dict)
names = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= iv:
        continue
    scale = SCALE.get(r[iu], 1.0) if iu is not None else 1.0
    per[r[iid]][r[im]] = float(r[iv].replace(",", "")) * scale
    names[r[iid]] = r[ik]
tot = collections.Counter()
by_kernel = collections.defaultdict(lambda: [0, 0.0, 0.0])
for k, m in per.items():
    name = names[k].split("(")[0]
    t = m.get("gpu__time_duration.sum", 0.0)
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot["time_ns"] += t
    tot["bytes"] += b
    by_kernel[name][0] += 1
    by_kernel[name][1] += t
    by_kernel[name][2] += b
print(json.dumps({"launches": len(per), "sum_gpu_time_us": tot["time_ns"] / 1e3, "dram_bytes": tot["bytes"],
                  "kernels": {k: {"launches": v[0], "time_us": v[1] / 1e3, "dram_bytes": v[2]} for k, v in by_kernel.items()}},
                 indent=1))
