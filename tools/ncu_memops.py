"""Per-launch DRAM throughput of memory-bound single-op stages from an ncu CSV launch list
(tools/ncu_ops.py under `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv`).

  python tools/ncu_memops.py gpurun_out/f4_ncu_memops_squeezenet_b128.csv [hbm_peak_gbs]
"""
import collections
import csv
import json
import os
import sys

path = sys.argv[1]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else None
if peak is None:
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        peak = float(json.load(open(mp))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        peak = 6553.6
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hdr = rows[hdr_i]
iid, ik, imn, imu, imv = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
launch = collections.OrderedDict()
for r in rows[hdr_i + 1:]:
    d = launch.setdefault(r[iid], {"kernel": r[ik]})
    v = float(r[imv].replace(",", ""))
    unit = r[imu]
    if r[imn] == "gpu__time_duration.sum":
        d["us"] = v / 1000.0 if unit in ("ns", "nsecond") else v * (1000.0 if unit in ("ms", "msecond") else 1.0)
    elif r[imn].startswith("dram__bytes"):
        scale = {"byte": 1, "B": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        d["bytes"] = d.get("bytes", 0.0) + v * scale
    elif r[imn].startswith("dram__throughput"):
        d["pct"] = v
print(f"HBM peak used: {peak:.1f} GB/s")
for k, d in launch.items():
    if "us" not in d:
        continue
    gbs = d.get("bytes", 0.0) / (d["us"] * 1e3)
    print(f"{k:>4} {d['kernel'][:34]:34s} {d['us']:9.2f} us {d.get('bytes', 0) / 1e6:9.2f} MB {gbs:8.1f} GB/s "
          f"({100 * gbs / peak:5.1f} % of measured peak; ncu dram__throughput {d.get('pct', float('nan')):.1f} %)")
