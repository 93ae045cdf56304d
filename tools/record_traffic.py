#!/usr/bin/env python
"""Records the DRAM traffic of one ncu-profiled sampling launch in profiles/traffic.json.

usage: python tools/record_traffic.py <workload key> <report.ncu-rep> <samples in the profiled launch> <profile name>

bench.py multiplies dram_bytes_per_sample by the samples of one of its launches to get roofline.traffic /
roofline.achieved; the entry is stamped with the hash of the kernel's sources so that a capture taken on an
older kernel is recognisable (roofline.traffic_matches_kernel)."""
import csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import kernel_source_hash

key, rep, samples, name = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
best = None
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "sample_kernel" not in d["Kernel Name"]:
        continue
    if best is None or float(d["gpu__time_duration.sum"].replace(",", "")) > float(best["gpu__time_duration.sum"].replace(",", "")):
        best = d
u = dict(zip(hdr, units))
def val(k):
    v = float(best[k].replace(",", ""))
    unit = u[k].lower()
    scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
             "s": 1, "second": 1, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1)
    return v * scale
total = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
p = os.path.join(ROOT, "profiles", "traffic.json")
d = json.load(open(p)) if os.path.exists(p) else {}
if "dram_bytes_per_sample" in d:  # round-1 layout (one unkeyed entry)
    d = {}
d[key] = {"dram_bytes_per_sample": total / samples, "samples_in_capture": samples, "kernel": best["Kernel Name"],
          "dram_bytes_read": val("dram__bytes_read.sum"), "dram_bytes_write": val("dram__bytes_write.sum"),
          "duration_s_under_ncu": val("gpu__time_duration.sum"), "profile": name,
          "kernel_src_sha16": kernel_source_hash()}
json.dump(d, open(p, "w"), indent=1)
print(json.dumps(d[key], indent=1))
