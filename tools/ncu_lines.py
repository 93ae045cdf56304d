#!/usr/bin/env python
"""Attributes ncu warp-stall samples of a kernel to CUDA source lines.
usage: tools/ncu_lines.py report.ncu-rep lib.so kernel_mangled_name [top]"""
import csv, re, subprocess, sys, os, tempfile, collections
rep, so, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4].isdigit() else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
# locate the cubin and text section that hold the kernel (one cubin per translation unit)
dis, start = None, None
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    if kern.encode() not in open(os.path.join(tmp, cub), "rb").read():
        continue
    d = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.splitlines()
    st = next((i for i, l in enumerate(d) if l.strip().startswith(".section") and (".text." + kern) in l), None)
    if st is not None:
        dis, start = d, st
        break
assert dis is not None, "kernel not found in any cubin of " + so
line_of = {}
cur = None
for l in dis[start + 1:]:
    if l.strip().startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; ci = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
for k, r in enumerate(data): # (a report with several launches: the first one's table)
    if not r or r[0] in ("Kernel Name", "Address"):
        data = data[:k]; break
base = int(data[0][ci["Address"]], 16) if data[0][ci["Address"]].startswith("0x") else int(data[0][ci["Address"]])
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0.0])
sort_col = 4 if "--noinst" in sys.argv else 3 if "--byinst" in sys.argv else 0
tot = 0.0
for r in data:
    a = r[ci["Address"]]; a = int(a, 16) if a.startswith("0x") else int(a)
    key = line_of.get(a - base, ("?", 0))
    s = float(r[ci["# Samples"]] or 0); tot += s
    agg[key][0] += s
    agg[key][1] += float(r[ci["stall_long_sb"]] or 0)
    agg[key][2] += float(r[ci["stall_barrier"]] or 0)
    agg[key][3] += float(r[ci["Instructions Executed"]] or 0)
    agg[key][4] += float(r[ci["stall_no_inst"]] or 0)
src = {}
for (f, ln) in agg:
    if f != "?" and f not in src:
        for root in ("paper_1910_11039_b200/csrc", "."):
            p = os.path.join(root, f)
            if os.path.exists(p):
                src[f] = open(p).read().splitlines(); break
print(f"total samples {tot:.0f}")
for (f, ln), v in sorted(agg.items(), key=lambda x: -x[1][sort_col])[:top]:
    text = src.get(f, [""] * (ln + 1))[ln - 1].strip()[:90] if f in src and ln - 1 < len(src[f]) else ""
    print(f"{100*v[0]/tot:5.1f}%  long_sb {100*v[1]/max(v[0],1):3.0f}% bar {100*v[2]/max(v[0],1):3.0f}% noinst {100*v[4]/max(v[0],1):3.0f}%  inst {v[3]:11.0f}  {f}:{ln}: {text}")
