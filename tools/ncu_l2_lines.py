#!/usr/bin/env python
"""L2 sector requests (global and local) of a kernel per CUDA source line, from the source page of an ncu report.
usage: tools/ncu_l2_lines.py report.ncu-rep object-or-lib kernel_mangled_name [top]"""
import csv, re, subprocess, sys, os, tempfile, collections
rep, so, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
dis = start = None
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    if kern.encode() not in open(os.path.join(tmp, cub), "rb").read():
        continue
    d = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.splitlines()
    st = next((i for i, l in enumerate(d) if l.strip().startswith(".section") and (".text." + kern) in l), None)
    if st is not None:
        dis, start = d, st
        break
assert dis is not None
line_of, cur = {}, None
for l in dis[start + 1:]:
    if l.strip().startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", l)
    if m:
        line_of[int(m.group(1), 16)] = (cur, m.group(2).split()[0])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; ci = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
num = lambda x: float(x) if x not in ("", "-") else 0.0
base = int(data[0][ci["Address"]], 16) if data[0][ci["Address"]].startswith("0x") else int(data[0][ci["Address"]])
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0.0])
for r in data:
    a = r[ci["Address"]]; a = int(a, 16) if a.startswith("0x") else int(a)
    key, op = line_of.get(a - base, (("?", 0), "?"))
    k = (key, op.split(".")[0])
    agg[k][0] += num(r[ci["L2 Theoretical Sectors Global"]])
    agg[k][1] += num(r[ci["L2 Theoretical Sectors Local"]])
    agg[k][2] += num(r[ci["L1 Wavefronts Shared"]])
    agg[k][3] += num(r[ci["L1 Tag Requests Global"]])
    agg[k][4] += num(r[ci["Instructions Executed"]])
tg = sum(v[0] for v in agg.values()); tl = sum(v[1] for v in agg.values()); tsw = sum(v[2] for v in agg.values())
print(f"L2 theoretical sectors: global {tg:.3g}, local {tl:.3g}; shared wavefronts {tsw:.3g}")
src = open("paper_1910_11039_b200/csrc/sampler_kernels.cuh").read().splitlines()
print("--- by L2 sectors (global + local)")
for (key, op), v in sorted(agg.items(), key=lambda x: -(x[1][0] + x[1][1]))[:top]:
    f, ln = key
    text = src[ln - 1].strip()[:80] if f == "sampler_kernels.cuh" and 0 < ln <= len(src) else ""
    print(f"{100*(v[0]+v[1])/(tg+tl):5.1f}%  glob {v[0]:11.0f} loc {v[1]:10.0f} tagreq {v[3]:10.0f} {op:8s} {f}:{ln}: {text}")
print("--- by shared wavefronts")
for (key, op), v in sorted(agg.items(), key=lambda x: -x[1][2])[:top // 2]:
    f, ln = key
    text = src[ln - 1].strip()[:80] if f == "sampler_kernels.cuh" and 0 < ln <= len(src) else ""
    print(f"{100*v[2]/max(tsw,1):5.1f}%  wavefronts {v[2]:11.0f} inst {v[4]:10.0f} {op:8s} {f}:{ln}: {text}")
