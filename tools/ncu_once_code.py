#!/usr/bin/env python
"""Code a warp executes about once per sample (between LO and HI times), by source function and line: where the
instruction-fetch stalls of a kernel whose CTAs all sit in different phases come from.
usage: tools/ncu_once_code.py report.ncu-rep object kernel warp_samples [lo hi]"""
import csv, re, subprocess, sys, os, tempfile, collections, bisect
rep, so, kern, N = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
lo, hi = (float(sys.argv[5]), float(sys.argv[6])) if len(sys.argv) > 6 else (0.5, 4.0)
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
line_of, cur = {}, None
for l in dis[start + 1:]:
    if l.strip().startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
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
num = lambda x: float(x) if x not in ("", "-") else 0.0
base = int(data[0][ci["Address"]], 16) if data[0][ci["Address"]].startswith("0x") else int(data[0][ci["Address"]])
src = open("paper_1910_11039_b200/csrc/sampler_kernels.cuh").read().splitlines()
heads = []
for i, l in enumerate(src):
    m = re.match(r"(?:static )?__device__ .*?(\w+)\(", l) or re.match(r"__global__ .* (sample_kernel)\(", l)
    if m and not l.startswith(" "):
        heads.append((i + 1, m.group(1)))
def fn(key):
    if key is None: return "?"
    f, ln = key
    if f != "sampler_kernels.cuh": return f
    j = bisect.bisect_right([h[0] for h in heads], ln) - 1
    return heads[j][1] if j >= 0 else "?"
byfn = collections.defaultdict(lambda: [0, 0.0, 0.0]); byline = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in data:
    a = r[ci["Address"]]; a = int(a, 16) if a.startswith("0x") else int(a)
    e = num(r[ci["Instructions Executed"]]) / N
    if not (lo <= e < hi): continue
    key = line_of.get(a - base)
    for tab, k in ((byfn, fn(key)), (byline, key)):
        tab[k][0] += 1; tab[k][1] += num(r[ci["stall_no_inst"]]); tab[k][2] += num(r[ci["# Samples"]])
tot = sum(v[0] for v in byfn.values())
print(f"{tot} SASS instructions ({tot*16/1024:.1f} KB) executed between {lo} and {hi} times per warp and sample")
for k, v in sorted(byfn.items(), key=lambda x: -x[1][0])[:25]:
    print(f"  {v[0]:5d} instr  no-inst stall samples {v[1]:8.0f}  all {v[2]:8.0f}  {k}")
print("--- lines")
for k, v in sorted(byline.items(), key=lambda x: -x[1][0])[:40]:
    f, ln = k if k else ("?", 0)
    text = src[ln - 1].strip()[:90] if f == "sampler_kernels.cuh" and 0 < ln <= len(src) else ""
    print(f"  {v[0]:5d} instr  {f}:{ln}: {text}")
