#!/usr/bin/env python
"""SASS instruction count of a kernel per CUDA source line / per source function (code-size attribution).
usage: tools/sass_lines.py lib.so kernel_mangled_name [top]"""
import re, subprocess, sys, os, tempfile, collections
so, kern = sys.argv[1:3]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
dis, start = None, None  # (pass the object file of the kernel's translation unit: build/obj/sample_launch_b<BLOCK>.*.o)
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    if kern.encode() not in open(os.path.join(tmp, cub), "rb").read():
        continue
    d = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.splitlines()
    st = next((i for i, l in enumerate(d) if l.strip().startswith(".section") and (".text." + kern) in l), None)
    if st is not None:
        dis, start = d, st
        break
per_line = collections.Counter(); cur = None; total = 0
for l in dis[start + 1:]:
    if l.strip().startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    if re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", l):
        per_line[cur] += 1; total += 1
print("total SASS instructions", total, "=", total * 16 // 1024, "KB")
# function ranges of sampler_kernels.cuh
src = open("paper_1910_11039_b200/csrc/sampler_kernels.cuh").read().splitlines()
heads = []
for i, t in enumerate(src, 1):
    m = re.match(r"^(?:__device__|__global__|template).*?\b(\w+)\s*\(", t)
    if t.startswith("__device__") or t.startswith("__global__"):
        m = re.search(r"\b(\w+)\s*\(", t[t.find(" "):])
        if m: heads.append((i, m.group(1)))
per_fn = collections.Counter()
for (f, ln), c in per_line.items():
    if f == "sampler_kernels.cuh":
        name = "?"
        for (h, nm) in heads:
            if h <= ln: name = nm
        per_fn[name] += c
    else:
        per_fn[f] += c
for k, v in per_fn.most_common(top):
    print(f"{v:7d} {100*v/total:5.1f}%  {k}")
print("--- top lines")
for (k, v) in per_line.most_common(top):
    t = src[k[1] - 1].strip()[:80] if k and k[0] == "sampler_kernels.cuh" and k[1] <= len(src) else ""
    print(f"{v:6d}  {k}: {t}")
