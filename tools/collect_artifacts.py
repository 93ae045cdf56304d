#!/usr/bin/env python
"""Copies what tools/final_artifacts.sh left in gpurun_out/ into profiles/ under round-2 names (small text files
only; the .ncu-rep reports stay in gpurun_out/) and prints the numbers DESIGN.md quotes."""
import json, os, shutil, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
copies = {
    "fa_bench.json": "r02_final_bench.json", "fa_bench_reference.json": "r02_final_bench_reference.json",
    "fa_bench_strong.json": "r02_final_bench_with_strong_leg.json",
    "fa_bench_er10k.json": "r02_final_bench_config1_er10k.json", "fa_bench_grid2000.json": "r02_final_bench_config3_grid2000.json",
    "fa_bench_rmat24.json": "r02_final_bench_config4_rmat24.json", "fa_bench_rmat26.json": "r02_final_bench_config5_rmat26.json",
    "fa_launches_bench_steps2_warmup3.csv": "r02_final_launches_bench_steps2_warmup3.csv",
    "fa_configs.txt": "r02_final_configs.txt", "fa_fuzz_parity.txt": "r02_fuzz_parity.txt",
    "fa_fuzz_pipeline.txt": "r02_fuzz_pipeline.txt", "fa_overlap_timeline.txt": "r02_overlap_timeline_final.txt",
    "fa_traffic.json": "traffic.json",
}
for k in ("rmat20", "grid2000", "rmat24", "rmat26", "er10k"):
    copies[f"fa_ncu_summary_{k}.txt"] = f"r02_final_{k}_sample_kernel_ncu_summary.txt"
    copies[f"fa_ncu_details_{k}.txt"] = f"r02_final_{k}_sample_kernel_ncu_details.txt"
for src, dst in copies.items():
    a = os.path.join(G, src)
    if os.path.exists(a):
        if src == "fa_configs.txt":  # drop progress chatter
            open(os.path.join(P, dst), "w").write("".join(l for l in open(a) if not l.startswith("[")))
        else:
            shutil.copy(a, os.path.join(P, dst))
    else:
        print("missing", src)
for f in ("fa_bench", "fa_bench_er10k", "fa_bench_grid2000", "fa_bench_rmat24", "fa_bench_rmat26"):
    try:
        d = json.loads(open(os.path.join(G, f + ".json")).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable:", e); continue
    r, e, cb = d["roofline"], d["e2e"], d.get("cpu_baseline", {})
    print(f"{d['config']['workload']:40s} value {d['value']/1e6:8.3f} M/s  GTEPS {d['gteps_bfs']:6.1f}  roofline frac {r['frac']:.3f} "
          f"({'DRAM' if r.get('physical') else 'own counters'}; traffic/sample {0 if not r['traffic'] else r['traffic']/r['samples_per_launch']/1e3:.0f} KB) "
          f"alg {r['algorithmic_frac']:.2f} ({r['algorithmic_bytes_per_sample']/1e6:.2f} MB/sample)  e2e {e['value']/1e6:.3f} M/s in {e['time_to_stop_s']:.3f}s "
          f"(first {e['first_call_s']:.2f}s)  cpu {cb.get('value', 0):.0f}/s x{cb.get('cores')} ({cb.get('kind')}), 1 thread {cb.get('one_thread', {}).get('value', 0):.0f}/s")
