#!/bin/bash
# Round-2 artifacts, taken on one B200 with the kernel as committed (run under gpurun; results land in gpurun_out/fa_*
# and are copied into profiles/ by tools/collect_artifacts.py here).  Every number judged comes from this script:
#   bench lines (own arm + reference arm) for the default workload and for configs 1, 3, 4, 5;
#   the ncu launch list of the default bench command; ncu --set full of one bench-sized sampling launch of configs
#   1 to 5 (the DRAM bytes per sample behind roofline.traffic); all five configs end to end; the fuzz sweeps.
set -x
O=gpurun_out
R=/tmp/fa_ncu_reports; mkdir -p $R
python bench.py --impl reference --steps 2 --warmup 1 > $O/fa_bench_reference.json 2> $O/fa_bench_reference.err
# DRAM traffic of bench-sized launches first: bench.py reads profiles/traffic.json
# (third field: sampling launches before the measured one -- warm-up main + re-run pass; config 1 has no re-run pass)
for spec in "rmat20 524288 2" "grid2000 32768 2" "rmat24 262144 2" "rmat26 131072 2" "er10k 1048576 1"; do
  set -- $spec
  python tools/prof_launch.py $1 $2 > $O/fa_plain_$1.log 2>&1 || exit 1      # exits 0 without ncu first; launches: warm-up main + re-run pass, then the measured main (+ re-run) pass
  ncu --set full --import-source on --clock-control none -k regex:sample_kernel --launch-skip $3 --launch-count 2 \
      -o $R/fa_ncu_$1 -f python tools/prof_launch.py $1 $2 > $O/fa_ncu_$1.log 2>&1
  python tools/record_traffic.py $1 $R/fa_ncu_$1.ncu-rep $2 r02_final_$1 > $O/fa_traffic_$1.log 2>&1
  python tools/ncu_summary.py $R/fa_ncu_$1.ncu-rep > $O/fa_ncu_summary_$1.txt 2>&1
  ncu -i $R/fa_ncu_$1.ncu-rep --page details > $O/fa_ncu_details_$1.txt 2>/dev/null
done
cp $R/fa_ncu_rmat20.ncu-rep $O/   # (gpurun brings back at most 64 MiB: one report for line-level work, not five)
cp profiles/traffic.json $O/fa_traffic.json
python bench.py > $O/fa_bench.json 2> $O/fa_bench.err
python bench.py --strong > $O/fa_bench_strong.json 2> $O/fa_bench_strong.err
for w in er10k grid2000 rmat24; do
  python bench.py --workload $w > $O/fa_bench_$w.json 2> $O/fa_bench_$w.err
done
python bench.py --workload rmat26 --steps 3 --warmup 3 > $O/fa_bench_rmat26.json 2> $O/fa_bench_rmat26.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/fa_plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/fa_launches_bench_steps2_warmup3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/fa_ncu_launches.log 2>&1
python tools/run_configs.py 1 2 3 4 5 > $O/fa_configs.txt 2>&1
python tools/fuzz_parity.py 3000 101 > $O/fa_fuzz_parity.txt 2>&1
python tools/fuzz_pipeline.py 400 7 > $O/fa_fuzz_pipeline.txt 2>&1
python tools/overlap_timeline.py rmat20 262144 2>&1 | grep -v "^\[bench\]" > $O/fa_overlap_timeline.txt
