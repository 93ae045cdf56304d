python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo rc=$?; tail -4 gpurun_out/bench_r01.err
python bench.py --steps 2 --warmup 3 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
python tools/prof_epochs.py 32768 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 2 -c 1 -o gpurun_out/prof_v5 python tools/prof_epochs.py 32768 > gpurun_out/ncu5.log 2>&1
tail -2 gpurun_out/ncu5.log
