python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$?; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
python tools/prof_epochs.py 16384 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 2 -c 1 -o gpurun_out/prof_v3 python tools/prof_epochs.py 16384 > gpurun_out/ncu3.log 2>&1
tail -2 gpurun_out/ncu3.log
