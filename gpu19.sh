python bench.py --steps 5 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo rc=$?; grep "e2e run" gpurun_out/bench5.err
