timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo rc=$?; tail -3 gpurun_out/bench3.err; cat gpurun_out/bench3.json
