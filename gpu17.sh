timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo rc=$?; tail -3 gpurun_out/bench4.err; python -c "
import json; d=json.load(open('gpurun_out/bench4.json')); print('value',d['value'],'frac',d['roofline']['frac'],'e2e',d['e2e'])"
