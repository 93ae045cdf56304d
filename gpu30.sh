timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 5 --warmup 3 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo rc=$?; tail -2 gpurun_out/bench6.err; python -c "
import json; d=json.load(open('gpurun_out/bench6.json')); print('value',d['value'],'frac',d['roofline']['frac'],'ms/step',d['ms_per_step'],'kernel ms',d['roofline']['kernel_ms_per_step']); print(d['e2e']['value'], d['e2e']['time_to_stop_s'], d['e2e']['phases_s'])"
python tools/run_configs.py 1 3 2>&1 | grep -E "run 1|sustained"
