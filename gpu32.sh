timeout 1500 python -m pytest tests/test_gpu_stopping_pipeline.py tests/test_gpu_full_size.py -x -q 2>&1 | tail -4
python tools/e2e_breakdown.py 2>&1 | tail -3
python tools/run_configs.py 3 2>&1 | grep "run 1"
