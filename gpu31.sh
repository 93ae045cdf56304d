timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -4
python tools/sweep_c2.py "128,4,0" 400000
timeout 1300 python tools/run_configs.py 4 2>&1 | grep -E "config|run 1|sustained"
