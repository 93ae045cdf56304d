python tools/run_configs.py 2 2>&1 | grep -E "run 1|sustained"
timeout 1300 python tools/run_configs.py 4 2>&1 | grep -E "config|run 1|sustained"
