timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -5
EBC_BITMAP=1 timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -5
EBC_BITMAP=0 python tools/sweep_c2.py "128,4,0"
python tools/sweep_c2.py "128,4,0;64,4,0;128,2,0;256,4,0;256,2,0;64,2,0"
