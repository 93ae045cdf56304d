python tools/e2e_breakdown.py
