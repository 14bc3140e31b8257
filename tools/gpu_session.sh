timeout 900 python tools/prof_overhead.py
