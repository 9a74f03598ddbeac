# TransR iteration check: TransR/TransH GPU tests, C4 bench, phase trace
timeout 600 python -m pytest tests -x -q -m gpu -k "transr or ht or tc or shapes" 2>&1 | tail -4
bash tools/quick_bench.sh C4
timeout 120 python tools/transr_trace.py C4
