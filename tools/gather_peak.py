"""Random-row gather bandwidth vs table size (L2-resident vs HBM-resident), the
denominator of roofline.l2_frac in bench.py. Usage: python tools/gather_peak.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_16949_b200 import Engine  # noqa: E402

eng = Engine(0)
out = {}
for mb in (8, 16, 32, 64, 96, 128, 256, 2560):
    for rf in (128, 256):
        g = eng.measure_gather(mb << 20, rf)
        out[f"{mb}MB_d{rf}"] = round(g, 1)
        print(f"table {mb:5d} MB rows {rf * 4:4d} B: {g:9.1f} GB/s", flush=True)
print(json.dumps(out))
