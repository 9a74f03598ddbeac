#!/bin/bash
# A/B: run the C1 bench against each engine variant in tools/variants
for f in tools/variants/*.so; do
  r=$(SKGE_B200_LIB=$PWD/$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'M/s', round(d['ms_per_step'],3), 'ms', 'fwd', round(d['roofline']['fwd_ms_per_batch']*1e3,1), 'bwd', round(d['roofline']['bwd_ms_per_batch']*1e3,1))")
  echo "$f $r"
done
