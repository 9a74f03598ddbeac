#!/bin/bash
# A/B of engine variants in varlibs/ on one config: bash tools/ab_cfg.sh C2 [steps]
c=${1:-C1}; n=${2:-10}
for f in varlibs/*.so; do
  r=$(SKGE_B200_LIB=$PWD/$f timeout 300 python bench.py --config $c --steps $n --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e6,1), 'M/s', round(d['ms_per_step'],3), 'ms', 'fwd', round(r['fwd_ms_per_batch']*1e3,1), 'bwd', round(r['bwd_ms_per_batch']*1e3,1), 'plan', round(r['plan_ms_per_epoch'],3), 'loss', d['final_loss'])")
  echo "$c $(basename $f .so) $r"
done
