# A/B every variant in tools/variants over several configs (device value and backward per batch)
for i in 1 2; do for c in ${CONFIGS:-C1 C3 M1 C5}; do for f in tools/variants/*.so; do
  r=$(SKGE_B200_LIB=$PWD/$f timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'M/s', round(d['ms_per_step'],3), 'ms', 'fwd', round(d['roofline']['fwd_ms_per_batch']*1e3,1), 'bwd', round(d['roofline']['bwd_ms_per_batch']*1e3,1))")
  echo "$c $f $r"
done; done; done
