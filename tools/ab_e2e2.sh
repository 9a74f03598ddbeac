# e2e A/B across configs: the in-tree engine vs varlibs/old.so, alternating runs
for c in ${CONFIGS:-C1 C2}; do
for i in 1 2 3; do
  for f in in-tree varlibs/old.so; do
    if [ "$f" = in-tree ]; then unset SKGE_B200_LIB; else export SKGE_B200_LIB=$PWD/$f; fi
    r=$(timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['e2e']['breakdown']; print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), 'step', round(b['per_step_ms'],4), 'graph', round(b['graph_device_ms'],4), 'hits', b['spec_hits'])")
    echo "$c $f $r"
  done
done
done
unset SKGE_B200_LIB
