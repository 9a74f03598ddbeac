# e2e A/B: the in-tree engine vs each variant in tools/variants, alternating runs
for i in 1 2 3; do
  for f in in-tree tools/variants/*.so; do
    if [ "$f" = in-tree ]; then unset SKGE_B200_LIB; else export SKGE_B200_LIB=$PWD/$f; fi
    r=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1))")
    echo "$f $r"
  done
done
unset SKGE_B200_LIB
