# C1 e2e under host-narrowing variants (thread count, int64 DMA), alternating runs
for i in 1 2 3; do
  for v in ${VARIANTS:-"SKG_SPEC_I64=0" "SKG_SPEC_I64=1" "SKG_NARROW_THREADS=8"}; do
    r=$(env $v timeout 300 python bench.py --config ${CFG:-C1} --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['e2e']['breakdown']; print(round(d['e2e']['value']/1e6,1), 'step', round(b['per_step_ms'],4), 'med', round(b['step_ms_median'],3), 'max', round(b['step_ms_max'],3), 'graph', round(b['graph_device_ms'],4), 'h2d', round(b['h2d_probe_gbs'] or 0,1), b['pcie_link'], d['e2e']['h2d_bytes_per_step'])")
    echo "[$v] $r"
  done
done
