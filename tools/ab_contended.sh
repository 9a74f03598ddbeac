# C1 e2e of the upload variants with and without background CPU load (LOAD busy processes)
run() { for v in "SKG_SPEC_NO16=0" "SKG_SPEC_NO16=1" "SKG_NARROW_THREADS=8"; do
    r=$(env $v timeout 300 python bench.py --config ${CFG:-C1} --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['e2e']['breakdown']; print(round(d['e2e']['value']/1e6,1), 'step', round(b['per_step_ms'],4), 'med', round(b['step_ms_median'],3), 'max', round(b['step_ms_max'],3), 'graph', round(b['graph_device_ms'],4), d['e2e']['h2d_bytes_per_step'])")
    echo "load=$1 [$v] $r"; done; }
run 0; run 0
pids=""; for k in $(seq 1 ${LOAD:-4}); do (while :; do :; done) & pids="$pids $!"; done
run ${LOAD:-4}
kill $pids
