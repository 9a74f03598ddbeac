set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in C1 C2 C3 C4 C5; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 $( [ $c != C1 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2
for c in C1 C2 C3 C4 C5; do python -c "import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]);print('$c',round(d['value']/1e6,1),'M/s e2e',round(d['e2e']['value']/1e6,1),'fwd',d['roofline']['forward_gbs'],'bwd',d['roofline']['backward_gbs'], d['roofline'].get('fwd_ms_per_batch'), d['roofline'].get('bwd_ms_per_batch'))"; done
