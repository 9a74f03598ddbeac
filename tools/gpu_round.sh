# Round check on one B200: GPU tests, smoke, one bench line per BASELINE config.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in C1 C2 C3 C4 C5; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 $( [ $c != C1 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for c in C1 C2 C3 C4 C5; do python -c "import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c',round(d['value']/1e6,1),'M/s e2e',round(d['e2e']['value']/1e6,1),'frac',r.get('frac'),'fwd',r.get('fwd_ms_per_batch'),'bwd',r.get('bwd_ms_per_batch'),'plan',r.get('plan_ms_per_epoch'))" || tail -5 gpurun_out/bench_$c.err; done
