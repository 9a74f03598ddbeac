# quick multi-config bench summary (no CPU baseline); usage: bash tools/quick_bench.sh C1 C2 ...
for c in "$@"; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/qb_$c.json 2> gpurun_out/qb_$c.err
  python - $c <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/qb_{c}.json").read().strip().splitlines()[-1]); r=d["roofline"]
    print(c, f"{d['value']/1e6:.1f}M/s e2e {d['e2e']['value']/1e6:.1f} ms/ep {d['ms_per_step']:.3f} fwd {r['fwd_ms_per_batch']*1e3:.1f}us bwd {r['bwd_ms_per_batch']*1e3:.1f}us plan {r['plan_ms_per_epoch']:.3f}ms shuffle {r.get('shuffle_ms_per_epoch',0):.3f}ms loss {d['final_loss']:.7f}")
except Exception as e:
    print(c, "FAILED", e, open(f"gpurun_out/qb_{c}.err").read()[-500:])
PY
done
