import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig
from paper_2502_16949_b200.engine import generate_synthetic, init_store
c = bench.CONFIGS[sys.argv[1]]
h, r, t = generate_synthetic(c["N"], c["R"], c["n_total"], bench.SEED)
eng = Engine(0)
cfg = ModelConfig.make(c["model"], c["de"], c["dr"], c["norm"])
eng.store_upload(cfg, *init_store(c["model"], c["N"], c["R"], c["de"], c["dr"], bench.SEED))
eng.set_triples(h, r, t, c["N"], c["R"])
nh, nt = eng.negative_sample(bench.SEED)
tc = TrainConfig.make(lr=bench.LR, margin=bench.MARGIN, batch_size=c["B"], seed=bench.SEED)
for w in range(3): eng.train_epoch(cfg, tc, w, bench.LR)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int64)).pin_memory().numpy()
hp, rp, tp, nhp, ntp = pin(h), pin(r), pin(t), pin(nh), pin(nt)
eng.set_deferred_uploads(True)
for k in range(12):
    ta = time.perf_counter()
    eng.set_triples(hp, rp, tp, c["N"], c["R"]); eng.set_negatives(nhp, ntp)
    tb = time.perf_counter()
    rep = eng.train_epoch(cfg, tc, 10 + k, bench.LR)
    tcx = time.perf_counter()
    print(f"set {1e3*(tb-ta):.3f} ms call {1e3*(tcx-tb):.3f} ms graph {1e3*(rep.t_forward_s+rep.t_backward_s):.3f}", file=sys.stderr)
