"""Break the e2e epoch (set_triples + set_negatives + train_epoch) into parts."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig
from paper_2502_16949_b200.engine import init_store, generate_synthetic

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
h, r, t = generate_synthetic(cfg["N"], cfg["R"], cfg["n_total"], 1)
eng = Engine(0)
mcfg = ModelConfig.make(cfg["model"], cfg["de"], cfg["dr"], cfg["norm"])
ent, rel, proj, nrm = init_store(cfg["model"], cfg["N"], cfg["R"], cfg["de"], cfg["dr"], 1)
eng.store_upload(mcfg, ent, rel, proj, nrm)
eng.set_triples(h, r, t, cfg["N"], cfg["R"])
nh, nt = eng.negative_sample(1)
tc = TrainConfig.make(lr=4e-4, margin=0.5, batch_size=cfg["B"], seed=1)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int64)).pin_memory().numpy()
hp, rp, tp, nhp, ntp = pin(h), pin(r), pin(t), pin(nh), pin(nt)
for e in range(5):
    eng.train_epoch(mcfg, tc, e, 4e-4)
ts = {"set_triples": [], "set_negatives": [], "train_epoch": [], "train_epoch_only": []}
ep = 5
for k in range(20):
    t0 = time.perf_counter(); eng.set_triples(hp, rp, tp, cfg["N"], cfg["R"]); t1 = time.perf_counter()
    eng.set_negatives(nhp, ntp); t2 = time.perf_counter()
    eng.train_epoch(mcfg, tc, ep, 4e-4); t3 = time.perf_counter(); ep += 1
    ts["set_triples"].append(t1 - t0); ts["set_negatives"].append(t2 - t1); ts["train_epoch"].append(t3 - t2)
for k in range(20):
    t0 = time.perf_counter(); eng.train_epoch(mcfg, tc, ep, 4e-4); ts["train_epoch_only"].append(time.perf_counter() - t0); ep += 1
for k, v in ts.items():
    print(k, "median ms %.3f  min %.3f" % (1e3 * np.median(v), 1e3 * np.min(v)))
x = torch.empty(len(h) * 3, dtype=torch.int64).pin_memory()
d = torch.empty_like(x, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print("torch pinned H2D GB/s %.1f" % (x.numel() * 8 * 10 / (time.perf_counter() - t0) / 1e9))
