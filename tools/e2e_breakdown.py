"""Where the end-to-end step time goes (bench.py's e2e loop, split per call).

  python tools/e2e_breakdown.py [--config C1] [--steps 20]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    import torch
    from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig
    from paper_2502_16949_b200.engine import generate_synthetic, init_store
    h, r, t = generate_synthetic(c["N"], c["R"], c["n_total"], bench.SEED)
    M = len(h)
    eng = Engine(0)
    cfg = ModelConfig.make(c["model"], c["de"], c["dr"], c["norm"])
    eng.store_upload(cfg, *init_store(c["model"], c["N"], c["R"], c["de"], c["dr"], bench.SEED))
    eng.set_triples(h, r, t, c["N"], c["R"])
    nh, nt = eng.negative_sample(bench.SEED)
    tc = TrainConfig.make(lr=bench.LR, margin=bench.MARGIN, batch_size=c["B"], seed=bench.SEED)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int64)).pin_memory().numpy()
    hp, rp, tp, nhp, ntp = pin(h), pin(r), pin(t), pin(nh), pin(nt)
    for w in range(3):
        eng.set_triples(hp, rp, tp, c["N"], c["R"])
        eng.set_negatives(nhp, ntp)
        eng.train_epoch(cfg, tc, w, bench.LR)
    acc = np.zeros(4)
    per_step = []
    eng.synchronize()
    t_all = time.perf_counter()
    for k in range(args.steps):
        t0 = time.perf_counter()
        eng.set_triples(hp, rp, tp, c["N"], c["R"])
        t1 = time.perf_counter()
        eng.set_negatives(nhp, ntp)
        t2 = time.perf_counter()
        rep = eng.train_epoch(cfg, tc, 3 + k, bench.LR)
        t3 = time.perf_counter()
        acc += [t1 - t0, t2 - t1, t3 - t2, rep.t_backward_s]
        per_step.append((round((t3 - t0) * 1e3, 2), round(rep.t_backward_s * 1e3, 2)))
    tot = time.perf_counter() - t_all
    acc /= args.steps
    print(f"{args.config}: M={M} step {tot / args.steps * 1e3:.3f} ms  e2e {M * args.steps / tot / 1e6:.1f} M/s")
    print(f"  set_triples {acc[0] * 1e3:.3f} ms  set_negatives {acc[1] * 1e3:.3f} ms  "
          f"train_epoch {acc[2] * 1e3:.3f} ms (graph {acc[3] * 1e3:.3f} ms)")
    print("  per step (host ms, graph ms):", per_step)
    mb = 5 * M * 8 / 1e6
    print(f"  H2D {mb:.1f} MB -> {mb / 1e3 / (acc[0] + acc[1]):.1f} GB/s effective over the two set_* calls")
    # plain DMA of the same bytes for comparison
    d = torch.empty(5 * M, dtype=torch.int64, device="cuda")
    src = torch.from_numpy(np.concatenate([h, r, t, nh, nt]).astype(np.int64)).pin_memory()
    for _ in range(3):
        d.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"  cudaMemcpy DMA of the same {mb:.1f} MB: {dt * 1e3:.3f} ms ({mb / 1e3 / dt:.1f} GB/s)")
    eng.close()


if __name__ == "__main__":
    main()
