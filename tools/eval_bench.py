"""Link-prediction ranking throughput on a BASELINE graph shape.

Trains a few epochs on the synthetic train split, then ranks every test
triple on both sides (filtered protocol over train + valid + test) through the
C ABI, timed end to end (host ids in, ranks out); reports ranks/s, pair
energies/s and the fraction of the FP32 CUDA-core instruction rate the ranking
kernel sustains (each candidate energy is d x {sub, add, mul, add} in the
reference's order: no FMA, no GEMM reformulation). The oracle restatement
(eval.cpp) ranks a bounded sample on the host for the CPU baseline and checks
the device ranks of that sample bit-exactly.

  python tools/eval_bench.py [--config C1] [--epochs 3] [--cpu-queries 8]
"""
import argparse
import json
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
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--cpu-queries", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig
    from paper_2502_16949_b200.engine import generate_synthetic, init_store
    from oracle.oracle import Oracle

    orc = Oracle("f32")
    # full split of the reference generator (data_io.cpp:128-211): train / valid / test
    # generation order (data_io.cpp:189-199): test, valid, then train
    h, r, t = orc.generate_synthetic(c["N"], c["R"], c["n_total"], bench.SEED)
    n_te, n_va, _ = orc.split_sizes(c["n_total"])
    te = (h[:n_te], r[:n_te], t[:n_te])
    s0 = n_te + n_va
    tr = (h[s0:], r[s0:], t[s0:])
    eng = Engine(0)
    cfg = ModelConfig.make(c["model"], c["de"], c["dr"], c["norm"])
    ent, rel, proj, nrm = init_store(c["model"], c["N"], c["R"], c["de"], c["dr"], bench.SEED)
    eng.store_upload(cfg, ent, rel, proj, nrm)
    eng.set_triples(*tr, c["N"], c["R"])
    eng.fit(cfg, TrainConfig.make(lr=bench.LR, margin=bench.MARGIN, batch_size=c["B"], epochs=args.epochs,
                                  seed=bench.SEED))
    filt = (h, r, t)
    eng.rank_entities(cfg, te[0][:64], te[1][:64], te[2][:64], filt=filt)  # warm
    times = []
    for _ in range(args.reps):
        eng.synchronize()
        t0 = time.perf_counter()
        ranks = eng.rank_entities(cfg, *te, filt=filt)
        times.append(time.perf_counter() - t0)
    secs = min(times)
    q = len(te[0])
    pairs = 2.0 * q * c["N"]
    inst = pairs * c["de"] * 4
    peak_inst = 148 * 128 * 1.965e9
    mrr = float(np.mean(1.0 / ranks))
    hits10 = float(np.mean(ranks <= 10))
    # CPU baseline + bit-exact check on a sample
    ent_d, rel_d = eng.store_download()[:2]
    st = orc.init_store(c["model"], c["N"], c["R"], c["de"], c["dr"], bench.SEED)
    st.entity[:] = ent_d
    st.relation[:] = rel_d
    k = args.cpu_queries
    t0 = time.perf_counter()
    ref = orc.rank_entities(c["model"], st, te[0][:k], te[1][:k], te[2][:k], norm=c["norm"], filt=filt)
    cpu_s = time.perf_counter() - t0
    exact = bool(np.array_equal(ref, ranks[:k]))
    out = {"metric": "filtered link-prediction ranks/s (both sides of every test triple, all candidates)",
           "config": args.config, "model": c["model"], "entities": c["N"], "test_triples": q,
           "ranks_per_s": 2 * q / secs, "seconds": secs, "pair_energies_per_s": pairs / secs,
           "cuda_core_inst_frac": inst / secs / peak_inst, "mrr": mrr, "hits_at_10": hits10,
           "cpu_baseline": {"ranks_per_s": 2 * k / cpu_s, "sample": f"{k} test triples, oracle restatement, 1 thread",
                            "kind": "port"},
           "sample_bit_exact": exact, "train_epochs": args.epochs}
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()
