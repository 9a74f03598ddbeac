"""Epoch time of a bench config with the plan's shuffle on / off (is the plan branch the
critical path?). Debug tool: python tools/epoch_probe.py C2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig  # noqa: E402
from paper_2502_16949_b200.engine import generate_synthetic, init_store  # noqa: E402


def main():
    c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
    h, r, t = generate_synthetic(c["N"], c["R"], c["n_total"], bench.SEED)
    eng = Engine(0)
    cfg = ModelConfig.make(c["model"], c["de"], c["dr"], c["norm"])
    eng.store_upload(cfg, *init_store(c["model"], c["N"], c["R"], c["de"], c["dr"], bench.SEED))
    eng.set_triples(h, r, t, c["N"], c["R"])
    eng.negative_sample(bench.SEED)
    for shuffle in (True, False):
        tc = TrainConfig.make(lr=bench.LR, margin=bench.MARGIN, batch_size=c["B"], seed=bench.SEED, shuffle=shuffle)
        for w in range(3):
            eng.train_epoch(cfg, tc, w, bench.LR)
        ts = []
        for k in range(10):
            eng.flush_l2()
            rep = eng.train_epoch(cfg, tc, 3 + k, bench.LR)
            ts.append((rep.t_forward_s + rep.t_backward_s) * 1e3)
        ts.sort()
        print(f"shuffle={shuffle}: epoch ms median {ts[len(ts) // 2]:.4f} min {ts[0]:.4f}")


if __name__ == "__main__":
    main()
