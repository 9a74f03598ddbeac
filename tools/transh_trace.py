"""Phase timeline of the TransH pipelined training kernel (C2 shape, one minibatch).

Enables the kernel's globaltimer stamps for batch 1 of an epoch and prints, per
event, the median / max offset (us) from the earliest kernel start over CTAs.
Debug tool; not part of the product path.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig  # noqa: E402

EV = {0: "start", 1: "setup", 2: "chase0", 3: "copy0", 4: "copy1", 5: "copy2", 6: "copy3", 7: "full0", 8: "full1",
      9: "full2", 10: "full3", 11: "done0", 12: "done1", 13: "done2", 14: "done3", 15: "flush", 16: "flushed",
      17: "loss", 18: "end", 19: "t0_loaded", 20: "t0_v", 21: "t0_hinge", 22: "t0_dzw",
      23: "t1_loaded", 24: "t1_v", 25: "t1_hinge", 26: "t1_dzw"}


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
    c = bench.CONFIGS[cfgname]
    from paper_2502_16949_b200.engine import generate_synthetic, init_store
    h, r, t = generate_synthetic(c["N"], c["R"], c["n_total"], bench.SEED)
    eng = Engine(0)
    cfg = ModelConfig.make(c["model"], c["de"], c["dr"], c["norm"])
    eng.store_upload(cfg, *init_store(c["model"], c["N"], c["R"], c["de"], c["dr"], bench.SEED))
    eng.set_triples(h, r, t, c["N"], c["R"])
    eng.negative_sample(bench.SEED)
    tcfg = TrainConfig.make(lr=bench.LR, margin=bench.MARGIN, batch_size=c["B"], seed=bench.SEED)
    L = eng.L
    L.skg_debug_transh_trace.restype = ctypes.c_int64
    L.skg_debug_transh_trace.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64]
    eng.train_epoch(cfg, tcfg, 0, bench.LR)  # warm (graph capture)
    n = L.skg_debug_transh_trace(2, None, 0)  # trace batch 1
    eng.train_epoch(cfg, tcfg, 1, bench.LR)
    buf = np.zeros(n, np.uint64)
    L.skg_debug_transh_trace(0, buf.ctypes.data, n)
    tr = buf.reshape(160, 32).astype(np.int64)
    ok = tr[:, 0] > 0
    t0 = tr[ok, 0].min()
    print(f"{ok.sum()} CTAs traced; offsets from the first CTA start (us): median / max")
    for ev, name in EV.items():
        col = tr[ok, ev]
        col = col[col > 0]
        if len(col):
            print(f"  {name:8s} {np.median(col - t0) / 1e3:8.2f} {np.max(col - t0) / 1e3:8.2f}  (n={len(col)})")


if __name__ == "__main__":
    main()
