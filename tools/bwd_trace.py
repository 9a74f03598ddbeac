"""Per-warp timeline of the segment backward (bench config, one minibatch; needs a build with
-DSKG_BWD_TRACE, e.g. tools/build_variants.sh trace -DSKG_BWD_TRACE): when warps
that handled relation segments finish vs the others. Debug tool: python tools/bwd_trace.py C1"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig  # noqa: E402
from paper_2502_16949_b200.engine import generate_synthetic, init_store  # noqa: E402


def main():
    c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
    h, r, t = generate_synthetic(c["N"], c["R"], c["n_total"], bench.SEED)
    eng = Engine(0)
    cfg = ModelConfig.make(c["model"], c["de"], c["dr"], c["norm"])
    eng.store_upload(cfg, *init_store(c["model"], c["N"], c["R"], c["de"], c["dr"], bench.SEED))
    eng.set_triples(h, r, t, c["N"], c["R"])
    eng.negative_sample(bench.SEED)
    tc = TrainConfig.make(lr=bench.LR, margin=bench.MARGIN, batch_size=c["B"], seed=bench.SEED)
    L = eng.L
    L.skg_debug_bwd_trace.restype = ctypes.c_int64
    L.skg_debug_bwd_trace.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    eng.train_epoch(cfg, tc, 0, bench.LR)
    n = L.skg_debug_bwd_trace(3, None, None, 0)  # batch 2
    eng.train_epoch(cfg, tc, 1, bench.LR)
    buf = np.zeros(2 * n, np.uint64)
    info = np.zeros(n, np.uint32)
    L.skg_debug_bwd_trace(0, buf.ctypes.data, info.ctypes.data, n)
    st, en = buf[0::2].astype(np.int64), buf[1::2].astype(np.int64)
    ok = (st > 0) & (en > 0)
    t0 = st[ok].min()
    rel = (info >> 16) > 0
    ent = info & 0xFFFF
    for name, m in (("relation warps", ok & rel), ("entity-only warps", ok & ~rel)):
        if m.any():
            d = (en[m] - t0) / 1e3
            print(f"{name:18s} n={m.sum():5d} end median {np.median(d):6.2f} us  p90 {np.percentile(d, 90):6.2f}  max {d.max():6.2f}"
                  f"  entries median {np.median(ent[m]):.0f} max {ent[m].max()}")
    d = (st[ok] - t0) / 1e3
    print(f"warp start: median {np.median(d):.2f} us max {d.max():.2f}")


if __name__ == "__main__":
    main()
