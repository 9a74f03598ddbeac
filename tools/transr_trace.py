"""Phase timeline of the TransR tcgen05 training kernel (C4 shape, one minibatch).

Runs bench.py's C4 setup, enables the kernel's clock64 phase stamps for batch 0
and prints the mean per-tile offsets of each event relative to the tile's
producer start, plus per-tile period. Debug tool; not part of the product path.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig  # noqa: E402

EV = ["pro_start", "gathered", "u_full", "pro_dz", "g3_staged", "mma_u", "g1_issued", "g3_first", "g3_issued",
      "g2_start", "g2_issued", "epi_v", "epi_dz", "epi_g2", "epi_drained", "pro_g2ok"]


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
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
    L.skg_debug_transr_trace.restype = ctypes.c_int64
    L.skg_debug_transr_trace.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64]
    eng.train_epoch(cfg, tcfg, 0, bench.LR)  # warm (graph capture)
    tb = int(os.environ.get("TR_TRACE_BATCH", "0"))
    n = L.skg_debug_transr_trace(tb + 1, None, 0)  # trace batch tb
    eng.train_epoch(cfg, tcfg, 1, bench.LR)
    buf = np.zeros(n, np.uint64)
    L.skg_debug_transr_trace(0, buf.ctypes.data, n)
    tr = buf.reshape(160, 16, 16).astype(np.int64)
    rows = []
    for cta in range(148):
        for it in range(16):
            e = tr[cta, it]
            if e[0] == 0 or e[14] == 0:
                continue
            rows.append(e[:16] - e[0])
    rows = np.array(rows)
    print(f"{len(rows)} traced tiles; offsets from pro_start (cycles), median:")
    for i, name in enumerate(EV):
        print(f"  {name:12s} {int(np.median(rows[:, i])):8d}")
    per = []
    for cta in range(148):
        s = [tr[cta, it, 0] for it in range(16) if tr[cta, it, 0] and tr[cta, it, 14]]
        per += list(np.diff(s))
    print("tile period (median cycles):", int(np.median(per)) if per else None)
    st = tr[:148, 15, 15]
    st = st[st > 0]
    if len(st):
        d = (st - st.min()) / 1e3
        print(f"CTA start (globaltimer): median {np.median(d):.2f} us, p90 {np.percentile(d, 90):.2f}, max {d.max():.2f}")


if __name__ == "__main__":
    main()
