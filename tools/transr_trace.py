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
    if os.environ.get("TR_TRACE_ALL"):  # one line per minibatch (one epoch each): kernel span
        nb = (len(h) + c["B"] - 1) // c["B"]
        for b in range(nb):
            n = L.skg_debug_transr_trace(b + 1, None, 0)
            eng.train_epoch(cfg, tcfg, 1 + b, bench.LR)
            buf = np.zeros(n, np.uint64)
            L.skg_debug_transr_trace(0, buf.ctypes.data, n)
            g = buf.reshape(160, 16, 16).astype(np.int64)[:148, 15, 12:16]
            ok = g[:, 3] > 0
            t0 = g[ok, 3].min()
            print(f"batch {b:3d}: CTA start max {(g[ok, 3].max() - t0) / 1e3:7.2f} us, loops done max "
                  f"{(g[ok, 1].max() - t0) / 1e3:7.2f}, loss {(g[:, 0].max() - t0) / 1e3:7.2f}")
        return
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
    g = tr[:148, 15, 12:16]  # globaltimer: loss written, loops done, first tile, CTA start
    ok = g[:, 3] > 0
    if ok.any():
        t0 = g[ok, 3].min()
        nt_all = np.array([sum(1 for it in range(15) if tr[c, it, 0] and tr[c, it, 14]) for c in range(148)])
        ok &= nt_all > 0
        st, ft, dn = (g[ok, 3] - t0) / 1e3, (g[ok, 2] - t0) / 1e3, (g[ok, 1] - t0) / 1e3
        nt = nt_all[ok]
        q = lambda x: f"median {np.median(x):6.2f} p10 {np.percentile(x, 10):6.2f} p90 {np.percentile(x, 90):6.2f} max {x.max():6.2f}"
        print("globaltimer, us from the first CTA start:")
        print("  CTA start      ", q(st))
        print("  first tile     ", q(ft))
        print("  loops done     ", q(dn))
        print("  tile loop / ntile (us per tile)", q((dn - ft) / np.maximum(nt, 1)))
        print("  tiles per CTA  ", np.bincount(nt))
        lw = g[:, 0][g[:, 0] > 0]
        if len(lw):
            print(f"  loss written    {(lw.max() - t0) / 1e3:.2f}")


if __name__ == "__main__":
    main()
