"""Writes tests/golden/goldens.npz: derived golden vectors of the hot path.

The reference (a CMake C++ project needing Eigen3 / CLI11 / doctest) cannot be
built here, so these vectors come from the oracle restatement (oracle/, itself
pinned by the reference's own known-answer tests in tests/test_oracle_goldens.py).
They freeze, for fixed seeds: the negative sampler (training.cpp:51-71), the
epoch permutations (training.cpp:106-112), the incidence CSR (incidence.hpp:38-85),
two short training runs (TransE L2, TorusE L1; training.cpp:96-195) and filtered
ranks (eval.cpp:16-63). tests/test_goldens.py checks the oracle (CPU) and the
engine (GPU) against them.

  python tests/golden/make_goldens.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle  # noqa: E402

N, R, NT, SEED = 2000, 40, 10000, 1


def build(orc):
    g = {}
    h, r, t = orc.generate_synthetic(N, R, NT, SEED)
    n_te, n_va, _ = orc.split_sizes(NT)
    s0 = n_te + n_va
    th, tr, tt = h[s0:], r[s0:], t[s0:]
    g["train_h"], g["train_r"], g["train_t"] = th, tr, tt
    g["test_h"], g["test_r"], g["test_t"] = h[:n_te], r[:n_te], t[:n_te]
    g["all_h"], g["all_r"], g["all_t"] = h, r, t
    nh, nt = orc.negative_sample(th, tr, tt, N, R, SEED)
    g["neg_h"], g["neg_t"] = nh, nt
    nh7, nt7 = orc.negative_sample(th, tr, tt, N, R, 7, avoid_self_loops=True)
    g["neg7_h"], g["neg7_t"] = nh7, nt7
    for e in range(3):
        g[f"order_e{e}"] = orc.epoch_order(len(th), SEED, e)
    for kind in ("hrt", "ht"):
        rp, ci, va = orc.build_incidence(kind, th[:64], tr[:64], tt[:64], N, R)
        g[f"csr_{kind}_rp"], g[f"csr_{kind}_ci"], g[f"csr_{kind}_val"] = rp, ci, va
    for model, norm, d in (("transe", "l2", 16), ("toruse", "l1", 12)):
        st = orc.init_store(model, N, R, d, d, SEED)
        tc = orc.train_config(lr=0.01, batch_size=256, epochs=2, seed=SEED)
        reps = orc.fit(model, st, th, tr, tt, tc, norm=norm)
        g[f"{model}_entity"], g[f"{model}_relation"] = st.entity.copy(), st.relation.copy()
        g[f"{model}_losses"] = np.array([x.loss for x in reps], np.float64)
        if model == "transe":
            g["transe_ranks"] = orc.rank_entities("transe", st, h[:20], r[:20], t[:20], norm="l2",
                                                  filt=(h, r, t))
    return g


if __name__ == "__main__":
    g = build(Oracle("f32"))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "goldens.npz")
    g = {k: (np.asarray(v).astype(np.int32) if np.asarray(v).dtype == np.int64 else v) for k, v in g.items()}
    np.savez_compressed(out, **g)
    print(out, os.path.getsize(out), "bytes,", len(g), "arrays")
