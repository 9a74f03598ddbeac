"""Frozen golden vectors (tests/golden/goldens.npz, written by make_goldens.py).

CPU: the oracle still reproduces every vector bit for bit (pins the restatement
against drift). GPU: the engine reproduces the integer vectors (negatives,
epoch permutations, incidence CSR, filtered ranks) and the trained TransE /
TorusE tables bit-exactly, the epoch losses within 1e-5 (batch loss sums use a
deterministic tree, not the reference's sequential order).
"""
import os
import sys

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, HERE)
from make_goldens import N, R, SEED  # noqa: E402


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(HERE, "goldens.npz")))


def test_oracle_reproduces_goldens(gold):
    from make_goldens import build
    from oracle.oracle import Oracle
    g = build(Oracle("f32"))
    assert set(g) == set(gold)
    for k in gold:
        assert np.array_equal(np.asarray(g[k]), gold[k]), k


@pytest.mark.gpu
def test_engine_reproduces_goldens(gold):
    from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig
    from paper_2502_16949_b200.engine import init_store
    eng = Engine(0)
    th, tr, tt = (gold[k].astype(np.int64) for k in ("train_h", "train_r", "train_t"))
    eng.set_triples(th, tr, tt, N, R)
    nh, nt = eng.negative_sample(SEED)
    assert np.array_equal(nh, gold["neg_h"]) and np.array_equal(nt, gold["neg_t"])
    nh7, nt7 = eng.negative_sample(7, avoid_self_loops=True)
    assert np.array_equal(nh7, gold["neg7_h"]) and np.array_equal(nt7, gold["neg7_t"])
    for e in range(3):
        assert np.array_equal(eng.epoch_order(len(th), SEED, e), gold[f"order_e{e}"])
    for kind in ("hrt", "ht"):
        rp, ci, va = eng.build_incidence(kind, th[:64], tr[:64], tt[:64], N, R)
        assert np.array_equal(rp, gold[f"csr_{kind}_rp"]) and np.array_equal(ci, gold[f"csr_{kind}_ci"])
        assert np.array_equal(va, gold[f"csr_{kind}_val"])
    for model, norm, d in (("transe", "l2", 16), ("toruse", "l1", 12)):
        cfg = ModelConfig.make(model, d, d, norm)
        eng.store_upload(cfg, *init_store(model, N, R, d, d, SEED))
        eng.set_triples(th, tr, tt, N, R)
        eng.negative_sample(SEED)
        reps = eng.fit(cfg, TrainConfig.make(lr=0.01, batch_size=256, epochs=2, seed=SEED))
        ent, rel = eng.store_download()[:2]
        assert np.array_equal(ent, gold[f"{model}_entity"]), model
        assert np.array_equal(rel, gold[f"{model}_relation"]), model
        for a, b in zip(reps, gold[f"{model}_losses"]):
            assert abs(a.loss - b) <= 1e-5 * max(1.0, abs(b))
        if model == "transe":
            h, r, t = (gold[k].astype(np.int64) for k in ("all_h", "all_r", "all_t"))
            ranks = eng.rank_entities(cfg, h[:20], r[:20], t[:20], filt=(h, r, t))
            assert np.array_equal(ranks, gold["transe_ranks"])
    eng.close()
