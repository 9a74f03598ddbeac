"""Data-parallel engine path on one GPU (NCCL communicator of size 1).

The multi-rank path is the same code with world > 1: shards of every global
minibatch, dense gradient sink, ncclAllReduce, identical dense step. With
world = 1 the dense step p - lr*g equals the touched-row step bitwise
(p - lr*0 == p), so the run must match the oracle bitwise.
"""
import numpy as np
import pytest

from paper_2502_16949_b200 import Engine, EngineError, ModelConfig, TrainConfig

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model,norm", [("transe", "l2"), ("toruse", "l1"), ("distmult", "l2"), ("complex", "l2"),
                                        ("rotate", "l2")])
def test_dp_world1_matches_oracle_bitwise(orc32, model, norm):
    n, r, d = 1500, 30, 32
    h, rel, t = orc32.synthetic_train(n, r, 12000, 2)
    st = orc32.init_store(model, n, r, d, d, 2)  # complex models: 2 * d floats per row
    eng = Engine(0)
    eng.dp_init(Engine.nccl_unique_id(), 0, 1)
    cfg = ModelConfig.make(model, d, d, norm)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(h, rel, t, n, r)
    kw = dict(lr=0.05, batch_size=1000, seed=9)
    rg = eng.fit(cfg, TrainConfig.make(epochs=3, **kw))
    ro = orc32.fit(model, st, h, rel, t, orc32.train_config(epochs=3, **kw), norm=norm)
    for a, b in zip(rg, ro):
        assert abs(a.loss - b.loss) <= 1e-5 * max(1.0, abs(b.loss))
    ge, gr, _, _ = eng.store_download()
    assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)
    eng.close()


@pytest.mark.parametrize("model,norm,d,dr", [("transh", "l2", 128, 128), ("transh", "l1", 16, 16),
                                             ("transr", "l2", 128, 128), ("transr", "l1", 16, 12)])
def test_dp_world1_ht_models(orc32, model, norm, d, dr):
    """TransH / TransR under data parallel (replicated tables for C1-C4): each rank's
    gradients go to the dense sink (relation, projection and normal sinks included), NCCL sums
    them, one dense step (+ normal renormalization). Tolerance-only models: 1e-5."""
    n, r = 1500, 12
    h, rel, t = orc32.synthetic_train(n, r, 4000, 3)
    st = orc32.init_store(model, n, r, d, dr, 3)
    if model == "transr":
        st.proj += np.random.default_rng(3).uniform(-0.1, 0.1, st.proj.shape).astype(np.float32)
    eng = Engine(0)
    eng.dp_init(Engine.nccl_unique_id(), 0, 1)
    cfg = ModelConfig.make(model, d, dr, norm)
    eng.store_upload(cfg, st.entity, st.relation, st.proj, st.normals)
    eng.set_triples(h, rel, t, n, r)
    kw = dict(lr=0.05, batch_size=512, seed=4)
    rg = eng.fit(cfg, TrainConfig.make(epochs=2, **kw))
    ro = orc32.fit(model, st, h, rel, t, orc32.train_config(epochs=2, **kw), norm=norm)
    for a, b in zip(rg, ro):
        assert abs(a.loss - b.loss) <= 1e-5 * max(1.0, abs(b.loss)), (a.loss, b.loss)
    ge, gr, gp, gn = eng.store_download()

    def rel_err(a, b):
        return float(np.max(np.abs(a.astype(np.float64) - b) / np.maximum(1.0, np.abs(b))))
    assert rel_err(ge, st.entity) <= 1e-5 and rel_err(gr, st.relation) <= 1e-5
    if gp is not None:
        assert rel_err(gp, st.proj) <= 1e-5
    if gn is not None:
        assert rel_err(gn, st.normals) <= 1e-5
    eng.close()


def test_dp_world1_bench_paths(orc32):
    """Every engine call bench.py makes under torchrun (N > 1 uses the same code with a
    larger communicator): graph-captured epochs, the evented profiling epoch and the e2e
    re-upload loop, on an NCCL communicator of size 1; tables stay equal to the oracle."""
    n, r, d = 1500, 30, 32
    h, rel, t = orc32.synthetic_train(n, r, 12000, 5)
    st = orc32.init_store("transe", n, r, d, d, 5)
    eng = Engine(0)
    cfg = ModelConfig.make("transe", d, d, "l2")
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(h, rel, t, n, r)
    nh, nt = eng.negative_sample(5)
    eng.dp_init(Engine.nccl_unique_id(), 0, 1)
    tc_e = TrainConfig.make(lr=0.05, batch_size=1000, seed=9)
    tc_o = orc32.train_config(lr=0.05, batch_size=1000, seed=9)
    ep = 0
    for _ in range(2):  # captured epoch graphs
        eng.train_epoch(cfg, tc_e, ep, 0.05)
        orc32.train_epoch("transe", st, (h, rel, t), (nh, nt), tc_o, ep, 0.05)
        ep += 1
    rep, fwd_ms, bwd_ms, plan_ms = eng.profile_epoch(cfg, tc_e, ep, 0.05)  # evented, eager
    orc32.train_epoch("transe", st, (h, rel, t), (nh, nt), tc_o, ep, 0.05)
    ep += 1
    assert fwd_ms > 0 and bwd_ms > 0
    for _ in range(2):  # e2e loop: host ids re-uploaded every epoch (synchronous under data parallel)
        eng.set_triples(h, rel, t, n, r)
        eng.set_negatives(nh, nt)
        eng.train_epoch(cfg, tc_e, ep, 0.05)
        orc32.train_epoch("transe", st, (h, rel, t), (nh, nt), tc_o, ep, 0.05)
        ep += 1
    ge, gr, _, _ = eng.store_download()
    assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)
    eng.close()
