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


def test_dp_rejects_ht_models(orc32):
    eng = Engine(0)
    eng.dp_init(Engine.nccl_unique_id(), 0, 1)
    st = orc32.init_store("transh", 50, 3, 8, 8, 1)
    cfg = ModelConfig.make("transh", 8, 8)
    eng.store_upload(cfg, st.entity, st.relation, None, st.normals)
    eng.set_triples([0, 1], [0, 1], [1, 2], 50, 3)
    eng.negative_sample(1)
    with pytest.raises(EngineError) as e:
        eng.train_epoch(cfg, TrainConfig.make(batch_size=2), 0, 0.1)
    assert e.value.kind == "ConfigError"
    eng.close()
