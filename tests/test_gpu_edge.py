"""Empty and boundary inputs through the C ABI vs the oracle (pytest -m gpu).

The reference handles empty batches without error where its code allows it
(coo_to_csr / spmm on 0 rows, margin_ranking_loss with m = 0 -> loss 0,
negative_sample of an empty set) and rejects training on an empty triple set
(training.cpp:101: ConfigError). The engine must agree, and single-element
batches / the last partial minibatch must train exactly as the oracle does.
"""
import numpy as np
import pytest

from paper_2502_16949_b200 import Engine, EngineError, ModelConfig, TrainConfig

pytestmark = pytest.mark.gpu

E = np.zeros(0, np.int64)


@pytest.fixture(scope="module")
def eng():
    e = Engine(0)
    yield e
    e.close()


def test_empty_incidence(eng, orc32):  # sparse.hpp:110-161 on zero rows
    for layout in ("ht", "hrt", "mult", "mult_conj"):
        rp, col, val = eng.build_incidence(layout, E, E, E, 10, 3)
        orp, ocol, oval = orc32.build_incidence(layout, E, E, E, 10, 3)
        assert rp.tolist() == orp.tolist() == [0] and len(col) == len(ocol) == 0


@pytest.mark.parametrize("model", ["transe", "toruse", "transh", "transr", "distmult", "complex", "rotate"])
def test_empty_score_and_backward(eng, orc32, model):
    st = orc32.init_store(model, 10, 3, 4, 4, 1)
    w = 2 if model in ("complex", "rotate") else 1
    cfg = ModelConfig.make(model, st.entity.shape[1] // w, st.relation.shape[1] // w)
    eng.store_upload(cfg, st.entity, st.relation, st.proj, st.normals)
    assert len(eng.score_batch(cfg, E, E, E)) == 0
    ge = np.ones_like(st.entity)
    gr = np.ones_like(st.relation)
    eng.score_backward(cfg, E, E, E, np.zeros(0, np.float32), (ge, gr, None, None))
    assert (ge == 1).all() and (gr == 1).all()  # accumulate of nothing


def test_empty_margin_loss(eng, orc32):  # training.cpp:81: m == 0 -> zero loss, empty grads
    loss, dp, dn = eng.margin_ranking_loss(np.zeros(0, np.float32), np.zeros(0, np.float32), 0.5)
    oloss, odp, odn = orc32.margin_ranking_loss(np.zeros(0), np.zeros(0), 0.5)
    assert loss == oloss == 0.0 and len(dp) == len(dn) == 0


def test_training_requires_triples(eng, orc32):  # training.cpp:101
    st = orc32.init_store("transe", 10, 3, 4, 4, 1)
    cfg = ModelConfig.make("transe", 4, 4)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(E, E, E, 10, 3)
    eng.set_negatives(E, E)
    with pytest.raises(EngineError) as e:
        eng.train_epoch(cfg, TrainConfig.make(batch_size=4), 0, 0.1)
    assert e.value.kind == "ConfigError" and "at least one triple" in e.value.msg


def test_empty_ranking(eng, orc32):
    st = orc32.init_store("transe", 10, 3, 4, 4, 1)
    cfg = ModelConfig.make("transe", 4, 4)
    eng.store_upload(cfg, st.entity, st.relation)
    assert eng.rank_entities(cfg, E, E, E).shape == (0, 2)


@pytest.mark.parametrize("model", ["transe", "toruse", "distmult", "rotate"])
@pytest.mark.parametrize("m,bs", [(1, 1), (1, 8), (7, 3), (33, 32)])
def test_tiny_and_ragged_batches(eng, orc32, model, m, bs):
    """Single triples, batch_size larger than the set, and ragged last minibatches."""
    n, r, d = 12, 3, 6
    rng = np.random.default_rng(m * 10 + bs)
    h = rng.integers(0, n, m)
    t = (h + rng.integers(1, n, m)) % n
    rel = rng.integers(0, r, m)
    st = orc32.init_store(model, n, r, d, d, 2)
    w = 2 if model == "rotate" else 1
    cfg = ModelConfig.make(model, d, d)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(h, rel, t, n, r)
    avoid = model in ("distmult", "rotate")
    nh, nt = eng.negative_sample(3, avoid)
    onh, ont = orc32.negative_sample(h, rel, t, n, r, 3, avoid)
    assert np.array_equal(nh, onh) and np.array_equal(nt, ont)
    tc_e = TrainConfig.make(batch_size=bs, seed=5, lr=0.1)
    tc_o = orc32.train_config(batch_size=bs, seed=5, lr=0.1)
    for ep in range(3):
        re = eng.train_epoch(cfg, tc_e, ep, 0.1)
        ro = orc32.train_epoch(model, st, (h, rel, t), (nh, nt), tc_o, ep, 0.1)
        assert abs(re.loss - ro.loss) <= 1e-5 * max(1.0, abs(ro.loss))
    ge, gr, _, _ = eng.store_download()
    assert ge.shape[1] == w * d
    assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)


@pytest.mark.parametrize("model", ["transe", "complex"])
def test_fit_with_entity_renormalization(eng, orc32, model):  # training.cpp:187, embedding.cpp:192-198
    """fit(renorm_entities): every entity row back to unit norm after each epoch (row.norm()
    is an Eigen reduction: tolerance). Complex rows normalise over their (re, im) pairs."""
    n, r, d = 1500, 12, 8
    h, rel, t = orc32.synthetic_train(n, r, 4000, 4)
    st = orc32.init_store(model, n, r, d, d, 4)
    cfg = ModelConfig.make(model, d, d)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(h, rel, t, n, r)
    kw = dict(lr=0.05, batch_size=128, seed=6, renorm_entities=True)
    rg = eng.fit(cfg, TrainConfig.make(epochs=3, **kw))
    ro = orc32.fit(model, st, h, rel, t, orc32.train_config(epochs=3, **kw))
    for a, b in zip(rg, ro):
        assert abs(a.loss - b.loss) <= 1e-5 * max(1.0, abs(b.loss))
    ge, gr, _, _ = eng.store_download()
    err = np.max(np.abs(ge.astype(np.float64) - st.entity) / np.maximum(1.0, np.abs(st.entity)))
    assert err <= 1e-5, err
    assert np.allclose(np.linalg.norm(ge.astype(np.float64), axis=1), 1.0, atol=1e-5)
