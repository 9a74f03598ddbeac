"""DistMult / ComplEx / RotatE on the B200 vs the oracle (pytest -m gpu).

The multiplicative family (models.cpp:201-263) runs through mult_forward
(times-times / mulsub row, exact-order score, hinge, per-entry gradient
planes) and the shared segment backward + SGD. Complex tables are
interleaved (re, im) float pairs. Bars: scores, RotatE residuals, gradients
and trained tables bit-exact against the oracle restatement (the engine
reproduces the reference's complex-product order and hypotf); losses within
1e-5. Goldens: test_models.cpp:174-221, test_eval.cpp:185-197.
"""
import numpy as np
import pytest

from paper_2502_16949_b200 import Engine, EngineError, ModelConfig, TrainConfig

pytestmark = pytest.mark.gpu

TOL = 1e-5
MODELS = ["distmult", "complex", "rotate"]


@pytest.fixture(scope="module")
def eng():
    e = Engine(0)
    yield e
    e.close()


def cpx(a):
    """complex array -> interleaved float32 table (std::complex<float> layout)"""
    a = np.ascontiguousarray(np.asarray(a, np.complex64))
    return a.view(np.float32).reshape(a.shape[0], -1).copy()


def loopfree(rng, m, n, r):
    h = rng.integers(0, n, m)
    t = (h + rng.integers(1, n, m)) % n
    return h, rng.integers(0, r, m), t


def upload(eng, model, st):
    w = 2 if model in ("complex", "rotate") else 1
    d = st.entity.shape[1] // w
    cfg = ModelConfig.make(model, d, d)
    eng.store_upload(cfg, st.entity, st.relation)
    return cfg


def test_goldens(eng):  # test_models.cpp:174-211
    cfg = ModelConfig.make("distmult", 1, 1)
    eng.store_upload(cfg, [[2.0], [5.0]], [[3.0]])
    assert eng.score_batch(cfg, [0], [0], [1])[0] == 30.0
    cfg = ModelConfig.make("complex", 1, 1)
    eng.store_upload(cfg, cpx([[1j], [1j]]), cpx([[1.0]]))
    assert eng.score_batch(cfg, [0], [0], [1])[0] == 1.0  # Re(i * 1 * conj(i)) = 1
    cfg = ModelConfig.make("rotate", 1, 1)
    eng.store_upload(cfg, cpx([[1.0], [1j]]), cpx([[1j]]))
    assert eng.score_batch(cfg, [0], [0], [1])[0] == 0.0
    eng.store_upload(cfg, cpx([[1.0], [0.0]]), cpx([[1j]]))
    assert eng.score_batch(cfg, [0], [0], [1])[0] == 1.0


@pytest.mark.parametrize("model", MODELS)
def test_rejects_self_loops_and_wrong_store(eng, orc32, model):  # test_models.cpp:213-221, 450-460
    st = orc32.init_store(model, 5, 2, 3, 3, 1)
    cfg = upload(eng, model, st)
    with pytest.raises(EngineError) as e:
        eng.score_batch(cfg, [1, 2], [0, 0], [3, 2])
    assert e.value.kind == "DegenerateTripleError" and "triple 1: head == tail" in e.value.msg
    other = "transe" if model != "distmult" else "complex"
    bad = ModelConfig.make(other, 3, 3)
    with pytest.raises(EngineError) as e:
        eng.score_batch(bad, [0], [0], [1])
    assert e.value.kind == "ConfigError"


@pytest.mark.parametrize("layout,conj", [("mult", False), ("mult_conj", True)])
def test_incidence_bitexact(eng, orc32, layout, conj):  # incidence.hpp:93-121
    rng = np.random.default_rng(3)
    h, r, t = loopfree(rng, 300, 50, 7)
    got = eng.build_incidence(layout, h, r, t, 50, 7)
    ref = orc32.build_incidence(layout, h, r, t, 50, 7)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("model", MODELS)
@pytest.mark.parametrize("d", [1, 3, 6, 16, 64, 128, 200])
def test_scores_bitexact(eng, orc32, model, d):
    rng = np.random.default_rng(d * 7 + len(model))
    n, r, m = 60, 5, 300
    st = orc32.init_store(model, n, r, d, d, d)
    h, rel, t = loopfree(rng, m, n, r)
    cfg = upload(eng, model, st)
    sc, aux = orc32.score_batch(model, st, h, rel, t)
    if model == "rotate":
        got, q = eng.score_batch(cfg, h, rel, t, residual=True)
        assert np.array_equal(q, aux["v"])
    else:
        got = eng.score_batch(cfg, h, rel, t)
    assert np.array_equal(got, sc), np.argwhere(got != sc)[:4]


@pytest.mark.parametrize("model", MODELS)
@pytest.mark.parametrize("d", [1, 5, 32, 128])
def test_score_backward_bitexact(eng, orc32, model, d):
    rng = np.random.default_rng(100 + d)
    n, r, m = 40, 5, 257
    st = orc32.init_store(model, n, r, d, d, 9)
    h, rel, t = loopfree(rng, m, n, r)
    up = rng.uniform(-1, 1, m).astype(np.float32)
    up[::7] = 0
    cfg = upload(eng, model, st)
    g0e = rng.uniform(-1, 1, st.entity.shape).astype(np.float32)
    g0r = rng.uniform(-1, 1, st.relation.shape).astype(np.float32)
    ge, gr = g0e.copy(), g0r.copy()
    eng.score_backward(cfg, h, rel, t, up, (ge, gr, None, None))
    og = st.zeros_like()
    og.entity[:] = g0e
    og.relation[:] = g0r
    orc32.score_backward(model, st, h, rel, t, up, og)
    assert np.array_equal(ge, og.entity), np.argwhere(ge != og.entity)[:4]
    assert np.array_equal(gr, og.relation)


def _fit_pair(eng, orc32, model, n, r, d, m, tc_kw, epochs, seed=3):
    h, rel, t = orc32.synthetic_train(n, r, m, seed)
    st = orc32.init_store(model, n, r, d, d, seed)
    cfg = upload(eng, model, st)
    eng.set_triples(h, rel, t, n, r)
    rg = eng.fit(cfg, TrainConfig.make(epochs=epochs, **tc_kw))
    ro = orc32.fit(model, st, h, rel, t, orc32.train_config(epochs=epochs, **tc_kw))
    ge, gr, _, _ = eng.store_download()
    for a, b in zip(rg, ro):
        assert abs(a.loss - b.loss) <= TOL * max(1.0, abs(b.loss)), (a.loss, b.loss)
    assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)
    return rg


@pytest.mark.parametrize("model", MODELS)
def test_fit_small_bitexact(eng, orc32, model):  # test_training.cpp:290-320 shape, exact tables
    _fit_pair(eng, orc32, model, 125, 6, 16, 150, dict(lr=0.1, batch_size=16, seed=20), 5)


@pytest.mark.parametrize("model", MODELS)
def test_fit_resample_scheduler(eng, orc32, model):
    _fit_pair(eng, orc32, model, 300, 9, 12, 700,
              dict(lr=0.05, batch_size=100, seed=8, resample_negatives=True, scheduler=(2, 0.5)), 4)


@pytest.mark.parametrize("model,d", [("distmult", 128), ("complex", 64), ("rotate", 64)])
def test_train_epoch_fb15k_shape(eng, orc32, model, d):
    # an FB15k-shaped graph at the C1 batch: every row kernel path at size
    _fit_pair(eng, orc32, model, 14951, 1345, d, 120000, dict(lr=4e-4, margin=0.5, batch_size=32768, seed=1), 2)


@pytest.mark.parametrize("model", MODELS)
def test_degenerate_negative_stops_at_its_batch(eng, orc32, model):
    """training.cpp:117-125: batches before the one holding a self-loop train, then
    score_batch throws DegenerateTripleError; the tables match the oracle's."""
    n, r, d = 50, 4, 6
    rng = np.random.default_rng(5)
    h, rel, t = loopfree(rng, 200, n, r)
    st = orc32.init_store(model, n, r, d, d, 5)
    nh, nt = orc32.negative_sample(h, rel, t, n, r, 5, True)
    order = orc32.epoch_order(200, 9, 0)
    k = 97  # epoch position of the bad negative: batch 3 of 32
    nh, nt = nh.copy(), nt.copy()
    nt[order[k]] = nh[order[k]]
    cfg = upload(eng, model, st)
    eng.set_triples(h, rel, t, n, r)
    eng.set_negatives(nh, nt)
    tc_e = TrainConfig.make(lr=0.05, batch_size=32, seed=9)
    with pytest.raises(EngineError) as e:
        eng.train_epoch(cfg, tc_e, 0, 0.05)
    assert e.value.kind == "DegenerateTripleError" and f"triple {k - 96}:" in e.value.msg
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as eo:
        orc32.train_epoch(model, st, (h, rel, t), (nh, nt), orc32.train_config(lr=0.05, batch_size=32, seed=9), 0, 0.05)
    assert eo.value.msg == e.value.msg
    ge, gr, _, _ = eng.store_download()
    assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)


@pytest.mark.parametrize("model", MODELS)
def test_nonfinite_gradient_raises(eng, orc32, model):
    n, r, d = 30, 3, 4
    rng = np.random.default_rng(2)
    h, rel, t = loopfree(rng, 64, n, r)
    st = orc32.init_store(model, n, r, d, d, 2)
    st.relation[int(rel[0])] = np.inf
    cfg = upload(eng, model, st)
    eng.set_triples(h, rel, t, n, r)
    eng.negative_sample(2, True)
    with pytest.raises(EngineError) as e:
        eng.train_epoch(cfg, TrainConfig.make(batch_size=16, seed=2, lr=0.1), 0, 0.1)
    assert e.value.kind == "TrainingError"


def test_degenerate_queries_rank_last(eng, orc32):  # test_eval.cpp:185-197
    st = orc32.init_store("distmult", 5, 1, 3, 3, 4)
    cfg = upload(eng, "distmult", st)
    assert eng.rank_entities(cfg, [2], [0], [2]).tolist() == [[5, 5]]
    got = eng.rank_entities(cfg, [2], [0], [1])
    assert 1 <= got[0, 0] <= 4
    assert np.array_equal(got, orc32.rank_entities("distmult", st, [2], [0], [1]))


@pytest.mark.parametrize("model", MODELS)
@pytest.mark.parametrize("d", [1, 6, 32])
@pytest.mark.parametrize("filtered", [False, True])
def test_ranks_bitexact(eng, orc32, model, d, filtered):  # eval.cpp:16-63
    n, r, q = 300, 5, 20
    rng = np.random.default_rng(d * 11 + filtered)
    st = orc32.init_store(model, n, r, d, d, 7)
    if d == 1:  # coarse values: exact ties
        st.entity[:] = rng.integers(-3, 4, st.entity.shape) / 4.0
        st.relation[:] = rng.integers(-3, 4, st.relation.shape) / 4.0
    h, rel, t = rng.integers(0, n, q), rng.integers(0, r, q), rng.integers(0, n, q)
    h[:2] = t[:2]  # self-loop queries rank dead last
    filt = None
    if filtered:
        fh, fr, ft = rng.integers(0, n, 3000), rng.integers(0, r, 3000), rng.integers(0, n, 3000)
        filt = (np.concatenate([fh, h]), np.concatenate([fr, rel]), np.concatenate([ft, t]))
    cfg = upload(eng, model, st)
    got = eng.rank_entities(cfg, h, rel, t, filt=filt)
    ref = orc32.rank_entities(model, st, h, rel, t, filt=filt)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:5]
