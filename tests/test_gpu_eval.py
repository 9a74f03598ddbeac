"""Link-prediction ranking on the B200 vs the oracle (run under gpurun: pytest -m gpu).

rank_entity / evaluate (eval.cpp:16-96): ranks are integers computed from
energies in the reference's exact arithmetic, so the bar is bit-exact ranks
(raw and filtered protocols), including the reference's own known answers
(test_eval.cpp:55-115).
"""
import numpy as np
import pytest

from paper_2502_16949_b200 import Engine, ModelConfig
from paper_2502_16949_b200.engine import EngineError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    e = Engine(0)
    yield e
    e.close()


def upload(eng, st, model, norm):
    d = st.entity.shape[1]
    cfg = ModelConfig.make(model, d, st.relation.shape[1], norm)
    eng.store_upload(cfg, st.entity, st.relation, st.proj, st.normals)
    return cfg


def plane(orc):  # test_eval.cpp:47-53
    st = orc.init_store("transe", 5, 1, 2, 2, 0)
    st.entity[:] = np.array([[0, 0], [0, 1], [1, 0], [2, 0], [0.5, 0]])
    st.relation[:] = np.array([[1, 0]])
    return st


def test_rank_goldens(eng, orc32):  # test_eval.cpp:55-79
    st = plane(orc32)
    cfg = upload(eng, st, "transe", "l2")
    assert eng.rank_entities(cfg, [0], [0], [3]).tolist() == [[3, 3]]
    assert eng.rank_entities(cfg, [0], [0], [3], filt=([0, 0, 0], [0, 0, 0], [2, 4, 3]))[0, 0] == 1
    tie = orc32.init_store("transe", 6, 1, 3, 3, 0)
    tie.entity[:] = 0.25
    tie.relation[:] = 0.0
    cfg = upload(eng, tie, "transe", "l2")
    assert (eng.rank_entities(cfg, [0], [0], [4]) == 1).all()


def test_mrr_and_translations(eng, orc32):  # test_eval.cpp:87-115
    st = orc32.init_store("transe", 5, 1, 2, 2, 0)
    st.entity[:] = np.array([[0, 0], [-0.4, 0], [-0.6, 0], [-0.5, 0.1], [0.5, 0]])
    st.relation[:] = np.array([[1, 0]])
    cfg = upload(eng, st, "transe", "l2")
    rk = eng.rank_entities(cfg, [0], [0], [4])
    assert rk.tolist() == [[1, 4]]
    st = orc32.init_store("transe", 4, 1, 2, 2, 0)
    st.entity[:] = np.array([[0, 0], [1, 0], [0, 1], [1, 1]])
    st.relation[:] = np.array([[1, 0]])
    cfg = upload(eng, st, "transe", "l2")
    assert (eng.rank_entities(cfg, [0, 2], [0, 0], [1, 3]) == 1).all()


def test_rejects_bad_ids(eng, orc32):  # test_eval.cpp:81-85
    cfg = upload(eng, plane(orc32), "transe", "l2")
    with pytest.raises(EngineError):
        eng.rank_entities(cfg, [0], [0], [9])
    with pytest.raises(EngineError):
        eng.rank_entities(cfg, [0], [3], [1])


CASES = [("transe", "l2", 2), ("transe", "l1", 3), ("transe", "l2", 16), ("transe", "l1", 128),
         ("transe", "l2", 128), ("transe", "l2", 256), ("toruse", "l2", 16), ("toruse", "l1", 12),
         ("toruse", "l2", 256), ("transe", "l2", 6)]


@pytest.mark.parametrize("model,norm,d", CASES)
@pytest.mark.parametrize("filtered", [False, True])
def test_ranks_match_oracle(eng, orc32, model, norm, d, filtered):
    n, r, q = 700, 7, 37
    rng = np.random.default_rng(d * 3 + filtered)
    st = orc32.init_store(model, n, r, d, d, 5)
    if d <= 3:  # coarse values: plenty of exact ties and near ties
        st.entity[:] = rng.integers(-3, 4, st.entity.shape) / 4.0
        st.relation[:] = rng.integers(-3, 4, st.relation.shape) / 4.0
    h, rel, t = rng.integers(0, n, q), rng.integers(0, r, q), rng.integers(0, n, q)
    h[:3] = t[:3]  # self-loop queries
    filt = None
    if filtered:
        m = 4000
        fh, fr, ft = rng.integers(0, n, m), rng.integers(0, r, m), rng.integers(0, n, m)
        filt = (np.concatenate([fh, h]), np.concatenate([fr, rel]), np.concatenate([ft, t]))
    cfg = upload(eng, st, model, norm)
    got = eng.rank_entities(cfg, h, rel, t, filt=filt)
    ref = orc32.rank_entities(model, st, h, rel, t, norm=norm, filt=filt)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:5]


def test_trained_c1_shape_slice(eng, orc32):
    """FB15k-shaped ids after a short training run: ranks of 24 test triples, both protocols."""
    from paper_2502_16949_b200 import TrainConfig
    n, r = 14951, 1345
    h, rel, t = orc32.synthetic_train(n, r, 60000, 1)
    st = orc32.init_store("transe", n, r, 128, 128, 1)
    cfg = upload(eng, st, "transe", "l2")
    eng.set_triples(h, rel, t, n, r)
    eng.fit(cfg, TrainConfig.make(lr=0.01, batch_size=8192, epochs=2, seed=1))
    ent, relt = eng.store_download()[:2]
    st.entity[:] = ent
    st.relation[:] = relt
    qh, qr, qt = h[:24], rel[:24], t[:24]
    for filt in (None, (h, rel, t)):
        got = eng.rank_entities(cfg, qh, qr, qt, filt=filt)
        ref = orc32.rank_entities("transe", st, qh, qr, qt, norm="l2", filt=filt)
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("model,norm,de,dr", [("transh", "l2", 16, 16), ("transh", "l1", 128, 128),
                                              ("transr", "l2", 16, 12), ("transr", "l1", 32, 32),
                                              ("transr", "l2", 128, 128)])
@pytest.mark.parametrize("filtered", [False, True])
def test_ht_ranks_within_tolerance(eng, orc32, model, norm, de, dr, filtered):
    """TransH / TransR scores are tolerance-only (Eigen reductions in the reference):
    a device rank may differ from the oracle's only by candidates whose energy lies
    within 1e-5 (relative) of the truth's."""
    n, r, q = 400, 5, 12
    rng = np.random.default_rng(de * 5 + dr + filtered)
    st = orc32.init_store(model, n, r, de, dr, 3)
    if model == "transr":
        st.proj += rng.uniform(-0.2, 0.2, st.proj.shape).astype(np.float32)
    h, rel, t = rng.integers(0, n, q), rng.integers(0, r, q), rng.integers(0, n, q)
    h[0] = t[0]
    filt = None
    if filtered:
        fh, fr, ft = rng.integers(0, n, 2000), rng.integers(0, r, 2000), rng.integers(0, n, 2000)
        filt = (np.concatenate([fh, h]), np.concatenate([fr, rel]), np.concatenate([ft, t]))
    cfg = ModelConfig.make(model, de, dr, norm)
    eng.store_upload(cfg, st.entity, st.relation, st.proj, st.normals)
    got = eng.rank_entities(cfg, h, rel, t, filt=filt)
    ref = orc32.rank_entities(model, st, h, rel, t, norm=norm, filt=filt)
    c = np.arange(n)
    for i in range(q):
        for side in (0, 1):
            ch = np.full(n, h[i]) if side == 0 else c
            ct = c if side == 0 else np.full(n, t[i])
            e, _ = orc32.score_batch(model, st, ch, np.full(n, rel[i]), ct, norm=norm)
            truth = t[i] if side == 0 else h[i]
            near = np.abs(e - e[truth]) <= 1e-5 * np.maximum(1.0, np.abs(e[truth]))
            assert abs(int(got[i, side]) - int(ref[i, side])) <= int(near.sum()) - 1, (i, side, got[i], ref[i])
