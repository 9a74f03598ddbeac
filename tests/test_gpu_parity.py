"""CUDA engine vs CPU oracle parity (run on a B200: pytest -m gpu).

Bars (BASELINE north_star):
  - incidence CSR, negative indices and epoch permutations: bit-exact;
  - TransE / TorusE scores, residuals, gradients and trained embeddings:
    bit-exact (the engine reproduces the reference's float association);
  - losses and embeddings after N steps: max_rel_err <= 1e-5 where the
    reference order is not reproduced (batch loss sums).
"""
import numpy as np
import pytest

from paper_2502_16949_b200 import Engine, EngineError, ModelConfig, TrainConfig

pytestmark = pytest.mark.gpu

TOL = 1e-5  # north_star: within 1e-5 relative after N fp32 steps


def max_rel_err(a, b):  # test_util.hpp:102-113
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))


@pytest.fixture(scope="module")
def eng():
    e = Engine(0)
    yield e
    e.close()


def rand_triples(rng, m, n, r, self_loops=True):
    h = rng.integers(0, n, m)
    t = rng.integers(0, n, m) if self_loops else (h + rng.integers(1, n, m)) % n
    return h, rng.integers(0, r, m), t


# ------------------------------------------------------------------ RNG streams
@pytest.mark.parametrize("m,n,seed", [(4, 10, 7), (1000, 40, 11), (100003, 14951, 1), (5, 2, 3)])
@pytest.mark.parametrize("avoid", [False, True])
def test_negative_sample_bitexact(eng, orc32, m, n, seed, avoid):
    if avoid and n < 3:
        pytest.skip("avoid mode needs 3 entities")
    rng = np.random.default_rng(seed)
    h, r, t = rand_triples(rng, m, n, 3, self_loops=not avoid)
    eng.set_triples(h, r, t, n, 3)
    gh, gt = eng.negative_sample(seed, avoid)
    oh, ot = orc32.negative_sample(h, r, t, n, 3, seed, avoid)
    assert np.array_equal(gh, oh) and np.array_equal(gt, ot)


def test_negative_sample_toy_vector(eng):  # SURVEY §8c derived vector
    eng.set_triples([0, 1, 2, 3], [0, 0, 0, 0], [5, 6, 7, 8], 10, 1)
    nh, nt = eng.negative_sample(7)
    assert nh.tolist() == [0, 9, 0, 3] and nt.tolist() == [9, 6, 7, 9]


def test_negative_sample_config_errors(eng):
    eng.set_triples([0], [0], [0], 1, 1)
    with pytest.raises(EngineError) as e:
        eng.negative_sample(0)
    assert e.value.kind == "ConfigError"


@pytest.mark.parametrize("m", [0, 1, 2, 3, 4, 10, 11, 1000, 4097, 483142])
def test_epoch_order_bitexact(eng, orc32, m):
    for epoch in (0, 1, 7):
        g = eng.epoch_order(m, 42, epoch)
        o = orc32.epoch_order(m, 42, epoch)
        assert np.array_equal(g, o), (m, epoch)
    assert np.array_equal(eng.epoch_order(m, 42, 0, shuffle=False), np.arange(m))


@pytest.mark.slow
def test_epoch_order_bitexact_large(eng, orc32):
    # 16.1M (ogbl-wikikg2 train size): Lemire rejections occur at this scale.
    m = 16109182
    assert np.array_equal(eng.epoch_order(m, 1, 0), orc32.epoch_order(m, 1, 0))


# ------------------------------------------------------------------ incidence
@pytest.mark.parametrize("layout", ["ht", "hrt"])
def test_build_incidence_bitexact(eng, orc32, layout):
    rng = np.random.default_rng(5)
    for m, n, r in ((1, 22, 1), (37, 10, 4), (5000, 300, 17)):
        h, rel, t = rand_triples(rng, m, n, r)
        h[0] = t[0]  # force a self-loop
        g = eng.build_incidence(layout, h, rel, t, n, r)
        o = orc32.build_incidence(layout, h, rel, t, n, r)
        for a, b in zip(g, o):
            assert np.array_equal(a, b)


def test_incidence_goldens(eng):  # test_incidence.cpp:30-77
    rp, c, v = eng.build_incidence("ht", [5], [0], [15], 22, 1)
    assert rp.tolist() == [0, 2] and c.tolist() == [5, 15] and v.tolist() == [1, -1]
    rp, c, v = eng.build_incidence("hrt", [5], [2], [15], 20, 3)
    assert c.tolist() == [5, 15, 22] and v.tolist() == [1, -1, 1]
    rp, c, v = eng.build_incidence("hrt", [4], [1], [4], 7, 3)
    assert rp.tolist() == [0, 1] and c.tolist() == [8]
    rp, c, v = eng.build_incidence("ht", [3], [0], [3], 8, 1)
    assert rp.tolist() == [0, 0] and len(c) == 0
    with pytest.raises(EngineError) as e:
        eng.build_incidence("ht", [3], [0], [0], 3, 1)
    assert e.value.kind == "ShapeError"


# ------------------------------------------------------------------ scoring
HRT = [("transe", "l2"), ("transe", "l1"), ("toruse", "l2"), ("toruse", "l1")]


@pytest.mark.parametrize("model,norm", HRT)
@pytest.mark.parametrize("d", [1, 3, 6, 8, 128, 256])
def test_score_batch_bitexact(eng, orc32, model, norm, d):
    rng = np.random.default_rng(d)
    n, r, m = 50, 7, 333
    st = orc32.init_store(model, n, r, d, d, 3)
    h, rel, t = rand_triples(rng, m, n, r)
    h[:3] = t[:3]
    cfg = ModelConfig.make(model, d, d, norm)
    eng.store_upload(cfg, st.entity, st.relation)
    gs, gres = eng.score_batch(cfg, h, rel, t, residual=True)
    os_, aux = orc32.score_batch(model, st, h, rel, t, norm=norm)
    assert np.array_equal(gs, os_)
    assert np.array_equal(gres, aux["delta"] if model == "toruse" else aux["v"])


@pytest.mark.parametrize("model,norm", HRT)
@pytest.mark.parametrize("d", [1, 5, 8, 128, 256])
def test_score_backward_bitexact(eng, orc32, model, norm, d):
    rng = np.random.default_rng(100 + d)
    n, r, m = 40, 5, 257
    st = orc32.init_store(model, n, r, d, d, 9)
    h, rel, t = rand_triples(rng, m, n, r)
    h[:2] = t[:2]
    up = rng.uniform(-1, 1, m).astype(np.float32)
    up[::7] = 0
    cfg = ModelConfig.make(model, d, d, norm)
    eng.store_upload(cfg, st.entity, st.relation)
    g0e = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    g0r = rng.uniform(-1, 1, (r, d)).astype(np.float32)
    ge, gr = g0e.copy(), g0r.copy()
    eng.score_backward(cfg, h, rel, t, up, (ge, gr, None, None))
    og = st.zeros_like()
    og.entity[:] = g0e
    og.relation[:] = g0r
    orc32.score_backward(model, st, h, rel, t, up, og, norm=norm)
    assert np.array_equal(ge, og.entity)
    assert np.array_equal(gr, og.relation)


def test_model_goldens(eng):  # test_models.cpp:54-102
    cfg = ModelConfig.make("transe", 2, 2, "l2")
    eng.store_upload(cfg, [[1, 2], [0, 0]], [[0, 0]])
    assert eng.score_batch(cfg, [0], [0], [1])[0] == np.float32(np.sqrt(np.float32(5)))
    cfg1 = ModelConfig.make("transe", 2, 2, "l1")
    assert eng.score_batch(cfg1, [0], [0], [1])[0] == 3.0
    eng.store_upload(cfg, [[3, 4], [0, 0]], [[0, 0]])
    ge, gr = np.zeros((2, 2), np.float32), np.zeros((1, 2), np.float32)
    eng.score_backward(cfg, [0], [0], [1], [1.0], (ge, gr, None, None))
    np.testing.assert_allclose(ge, [[0.6, 0.8], [-0.6, -0.8]], atol=1e-6)
    cfgt = ModelConfig.make("toruse", 1, 1, "l2")
    eng.store_upload(cfgt, [[0.75], [0]], [[0]])
    assert eng.score_batch(cfgt, [0], [0], [1])[0] == 0.0625
    eng.store_upload(cfgt, [[1.5], [0]], [[0]])
    assert eng.score_batch(cfgt, [0], [0], [1])[0] == 0.25
    assert eng.score_batch(ModelConfig.make("toruse", 1, 1, "l1"), [0], [0], [1])[0] == 0.5


def test_config_errors(eng):
    cfg = ModelConfig.make("transe", 4, 4)
    eng.store_upload(cfg, np.zeros((5, 4)), np.zeros((2, 4)))
    for bad in (ModelConfig.make("transe", 6, 6), ModelConfig.make("transr", 4, 4), ModelConfig.make("transh", 4, 4)):
        with pytest.raises(EngineError) as e:
            eng.score_batch(bad, [0], [0], [1])
        assert e.value.kind == "ConfigError"
    with pytest.raises(EngineError) as e:
        eng.score_batch(cfg, [0], [0], [7])
    assert e.value.kind == "ShapeError"


# ------------------------------------------------------------------ loss / sgd
def test_margin_ranking_loss_goldens(eng):  # test_training.cpp:103-136
    loss, dp, dn = eng.margin_ranking_loss([1.0], [0.2], 0.5)
    assert abs(loss - 1.3) < 1e-6 and dp[0] == 1.0 and dn[0] == -1.0
    loss, dp, _ = eng.margin_ranking_loss([0.7], [0.7], 0.0)
    assert loss == 0.0 and dp[0] == 0.0
    loss, dp, dn = eng.margin_ranking_loss([1.0, 0.0], [0.2, 5.0], 0.5)
    assert abs(loss - 0.65) < 1e-6 and dp.tolist() == [0.5, 0.0] and dn[0] == -0.5
    with pytest.raises(EngineError):
        eng.margin_ranking_loss([1.0, 0.0], [1.0, 2.0, 3.0], 0.5)


def test_margin_ranking_loss_matches_oracle(eng, orc32):
    rng = np.random.default_rng(21)
    p, n = rng.uniform(-5, 5, 10001).astype(np.float32), rng.uniform(-5, 5, 10001).astype(np.float32)
    a = eng.margin_ranking_loss(p, n, 0.5)
    b = orc32.margin_ranking_loss(p, n, 0.5)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_sgd_step_goldens(eng, orc32):  # test_embedding.cpp:128-179
    cfg = ModelConfig.make("transe", 1, 1)
    eng.store_upload(cfg, [[1.0]], [[0.0]])
    eng.sgd_step([[2.0]], [[0.0]], None, None, 0.1)
    assert eng.store_download()[0][0, 0] == np.float32(1) - np.float32(0.1) * np.float32(2)
    st = orc32.init_store("transe", 3, 2, 4, 4, 1)
    eng.store_upload(ModelConfig.make("transe", 4, 4), st.entity, st.relation)
    g = np.zeros((3, 4), np.float32)
    g[1, 2] = np.nan
    with pytest.raises(EngineError) as e:
        eng.sgd_step(g, np.zeros((2, 4)), None, None, 0.1)
    assert e.value.kind == "TrainingError" and "entity" in e.value.msg
    assert np.array_equal(eng.store_download()[0], st.entity)  # nothing applied


def test_renormalize_entities(eng):  # test_embedding.cpp:209-218
    cfg = ModelConfig.make("transe", 2, 2)
    eng.store_upload(cfg, [[3, 4], [0, 0], [0.5, 0]], [[0, 0]])
    eng.renormalize_entities()
    np.testing.assert_allclose(eng.store_download()[0], [[0.6, 0.8], [0, 0], [1, 0]], atol=1e-7)


# ------------------------------------------------------------------ training
def _train_pair(eng, orc32, model, norm, n, r, d, m, tc_kw, epochs, seed=3, check_exact=True):
    h, rel, t = orc32.synthetic_train(n, r, m, seed)
    st = orc32.init_store(model, n, r, d, d, seed)
    cfg = ModelConfig.make(model, d, d, norm)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(h, rel, t, n, r)
    tc_e = TrainConfig.make(epochs=epochs, **tc_kw)
    tc_o = orc32.train_config(epochs=epochs, **tc_kw)
    rg = eng.fit(cfg, tc_e)
    ro = orc32.fit(model, st, h, rel, t, tc_o, norm=norm)
    ge, gr, _, _ = eng.store_download()
    for a, b in zip(rg, ro):
        assert abs(a.loss - b.loss) <= TOL * max(1.0, abs(b.loss)), (a.loss, b.loss)
    assert max_rel_err(ge, st.entity) <= TOL and max_rel_err(gr, st.relation) <= TOL
    if check_exact:
        assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)
    return rg, ro


@pytest.mark.parametrize("model,norm", HRT)
def test_fit_small_bitexact_tables(eng, orc32, model, norm):
    _train_pair(eng, orc32, model, norm, 125, 6, 16, 150, dict(lr=0.1, batch_size=16, seed=20), 5)


def test_fit_scheduler_and_no_shuffle(eng, orc32):
    _train_pair(eng, orc32, "transe", "l2", 300, 9, 8, 700,
                dict(lr=0.05, batch_size=64, seed=4, scheduler=(2, 0.5), shuffle=False), 5)


def test_fit_resample_negatives(eng, orc32):
    _train_pair(eng, orc32, "transe", "l1", 300, 9, 12, 700,
                dict(lr=0.05, batch_size=100, seed=8, resample_negatives=True), 3)


def test_train_epoch_fb15k_shape(eng, orc32):
    # C1 (BASELINE configs[0]): TransE d=128 L2, 14,951 ent, 1,345 rel, batch 32768.
    _train_pair(eng, orc32, "transe", "l2", 14951, 1345, 128, 536824,
                dict(lr=4e-4, margin=0.5, batch_size=32768, seed=1), 2)


def test_train_epoch_toruse_fb15k237_shape(eng, orc32):
    # C3: TorusE d=256 L2-torus on an FB15k-237-shaped graph, batch 32768.
    _train_pair(eng, orc32, "toruse", "l2", 14541, 237, 256, 302349,
                dict(lr=4e-4, margin=0.5, batch_size=32768, seed=1), 1)


def test_nonfinite_loss_raises_with_epoch_and_batch(eng, orc32):
    n, r, d = 200, 5, 8
    h, rel, t = orc32.synthetic_train(n, r, 300, 2)
    st = orc32.init_store("transe", n, r, d, d, 2)
    st.entity[int(h[0])] = np.inf
    cfg = ModelConfig.make("transe", d, d)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(h, rel, t, n, r)
    eng.negative_sample(2)
    with pytest.raises(EngineError) as e:
        eng.train_epoch(cfg, TrainConfig.make(batch_size=16, seed=2), 0, 0.1)
    assert e.value.kind == "TrainingError" and "non-finite loss at epoch 0" in e.value.msg


def test_lr0_freezes(eng, orc32):
    n, r, d = 20, 4, 8
    st = orc32.init_store("transe", n, r, d, d, 5)
    h, rel, t = rand_triples(np.random.default_rng(5), 100, n, r, self_loops=False)
    cfg = ModelConfig.make("transe", d, d)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(h, rel, t, n, r)
    eng.negative_sample(6)
    rep = eng.train_epoch(cfg, TrainConfig.make(batch_size=32, margin=1.0), 0, 0.0)
    assert rep.loss > 0 and np.array_equal(eng.store_download()[0], st.entity)


@pytest.mark.parametrize("name", ["shim_drop_in", "ref_cases"])
def test_cpp_shim_drop_in_runs(name):
    """A reference-style C++ caller, and the reference's own unit-test case bodies
    (test_models / test_training / test_embedding / test_sparse / test_incidence,
    adapted to fp32, tests/cpp/ref_cases.cpp), run over the shim + C ABI."""
    import os
    import subprocess
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2502_16949_b200")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "shim")
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "cpp", name + ".cpp"), "-o", exe, "-L", lib,
                        "-lskge_b200", f"-Wl,-rpath,{lib}"], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stdout + out.stderr


def _pinned(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.int64)).pin_memory().numpy()


@pytest.mark.parametrize("pinned", [False, True])
def test_reupload_between_epochs_keeps_parity(eng, orc32, pinned):
    """The e2e loop re-uploads the same triples/negatives every epoch (identical
    content keeps the prefetched epoch plan); a changed upload must rebuild it.
    Pinned caller arrays take the zero-copy narrowing path."""
    n, r, d, m = 400, 7, 16, 900
    h, rel, t = orc32.synthetic_train(n, r, m, 9)
    if pinned:
        h, rel, t = _pinned(h), _pinned(rel), _pinned(t)
    st = orc32.init_store("transe", n, r, d, d, 9)
    cfg = ModelConfig.make("transe", d, d, "l2")
    tc_e = TrainConfig.make(batch_size=128, seed=5, lr=0.05)
    tc_o = orc32.train_config(batch_size=128, seed=5, lr=0.05)
    nh, nt = orc32.negative_sample(h, rel, t, n, r, 3)
    rng = np.random.default_rng(1)
    nh2, nt2 = rng.integers(0, n, len(h)), rng.integers(0, n, len(h))
    if pinned:
        nh, nt, nh2, nt2 = _pinned(nh), _pinned(nt), _pinned(nh2), _pinned(nt2)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_deferred_uploads(pinned)
    plan = [(nh, nt), (nh, nt), (nh2, nt2), (nh2, nt2), (nh, nt)]
    for ep, (a, b) in enumerate(plan):
        eng.set_triples(h, rel, t, n, r)
        eng.set_negatives(a, b)
        re = eng.train_epoch(cfg, tc_e, ep, 0.05)
        ro = orc32.train_epoch("transe", st, (h, rel, t), (a, b), tc_o, ep, 0.05)
        assert abs(re.loss - ro.loss) <= TOL * max(1.0, abs(ro.loss))
        ge, gr, _, _ = eng.store_download()
        assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation), ep
    # a changed positive set (same size) with the old negatives
    h3 = (h + 1) % n
    eng.set_triples(h3, rel, t, n, r)
    eng.set_negatives(nh, nt)
    eng.train_epoch(cfg, tc_e, 5, 0.05)
    orc32.train_epoch("transe", st, (h3, rel, t), (nh, nt), tc_o, 5, 0.05)
    ge, gr, _, _ = eng.store_download()
    assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)
    if pinned:
        hits, misses = eng.upload_stats()
        assert hits >= 1 and misses >= 1, (hits, misses)
    eng.set_deferred_uploads(False)


def test_default_upload_is_copied_inside_the_call(eng, orc32):
    """Deferral is opt-in: by default set_triples / set_negatives copy pinned arrays
    inside the call, so the caller may overwrite them before train_epoch
    (the reference's by-value TripleBatch semantics)."""
    n, r, d, m = 300, 5, 8, 700
    h, rel, t = orc32.synthetic_train(n, r, m, 6)
    st = orc32.init_store("transe", n, r, d, d, 6)
    cfg = ModelConfig.make("transe", d, d, "l2")
    tc_e = TrainConfig.make(batch_size=64, seed=3, lr=0.05)
    tc_o = orc32.train_config(batch_size=64, seed=3, lr=0.05)
    nh, nt = orc32.negative_sample(h, rel, t, n, r, 3)
    P = [_pinned(x) for x in (h, rel, t, nh, nt)]
    eng.store_upload(cfg, st.entity, st.relation)
    for ep in range(3):
        eng.set_triples(*P[:3], n, r)
        eng.set_negatives(*P[3:])
        for a in P:  # the caller reuses its buffers right after the calls
            a[:] = 0
        eng.train_epoch(cfg, tc_e, ep, 0.05)
        orc32.train_epoch("transe", st, (h, rel, t), (nh, nt), tc_o, ep, 0.05)
        for a, b in zip(P, (h, rel, t, nh, nt)):
            a[:] = b
    ge, gr, _, _ = eng.store_download()
    assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)


def test_pinned_upload_rejects_bad_ids(eng):
    h = _pinned(np.array([0, 1, 2, 3]))
    r = _pinned(np.array([0, 0, 1, 0]))
    t = _pinned(np.array([1, 2, 9, 0]))
    with pytest.raises(EngineError) as e:
        eng.set_triples(h, r, t, 5, 2)
    assert e.value.kind == "ShapeError" and "triple 2: entity id out of range" in e.value.msg
    r[1] = 7
    t[2] = 3
    with pytest.raises(EngineError) as e:
        eng.set_triples(h, r, t, 5, 2)
    assert "triple 1: relation id out of range" in e.value.msg


def test_deferred_reupload_invalid_ids_roll_back(eng, orc32):
    """A pinned identical-shape re-upload is copied while the next epoch trains
    (speculatively, on the previous ids). Invalid ids must surface as the
    set_triples / set_negatives ShapeError with the parameters untouched; changed
    ids must train exactly as a synchronous upload would."""
    n, r, d, m = 300, 5, 8, 700
    h, rel, t = orc32.synthetic_train(n, r, m, 4)
    m = len(h)
    st = orc32.init_store("transe", n, r, d, d, 4)
    cfg = ModelConfig.make("transe", d, d, "l2")
    tc_e = TrainConfig.make(batch_size=64, seed=3, lr=0.05)
    tc_o = orc32.train_config(batch_size=64, seed=3, lr=0.05)
    nh, nt = orc32.negative_sample(h, rel, t, n, r, 3)
    P = [_pinned(x) for x in (h, rel, t, nh, nt)]
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_deferred_uploads(True)
    try:
        _deferred_body(eng, orc32, cfg, tc_e, tc_o, st, P, h, rel, t, nh, nt, n, r)
    finally:
        eng.set_deferred_uploads(False)


def _deferred_body(eng, orc32, cfg, tc_e, tc_o, st, P, h, rel, t, nh, nt, n, r):
    eng.set_triples(*P[:3], n, r)
    eng.set_negatives(*P[3:])
    eng.train_epoch(cfg, tc_e, 0, 0.05)
    orc32.train_epoch("transe", st, (h, rel, t), (nh, nt), tc_o, 0, 0.05)
    before = eng.store_download()[0].copy()
    assert np.array_equal(before, st.entity)
    # invalid entity id in the triples: deferred, raised by train_epoch, nothing trained
    bad = P[2].copy()
    bad = _pinned(bad)
    bad[17] = n + 3
    eng.set_triples(P[0], P[1], bad, n, r)
    eng.set_negatives(*P[3:])
    with pytest.raises(EngineError) as e:
        eng.train_epoch(cfg, tc_e, 1, 0.05)
    assert e.value.kind == "ShapeError" and e.value.msg == "triple 17: entity id out of range"
    assert np.array_equal(eng.store_download()[0], before)
    # invalid negative: triples adopted, negatives rejected, nothing trained
    eng.set_triples(*P[:3], n, r)
    eng.set_negatives(*P[3:])
    eng.train_epoch(cfg, tc_e, 1, 0.05)
    orc32.train_epoch("transe", st, (h, rel, t), (nh, nt), tc_o, 1, 0.05)
    before = eng.store_download()[0].copy()
    badn = _pinned(P[3].copy())
    badn[5] = -1
    eng.set_triples(*P[:3], n, r)
    eng.set_negatives(badn, P[4])
    with pytest.raises(EngineError) as e:
        eng.train_epoch(cfg, tc_e, 2, 0.05)
    assert e.value.kind == "ShapeError" and e.value.msg == "triple 5: entity id out of range"
    assert np.array_equal(eng.store_download()[0], before)
    with pytest.raises(EngineError) as e:  # negatives are not valid any more
        eng.train_epoch(cfg, tc_e, 2, 0.05)
    assert e.value.kind == "ShapeError"
    # changed ids of the same shape: rolled back and retrained on the new ids
    h2 = _pinned((h + 7) % n)
    eng.set_negatives(*P[3:])
    eng.train_epoch(cfg, tc_e, 2, 0.05)
    orc32.train_epoch("transe", st, (h, rel, t), (nh, nt), tc_o, 2, 0.05)
    eng.set_triples(h2, P[1], P[2], n, r)
    eng.set_negatives(*P[3:])
    eng.train_epoch(cfg, tc_e, 3, 0.05)
    orc32.train_epoch("transe", st, ((h + 7) % n, rel, t), (nh, nt), tc_o, 3, 0.05)
    ge, gr, _, _ = eng.store_download()
    assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation)
    # a deferred upload is visible to every other call (negative_sample resolves it)
    eng.set_triples(*P[:3], n, r)
    gh, gt = eng.negative_sample(11)
    oh, ot = orc32.negative_sample(h, rel, t, n, r, 11)
    assert np.array_equal(gh, oh) and np.array_equal(gt, ot)


@pytest.mark.parametrize("n,wire", [(20000, 2), (65536, 2), (65537, 4), (70000, 4)])
def test_deferred_reupload_large_narrowing(eng, orc32, n, wire):
    """Host-narrowed deferred uploads at a size that spreads the five id arrays over
    every narrowing thread and all four DMA waves: an identical re-upload keeps the
    speculative epoch (hit), one changed negative id in the last wave is detected
    (miss) and retrained; tables stay bitwise the oracle's. Ids travel as uint16
    when every table has at most 65536 rows, else as int32."""
    r, d = 60, 8
    h, rel, t = orc32.synthetic_train(n, r, 220000, 11)
    m = len(h)
    st = orc32.init_store("transe", n, r, d, d, 11)
    cfg = ModelConfig.make("transe", d, d, "l2")
    tc_e = TrainConfig.make(batch_size=8192, seed=4, lr=0.05)
    tc_o = orc32.train_config(batch_size=8192, seed=4, lr=0.05)
    nh, nt = orc32.negative_sample(h, rel, t, n, r, 2)
    nh[m // 2] = n - 1  # the largest id the wire format must carry (65535 at n = 65536)
    P = [_pinned(x) for x in (h, rel, t, nh, nt)]
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(*P[:3], n, r)
    eng.set_negatives(*P[3:])
    eng.train_epoch(cfg, tc_e, 0, 0.05)
    orc32.train_epoch("transe", st, (h, rel, t), (nh, nt), tc_o, 0, 0.05)
    eng.set_deferred_uploads(True)
    try:
        hits0, miss0 = eng.upload_stats()
        bytes0 = eng.upload_bytes()
        for ep in (1, 2):
            if ep == 2:
                P[4][m - 3] = (P[4][m - 3] + 1) % n  # last wave, last array
            eng.set_triples(*P[:3], n, r)
            eng.set_negatives(*P[3:])
            eng.train_epoch(cfg, tc_e, ep, 0.05)
            orc32.train_epoch("transe", st, (h, rel, t), (np.asarray(P[3]), np.asarray(P[4])), tc_o, ep, 0.05)
            ge, gr, _, _ = eng.store_download()
            assert np.array_equal(ge, st.entity) and np.array_equal(gr, st.relation), ep
        hits1, miss1 = eng.upload_stats()
        assert (hits1 - hits0, miss1 - miss0) == (1, 1)
        assert eng.upload_bytes() - bytes0 == 2 * 5 * m * wire  # uint16 / int32 on the wire
    finally:
        eng.set_deferred_uploads(False)
