"""Pins the CPU oracle against the reference's own known-answer tests.

Each test names the reference test it restates (paths under
/root/reference/proj/tests). The oracle is only trusted as the parity checker
for the CUDA engine because these pass. CPU only.
"""
import math

import numpy as np
import pytest

from oracle.oracle import OracleError, Store


def one(h, r, t):
    return np.array([h]), np.array([r]), np.array([t])


# ---------------------------------------------------------------- RNG KATs
def test_mt19937_64_kat(orc64):
    # C++ standard [rand.predef]: 10000th output of default-seeded mt19937_64.
    assert orc64.mt19937_64_nth(5489, 9999) == 9981545732273789042


def test_negative_sample_toy_vector(orc64):
    # SURVEY §8c derived vector: N=10, seed 7, heads {0,1,2,3}, tails {5,6,7,8}
    # -> corrupt tail->9, head->9, head->0, tail->9.
    h, t = np.array([0, 1, 2, 3]), np.array([5, 6, 7, 8])
    nh, nt = orc64.negative_sample(h, np.zeros(4, np.int64), t, 10, 1, 7)
    assert nh.tolist() == [0, 9, 0, 3]
    assert nt.tolist() == [9, 6, 7, 9]


# ------------------------------------------------ incidence (test_incidence.cpp)
def test_build_ht_one_triple(orc64):  # test_incidence.cpp:30-37
    rp, col, val = orc64.build_incidence("ht", *one(5, 0, 15), 22, 1)
    assert rp.tolist() == [0, 2] and col.tolist() == [5, 15] and val.tolist() == [1.0, -1.0]


def test_build_ht_self_loop_cancels(orc64):  # :39-45
    rp, col, val = orc64.build_incidence("ht", *one(3, 0, 3), 8, 1)
    assert rp.tolist() == [0, 0] and len(col) == 0


def test_build_hrt_relation_offset(orc64):  # :58-64
    rp, col, val = orc64.build_incidence("hrt", *one(5, 2, 15), 20, 3)
    assert col.tolist() == [5, 15, 22] and val.tolist() == [1.0, -1.0, 1.0]


def test_build_hrt_self_loop_keeps_relation(orc64):  # :66-77
    n, k, j = 7, 4, 1
    rp, col, val = orc64.build_incidence("hrt", *one(k, j, k), n, 3)
    assert rp.tolist() == [0, 1] and col.tolist() == [n + j] and val.tolist() == [1.0]
    x = np.random.default_rng(6).uniform(-1, 1, (n + 3, 4))
    z = orc64.spmm(1, n + 3, rp, col, val, x)
    assert np.array_equal(z[0], x[n + j])


def test_build_hrt_rows_equal_gathered(orc64):  # :79-95
    rng = np.random.default_rng(43)
    m, n, r, d = 16, 10, 4, 6
    h = rng.integers(0, n, m)
    t = (h + rng.integers(1, n, m)) % n
    rel = rng.integers(0, r, m)
    rp, col, val = orc64.build_incidence("hrt", h, rel, t, n, r)
    assert rp[-1] == 3 * m
    x = rng.uniform(-1, 1, (n + r, d))
    z = orc64.spmm(m, n + r, rp, col, val, x)
    np.testing.assert_allclose(z, x[h] + x[n + rel] - x[t], atol=1e-12)


def test_incidence_nnz_and_density(orc64):  # :97-110
    rng = np.random.default_rng(2)
    n, r = 30, 5
    m = 8 + int(rng.integers(0, 20))
    h = rng.integers(0, n, m)
    t = (h + rng.integers(1, n, m)) % n
    rel = rng.integers(0, r, m)
    assert orc64.build_incidence("ht", h, rel, t, n, r)[0][-1] == 2 * m
    assert orc64.build_incidence("hrt", h, rel, t, n, r)[0][-1] == 3 * m


def test_validation_rejects_bad_ids(orc64):  # :134-145
    with pytest.raises(OracleError) as e:
        orc64.build_incidence("ht", *one(3, 0, 0), 3, 1)
    assert e.value.kind == "ShapeError"
    with pytest.raises(OracleError) as e:
        orc64.build_incidence("hrt", *one(0, 2, 1), 3, 2)
    assert e.value.kind == "ShapeError"


# ------------------------------------------------------- sparse (test_sparse.cpp)
def test_coo_to_csr_goldens(orc64):  # test_sparse.cpp:60-93
    rp, c, v = orc64.coo_to_csr(3, 3, [], [], [])
    assert rp.tolist() == [0, 0, 0, 0] and len(c) == 0
    rp, c, v = orc64.coo_to_csr(2, 3, [0, 0, 1], [2, 0, 1], [1.0, 1.0, -1.0])
    assert rp.tolist() == [0, 2, 3] and c.tolist() == [0, 2, 1] and v.tolist() == [1, 1, -1]
    rp, c, v = orc64.coo_to_csr(1, 2, [0, 0], [1, 1], [1.0, -1.0])
    assert rp.tolist() == [0, 0]
    rp, c, v = orc64.coo_to_csr(1, 3, [0, 0, 0], [1, 0, 1], [2.5, 1.0, 1.5])
    assert c.tolist() == [0, 1] and v.tolist() == [1.0, 4.0]
    for rows, cols in (([0], [3]), ([2], [0])):
        with pytest.raises(OracleError) as e:
            orc64.coo_to_csr(2, 3, rows, cols, [1.0])
        assert e.value.kind == "ShapeError"


def test_transpose_worked_example(orc64):  # :114-147
    rp, c, v = orc64.coo_to_csr(2, 3, [0, 0, 1], [0, 2, 1], [1.0, -1.0, 1.0])
    trp, tc, tv = orc64.transpose(2, 3, rp, c, v)
    assert trp.tolist() == [0, 1, 2, 3] and tc.tolist() == [0, 1, 0] and tv.tolist() == [1, 1, -1]


def test_spmm_worked_examples(orc64):  # :156-163, :245-257
    rp, c, v = orc64.coo_to_csr(2, 3, [0, 0, 1], [0, 2, 1], [1.0, -1.0, 1.0])
    x = np.array([[1, 2], [3, 4], [5, 6]], float)
    assert orc64.spmm(2, 3, rp, c, v, x).tolist() == [[-4, -4], [3, 4]]
    rp, c, v = orc64.coo_to_csr(1, 3, [0, 0], [0, 2], [1.0, -1.0])
    sink = np.zeros((3, 2))
    orc64.spmm_transpose_add(1, 3, rp, c, v, np.ones((1, 2)), sink)
    assert sink.tolist() == [[1, 1], [0, 0], [-1, -1]]


def test_adjoint_identity(orc64):  # :279-292
    rng = np.random.default_rng(80)
    for _ in range(20):
        m, k = (int(x) for x in rng.integers(1, 33, 2))
        d = int(rng.integers(1, 9))
        mask = rng.random((m, k)) < 0.3
        ri, ci = np.nonzero(mask)
        vi = rng.uniform(0.5, 2, len(ri)) * np.where(rng.random(len(ri)) < 0.5, 1, -1)
        rp, c, v = orc64.coo_to_csr(m, k, ri, ci, vi)
        x, g = rng.uniform(-1, 1, (k, d)), rng.uniform(-1, 1, (m, d))
        lhs = float((orc64.spmm(m, k, rp, c, v, x) * g).sum())
        at_g = orc64.spmm_transpose_add(m, k, rp, c, v, g, np.zeros((k, d)))
        rhs = float((x * at_g).sum())
        assert abs(lhs - rhs) / max(1, abs(lhs), abs(rhs)) < 1e-10


def test_thread_count_bitwise_invariance(orc64):  # :314-329
    rng = np.random.default_rng(11)
    ri, ci = np.nonzero(rng.random((200, 64)) < 0.05)
    rp, c, v = orc64.coo_to_csr(200, 64, ri, ci, rng.uniform(0.5, 2, len(ri)))
    x, g = rng.uniform(-1, 1, (64, 16)), rng.uniform(-1, 1, (200, 16))
    orc64.set_num_threads(1)
    z1 = orc64.spmm(200, 64, rp, c, v, x)
    y1 = orc64.spmm_transpose_add(200, 64, rp, c, v, g, np.zeros((64, 16)))
    for t in (2, 5):
        orc64.set_num_threads(t)
        assert np.array_equal(orc64.spmm(200, 64, rp, c, v, x), z1)
        assert np.array_equal(orc64.spmm_transpose_add(200, 64, rp, c, v, g, np.zeros((64, 16))), y1)
    orc64.set_num_threads(1)


# ------------------------------------------------------ models (test_models.cpp)
def mk(ent, rel, proj=None, normals=None, dt=np.float64):
    a = lambda x: None if x is None else np.ascontiguousarray(x, dtype=dt)
    return Store(a(ent), a(rel), a(proj), a(normals))


@pytest.mark.parametrize("norm", ["l2", "l1"])
def test_transe_perfect_translation_zero(orc64, norm):  # test_models.cpp:54-61
    s = mk([[1, 0], [1, 1]], [[0, 1]])
    assert orc64.score_batch("transe", s, *one(0, 0, 1), norm=norm)[0][0] == 0.0


def test_transe_sqrt5_and_l1_3(orc64):  # :63-70
    s = mk([[1, 2], [0, 0]], [[0, 0]])
    assert orc64.score_batch("transe", s, *one(0, 0, 1), norm="l2")[0][0] == math.sqrt(5)
    assert orc64.score_batch("transe", s, *one(0, 0, 1), norm="l1")[0][0] == 3.0


def test_transe_l2_direction(orc64):  # :72-88
    s = mk([[3, 4], [0, 0]], [[0, 0]])
    assert orc64.score_batch("transe", s, *one(0, 0, 1))[0][0] == 5.0
    g = orc64.score_backward("transe", s, *one(0, 0, 1), [1.0], s.zeros_like())
    np.testing.assert_allclose(g.entity, [[0.6, 0.8], [-0.6, -0.8]], atol=1e-12)
    np.testing.assert_allclose(g.relation, [[0.6, 0.8]], atol=1e-12)


def test_transe_l1_sign_zero_at_kink(orc64):  # :90-102
    s = mk([[3, -4, 0], [0, 0, 0]], [[0, 0, 0]])
    g = orc64.score_backward("transe", s, *one(0, 0, 1), [1.0], s.zeros_like(), norm="l1")
    assert g.relation.tolist() == [[1.0, -1.0, 0.0]]


def test_transr_identity_equals_transe_bitwise(orc64):  # :104-112
    st = orc64.init_store("transr", 12, 4, 5, 5, 41)
    rng = np.random.default_rng(41)
    h = rng.integers(0, 12, 20)
    t = (h + rng.integers(1, 12, 20)) % 12
    r = rng.integers(0, 4, 20)
    a = orc64.score_batch("transr", st, h, r, t)[0]
    b = orc64.score_batch("transe", Store(st.entity, st.relation), h, r, t)[0]
    assert np.array_equal(a, b)


def test_transr_zero_projection(orc64):  # :114-121
    st = orc64.init_store("transr", 4, 1, 3, 2, 1)
    st.proj[:] = 0
    st.relation[:] = [[3, 4]]
    assert orc64.score_batch("transr", st, *one(0, 0, 2))[0][0] == 5.0


def test_transh_goldens(orc64):  # :123-137
    s = mk([[1, 2, 0], [0, 0, 0]], [[0.5, -1, 0]], normals=[[0, 0, 1]])
    assert orc64.score_batch("transh", s, *one(0, 0, 1))[0][0] == math.sqrt(1.5 * 1.5 + 1.0)
    s = mk([[2, 0], [0, 0]], [[0, 0]], normals=[[1, 0]])
    assert orc64.score_batch("transh", s, *one(0, 0, 1))[0][0] == 0.0


def test_toruse_goldens(orc64):  # :139-150
    s = mk([[0.75], [0]], [[0]])
    assert orc64.score_batch("toruse", s, *one(0, 0, 1), norm="l2")[0][0] == 0.0625
    assert orc64.score_batch("toruse", s, *one(0, 0, 1), norm="l1")[0][0] == 0.25
    s = mk([[1.5], [0]], [[0]])
    assert orc64.score_batch("toruse", s, *one(0, 0, 1), norm="l2")[0][0] == 0.25
    assert orc64.score_batch("toruse", s, *one(0, 0, 1), norm="l1")[0][0] == 0.5


def test_toruse_integer_shift_invariance(orc64):  # :152-172
    rng = np.random.default_rng(7)
    n, nr, d = 8, 3, 4
    ent = np.round(rng.uniform(-1, 1, (n, d)) * 64) / 64
    rel = np.round(rng.uniform(-1, 1, (nr, d)) * 64) / 64
    h, r, t = rng.integers(0, n, 12), rng.integers(0, nr, 12), rng.integers(0, n, 12)
    base = orc64.score_batch("toruse", mk(ent, rel), h, r, t)[0]
    shifted = orc64.score_batch("toruse", mk(ent + rng.integers(-3, 4, ent.shape),
                                             rel + rng.integers(-3, 4, rel.shape)), h, r, t)[0]
    assert np.array_equal(base, shifted)


def _numeric_grad(f, x, step=1e-6):
    g = np.zeros_like(x)
    for idx in np.ndindex(x.shape):
        keep = x[idx]
        x[idx] = keep + step
        fp = f()
        x[idx] = keep - step
        fm = f()
        x[idx] = keep
        g[idx] = (fp - fm) / (2 * step)
    return g


def _max_rel_err(a, b):  # test_util.hpp:102-113
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


@pytest.mark.parametrize("model,de,dr", [("transe", 3, 3), ("transr", 3, 2), ("transh", 3, 3), ("toruse", 3, 3)])
@pytest.mark.parametrize("norm", ["l2", "l1"])
def test_finite_differences(orc64, model, de, dr, norm):  # test_models.cpp:372-410
    n, nr, m = 5, 2, 4
    for seed in range(1000, 1500):
        st = orc64.init_store(model, n, nr, de, dr, seed)
        rng = np.random.default_rng(seed * 13 + 1)
        h, r, t = rng.integers(0, n, m), rng.integers(0, nr, m), rng.integers(0, n, m)
        h[0] = t[0] = 0
        sc, aux = orc64.score_batch(model, st, h, r, t, norm=norm)
        if model == "toruse":
            a = np.abs(aux["delta"])
            if (a > 0.45).any() or (norm == "l1" and (a < 1e-3).any()):
                continue
        elif norm == "l1":
            if (np.abs(aux["v"]) <= 1e-3).any():
                continue
        elif (np.linalg.norm(aux["v"], axis=1) < 1e-2).any():
            continue
        break
    up = rng.uniform(0.25, 1, m) * np.where(np.arange(m) % 2, 1, -1)
    g = orc64.score_backward(model, st, h, r, t, up, st.zeros_like(), norm=norm)
    f = lambda: float(up @ orc64.score_batch(model, st, h, r, t, norm=norm)[0])
    for name in ("entity", "relation", "proj", "normals"):
        if getattr(st, name) is not None:
            assert _max_rel_err(getattr(g, name), _numeric_grad(f, getattr(st, name))) < 1e-5, name


def test_config_errors(orc64):  # :438-460
    st = orc64.init_store("transe", 5, 2, 4, 4, 1)
    for model in ("transr", "transh"):  # missing per-model tables
        with pytest.raises(OracleError) as e:
            orc64.score_batch(model, st, *one(0, 0, 1))
        assert e.value.kind == "ConfigError"
    with pytest.raises(OracleError) as e:  # non-projection models need d_e == d_r
        orc64.score_batch("transe", Store(st.entity, np.zeros((2, 3))), *one(0, 0, 1))
    assert e.value.kind == "ConfigError"
    with pytest.raises(OracleError) as e:  # out-of-range ids
        orc64.score_batch("transe", st, *one(0, 0, 7))
    assert e.value.kind == "ShapeError"


# ---------------------------------------------------- loss (test_training.cpp)
def test_margin_ranking_loss_goldens(orc64):  # test_training.cpp:103-136
    loss, dp, dn = orc64.margin_ranking_loss([0.2], [1.0], 0.5)
    assert loss == 0.0 and dp[0] == 0.0 and dn[0] == 0.0
    loss, dp, dn = orc64.margin_ranking_loss([1.0], [0.2], 0.5)
    assert abs(loss - 1.3) < 1e-15 and dp[0] == 1.0 and dn[0] == -1.0
    loss, dp, _ = orc64.margin_ranking_loss([0.7], [0.7], 0.0)
    assert loss == 0.0 and dp[0] == 0.0
    loss, dp, dn = orc64.margin_ranking_loss([1.0, 0.0], [0.2, 5.0], 0.5)
    assert abs(loss - 0.65) < 1e-15 and dp.tolist() == [0.5, 0.0] and dn[0] == -0.5
    with pytest.raises(OracleError):
        orc64.margin_ranking_loss([1.0, 0.0], [1, 2, 3], 0.5)


# ------------------------------------------------- sgd (test_embedding.cpp)
def test_sgd_goldens(orc64):  # test_embedding.cpp:128-207
    s = mk([[1.0]], [[0.0]])
    g = s.zeros_like()
    g.entity[0, 0] = 2.0
    orc64.sgd_step(s, g, 0.1)
    assert abs(s.entity[0, 0] - 0.8) < 1e-15
    s = orc64.init_store("transr", 6, 2, 5, 3, 21)
    before = s.copy()
    orc64.sgd_step(s, s.zeros_like(), 0.5)
    assert np.array_equal(s.entity, before.entity) and np.array_equal(s.proj, before.proj)
    s = orc64.init_store("transr", 4, 2, 3, 3, 2)
    before = s.copy()
    g = s.zeros_like()
    for a in (g.entity, g.relation, g.proj):
        a[:] = 1.0
    orc64.sgd_step(s, g, 0.25)
    assert np.array_equal(before.entity - s.entity, np.full((4, 3), 0.25))
    assert np.array_equal(before.proj - s.proj, np.full((2, 9), 0.25))
    s = orc64.init_store("transh", 5, 3, 8, 8, 13)
    g = s.zeros_like()
    g.normals[:] = np.random.default_rng(99).uniform(-1, 1, (3, 8))
    orc64.sgd_step(s, g, 0.3)
    assert np.allclose(np.linalg.norm(s.normals, axis=1), 1.0, atol=1e-12)
    s = orc64.init_store("transe", 3, 2, 4, 4, 1)
    for bad in (np.nan, np.inf):
        g = s.zeros_like()
        g.entity[1, 2] = bad
        with pytest.raises(OracleError) as e:
            orc64.sgd_step(s, g, 0.1)
        assert e.value.kind == "TrainingError"


def test_renormalize_entities(orc64):  # test_embedding.cpp:209-218
    s = mk([[3, 4], [0, 0], [0.5, 0]], [[0, 0]])
    orc64.renormalize_entities(s)
    assert np.allclose(s.entity, [[0.6, 0.8], [0, 0], [1, 0]], atol=1e-15)


def test_init_store_properties(orc64):  # test_embedding.cpp:24-78
    a = orc64.init_store("transe", 40, 6, 16, 16, 7)
    b = orc64.init_store("transe", 40, 6, 16, 16, 7)
    c = orc64.init_store("transe", 40, 6, 16, 16, 8)
    assert np.array_equal(a.entity, b.entity) and not np.array_equal(a.entity, c.entity)
    bound = 6 / math.sqrt(16)
    assert np.abs(a.entity).max() <= bound and np.abs(a.entity).max() > 0.5 * bound
    p = orc64.init_store("transr", 10, 3, 4, 3, 5).proj.reshape(3, 3, 4)
    assert np.array_equal(p[1], np.eye(3, 4))
    n = orc64.init_store("transh", 12, 9, 24, 24, 17).normals
    assert np.allclose(np.linalg.norm(n, axis=1), 1, atol=1e-12)


# ------------------------------------------------ trainer (test_training.cpp)
def _rand_batch(rng, m, n, r, self_loops=False):
    h = rng.integers(0, n, m)
    t = rng.integers(0, n, m) if self_loops else (h + rng.integers(1, n, m)) % n
    return h, rng.integers(0, r, m), t


def test_negative_sample_properties(orc64):  # test_training.cpp:25-101
    rng = np.random.default_rng(3)
    h, r, t = _rand_batch(rng, 500, 40, 6, True)
    nh, nt = orc64.negative_sample(h, r, t, 40, 6, 11)
    assert ((nh != h) != (nt != t)).all()
    assert ((0 <= nh) & (nh < 40) & (0 <= nt) & (nt < 40)).all()
    for seed in range(8):
        nh, nt = orc64.negative_sample([0], [0], [1], 2, 1, seed)
        assert (nh[0] == 1) or (nt[0] == 0)
    h, r, t = _rand_batch(rng, 100000, 50, 5, True)
    nh, nt = orc64.negative_sample(h, r, t, 50, 5, 123)
    assert 0.49 < (nh != h).mean() < 0.51
    h, r, t = _rand_batch(rng, 5000, 12, 3)
    nh, nt = orc64.negative_sample(h, r, t, 12, 3, 77, avoid_self_loops=True)
    assert (nh != nt).all()
    for n, avoid in ((1, False), (2, True)):
        with pytest.raises(OracleError) as e:
            orc64.negative_sample([0], [0], [n - 1], n, 1, 0, avoid_self_loops=avoid)
        assert e.value.kind == "ConfigError"


def test_lr0_freezes_and_determinism(orc32):  # test_training.cpp:151-164, 209-224
    o = orc32
    st = o.init_store("transe", 20, 4, 8, 8, 5)
    before = st.copy()
    rng = np.random.default_rng(5)
    h, r, t = _rand_batch(rng, 100, 20, 4)
    nh, nt = o.negative_sample(h, r, t, 20, 4, 6)
    tc = o.train_config(batch_size=32, margin=1.0)
    rep = o.train_epoch("transe", st, (h, r, t), (nh, nt), tc, 0, 0.0)
    assert np.array_equal(st.entity, before.entity) and rep.loss > 0
    tc = o.train_config(lr=0.05, epochs=5, batch_size=32, seed=99)
    s1, s2 = o.init_store("transe", 25, 5, 8, 8, 1), o.init_store("transe", 25, 5, 8, 8, 1)
    h, r, t = _rand_batch(rng, 120, 25, 5)
    r1 = o.fit("transe", s1, h, r, t, tc)
    r2 = o.fit("transe", s2, h, r, t, tc)
    assert [x.loss for x in r1] == [x.loss for x in r2] and np.array_equal(s1.entity, s2.entity)


def test_scheduler_replay(orc32):  # test_training.cpp:244-266
    o = orc32
    rng = np.random.default_rng(15)
    h, r, t = _rand_batch(rng, 60, 12, 3)
    tc = o.train_config(lr=0.2, epochs=2, batch_size=20, seed=5, scheduler=(1, 0.5))
    s1, s2 = o.init_store("transe", 12, 3, 4, 4, 2), o.init_store("transe", 12, 3, 4, 4, 2)
    run = o.fit("transe", s1, h, r, t, tc)
    nh, nt = o.negative_sample(h, r, t, 12, 3, 5)
    e0 = o.train_epoch("transe", s2, (h, r, t), (nh, nt), tc, 0, 0.2)
    e1 = o.train_epoch("transe", s2, (h, r, t), (nh, nt), tc, 1, 0.1)
    assert run[0].loss == e0.loss and run[1].loss == e1.loss
    assert np.array_equal(s1.entity, s2.entity)


def test_lattice_loss_drops(orc32):  # test_training.cpp:322-339
    o = orc32
    h, r, t = o.synthetic_train(125, 6, 150, 18)
    tc = o.train_config(lr=0.1, margin=0.5, epochs=100, batch_size=16, seed=20)
    st = o.init_store("transe", 125, 6, 16, 16, 6)
    run = [x.loss for x in o.fit("transe", st, h, r, t, tc)]
    assert np.mean(run[-5:]) < 0.5 * np.mean(run[:5])


def test_shuffle_is_a_permutation(orc64):  # training.cpp:106-112
    for m in (1, 2, 3, 10, 11, 1000):
        o = orc64.epoch_order(m, 42, 3)
        assert sorted(o.tolist()) == list(range(m))
    assert orc64.epoch_order(10, 1, 0, shuffle=False).tolist() == list(range(10))


# ---- link prediction (test_eval.cpp), the oracle's rank_entity restatement
def _plane_store(orc):  # test_eval.cpp:47-53
    st = orc.init_store("transe", 5, 1, 2, 2, 0)
    st.entity[:] = np.array([[0, 0], [0, 1], [1, 0], [2, 0], [0.5, 0]])
    st.relation[:] = np.array([[1, 0]])
    return st


def test_rank_entity_goldens(orc64):  # test_eval.cpp:55-79
    st = _plane_store(orc64)
    assert orc64.rank_entities("transe", st, [0], [0], [3])[0, 0] == 3
    filt = ([0, 0, 0], [0, 0, 0], [2, 4, 3])  # the query itself stays eligible
    assert orc64.rank_entities("transe", st, [0], [0], [3], filt=filt)[0, 0] == 1
    tie = orc64.init_store("transe", 6, 1, 3, 3, 0)
    tie.entity[:] = 0.25
    tie.relation[:] = 0.0
    assert (orc64.rank_entities("transe", tie, [0], [0], [4]) == 1).all()


def test_evaluate_mrr_0625(orc64):  # test_eval.cpp:87-101: ranks 1 (tail) and 4 (head)
    st = orc64.init_store("transe", 5, 1, 2, 2, 0)
    st.entity[:] = np.array([[0, 0], [-0.4, 0], [-0.6, 0], [-0.5, 0.1], [0.5, 0]])
    st.relation[:] = np.array([[1, 0]])
    rk = orc64.rank_entities("transe", st, [0], [0], [4])
    assert rk.tolist() == [[1, 4]]
    assert abs(np.mean(1.0 / rk) - 0.625) < 1e-12


def test_evaluate_exact_translations(orc64):  # test_eval.cpp:103-115
    st = orc64.init_store("transe", 4, 1, 2, 2, 0)
    st.entity[:] = np.array([[0, 0], [1, 0], [0, 1], [1, 1]])
    st.relation[:] = np.array([[1, 0]])
    assert (orc64.rank_entities("transe", st, [0, 2], [0, 0], [1, 3]) == 1).all()


def test_rank_entity_rejects_bad_ids(orc64):  # test_eval.cpp:81-85
    st = _plane_store(orc64)
    with pytest.raises(Exception):
        orc64.rank_entities("transe", st, [0], [0], [9])
    with pytest.raises(Exception):
        orc64.rank_entities("transe", st, [0], [3], [1])


# ---------------------------- multiplicative family (test_models.cpp:174-230)
def cstore(ent, rel):
    """Complex store from complex arrays: interleaved (re, im) float64 tables."""
    f = lambda a: np.ascontiguousarray(np.asarray(a, np.complex128)).view(np.float64).reshape(len(a), -1).copy()
    return Store(f(ent), f(rel))


def test_build_multiplicative_layout(orc64):  # incidence.hpp:93-121
    rp, col, val = orc64.build_incidence("mult", *one(5, 2, 3), 20, 4)
    assert col.tolist() == [3, 5, 22] and val.tolist() == [1.0, 1.0, 1.0]
    rp, col, val = orc64.build_incidence("mult_conj", *one(5, 2, 3), 20, 4)
    assert col.tolist() == [3, 5, 22] and val.tolist() == [-1.0, 1.0, 1.0]
    with pytest.raises(OracleError) as e:
        orc64.build_incidence("mult", *one(4, 0, 4), 20, 4)
    assert e.value.kind == "DegenerateTripleError" and "triple 0: head == tail" in e.value.msg


def test_distmult_golden_and_symmetry(orc64):  # test_models.cpp:174-189
    st = Store(np.array([[2.0], [5.0]]), np.array([[3.0]]))
    assert orc64.score_batch("distmult", st, *one(0, 0, 1))[0][0] == 30.0
    st = orc64.init_store("distmult", 10, 3, 6, 6, 19)
    rng = np.random.default_rng(19)
    h, r, t = rng.integers(0, 10, 15), rng.integers(0, 3, 15), rng.integers(0, 10, 15)
    t = np.where(t == h, (t + 1) % 10, t)
    a = orc64.score_batch("distmult", st, h, r, t)[0]
    b = orc64.score_batch("distmult", st, t, r, h)[0]
    assert np.array_equal(a, b)


def test_complex_tail_conjugated(orc64):  # :191-198
    st = cstore([[1j], [1j]], [[1.0]])
    assert orc64.score_batch("complex", st, *one(0, 0, 1))[0][0] == 1.0


def test_rotate_goldens(orc64):  # :200-211
    st = cstore([[1.0], [1j]], [[1j]])
    assert orc64.score_batch("rotate", st, *one(0, 0, 1))[0][0] == 0.0
    st.entity[1] = 0.0
    assert orc64.score_batch("rotate", st, *one(0, 0, 1))[0][0] == 1.0


@pytest.mark.parametrize("model", ["distmult", "complex", "rotate"])
def test_multiplicative_rejects_self_loops(orc64, model):  # :213-221
    st = orc64.init_store(model, 5, 2, 3, 3, 1)
    with pytest.raises(OracleError) as e:
        orc64.score_batch(model, st, *one(2, 0, 2))
    assert e.value.kind == "DegenerateTripleError"


@pytest.mark.parametrize("model", ["distmult", "complex", "rotate"])
def test_finite_differences_product_family(orc64, model):  # test_models.cpp:414-433
    n, nr, m = 5, 2, 4
    for seed in range(5000, 5500):
        st = orc64.init_store(model, n, nr, 3, 3, seed)
        rng = np.random.default_rng(seed * 13 + 1)
        h, r, t = rng.integers(0, n, m), rng.integers(0, nr, m), rng.integers(0, n, m)
        t = np.where(t == h, (t + 1) % n, t)
        sc, aux = orc64.score_batch(model, st, h, r, t)
        if model == "rotate":  # modulus gradient needs |q| clear of the origin
            q = aux["v"].view(np.complex128)
            if (np.abs(q) < 1e-2).any():
                continue
        break
    up = rng.uniform(0.25, 1, m) * np.where(np.arange(m) % 2, 1, -1)
    g = orc64.score_backward(model, st, h, r, t, up, st.zeros_like())
    f = lambda: float(up @ orc64.score_batch(model, st, h, r, t)[0])
    for name in ("entity", "relation"):
        assert _max_rel_err(getattr(g, name), _numeric_grad(f, getattr(st, name))) < 1e-5, name


def test_polarity_and_fit_product_family(orc64):  # test_models.cpp:223-231, test_training.cpp:290-320
    rng = np.random.default_rng(12)
    h, r, t = rng.integers(0, 10, 40), rng.integers(0, 3, 40), rng.integers(0, 10, 40)
    t = np.where(t == h, (t + 1) % 10, t)
    tc = orc64.train_config(lr=0.01, epochs=2, batch_size=16, seed=12)
    for model in ("distmult", "complex", "rotate"):
        st = orc64.init_store(model, 10, 3, 6, 6, 3)
        reps = orc64.fit(model, st, h, r, t, tc)
        assert len(reps) == 2 and math.isfinite(reps[-1].loss)
    # DistMult scores plausibility: the hinge sees -score (energy_sign = -1)
    st = Store(np.array([[1.0], [1.0], [3.0]]), np.array([[1.0]]))
    tc1 = orc64.train_config(lr=0.0, epochs=1, batch_size=4, seed=1, shuffle=False)
    rep = orc64.train_epoch("distmult", st, one(0, 0, 1), (np.array([0]), np.array([2])), tc1, 0, 0.0)
    # pos score 1, neg score 3: energies -1 and -3 -> term = 0.5 + (-1) - (-3) = 2.5
    assert rep.loss == 2.5


def test_complex_init_bound(orc64):  # test_embedding.cpp:44-53
    d = 8
    st = orc64.init_store("complex", 30, 4, d, d, 11)
    assert st.entity.shape == (30, 2 * d)
    assert (np.abs(st.entity) <= 6 / math.sqrt(d)).all()
    # draws: re then im per coordinate, entity then relation (embedding.cpp:17-30)
    real = orc64.init_store("distmult", 30, 4, 2 * d, 2 * d, 11)
    assert not np.array_equal(real.entity, st.entity)  # bound differs (6/sqrt(2d))
    assert np.allclose(real.entity * math.sqrt(2 * d), st.entity * math.sqrt(d))


def test_degenerate_multiplicative_queries_rank_last(orc64):  # test_eval.cpp:185-197
    st = orc64.init_store("distmult", 5, 1, 3, 3, 4)
    assert orc64.rank_entities("distmult", st, [2], [0], [2]).tolist() == [[5, 5]]
    r = orc64.rank_entities("distmult", st, [2], [0], [1])[0, 0]
    assert 1 <= r <= 4
