"""The reference's generic sparse layer on device (skg_coo_to_csr, skg_csr_transpose,
skg_spmm, skg_spmm_transpose_add) vs the oracle, bit for bit, plus the known-answer
cases of test_sparse.cpp (restated; line numbers cite the reference test)."""
import numpy as np
import pytest

from paper_2502_16949_b200 import Engine, EngineError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    e = Engine(0)
    yield e
    e.close()


def random_coo(rng, rows, cols, density, dups=True):
    """test_util.hpp:44-58 shape: values bounded away from zero, plus injected duplicates
    (one of them an exact cancellation) like test_sparse.cpp:92-112."""
    mask = rng.random((rows, cols)) < density
    ri, ci = np.nonzero(mask)
    v = rng.uniform(0.5, 2.0, len(ri)) * np.where(rng.random(len(ri)) < 0.5, 1, -1)
    ri, ci, v = list(ri), list(ci), list(v.astype(np.float32))
    if dups and len(ri) >= 2:
        ri += [ri[0], ri[1]]
        ci += [ci[0], ci[1]]
        v += [np.float32(0.75), np.float32(-v[1])]
    perm = rng.permutation(len(ri))  # arbitrary input order
    return (np.array(ri, np.int64)[perm], np.array(ci, np.int64)[perm], np.array(v, np.float32)[perm])


def test_coo_to_csr_goldens(eng):
    rp, c, v = eng.coo_to_csr(3, 3, [], [], [])  # test_sparse.cpp:60-67
    assert rp.tolist() == [0, 0, 0, 0] and len(c) == 0
    rp, c, v = eng.coo_to_csr(2, 3, [0, 0, 1], [2, 0, 1], [1, 1, -1])  # :69-76
    assert rp.tolist() == [0, 2, 3] and c.tolist() == [0, 2, 1] and v.tolist() == [1, 1, -1]
    rp, c, v = eng.coo_to_csr(1, 2, [0, 0], [1, 1], [1, -1])  # :78-82 exact cancellation
    assert rp.tolist() == [0, 0] and len(c) == 0
    rp, c, v = eng.coo_to_csr(1, 3, [0, 0, 0], [1, 0, 1], [2.5, 1.0, 1.5])  # :84-88
    assert c.tolist() == [0, 1] and v.tolist() == [1.0, 4.0]
    for bad in (([0], [3]), ([2], [0])):  # :90-93
        with pytest.raises(EngineError) as e:
            eng.coo_to_csr(2, 3, bad[0], bad[1], [1.0])
        assert e.value.kind == "ShapeError" and e.value.msg == "coo: entry 0 outside declared shape"


@pytest.mark.parametrize("seed", range(8))
def test_coo_to_csr_matches_oracle(eng, orc32, seed):
    rng = np.random.default_rng(seed)
    rows, cols = (13, 17) if seed < 6 else (400, 300)
    ri, ci, v = random_coo(rng, rows, cols, 0.2 if seed < 6 else 0.01)
    g = eng.coo_to_csr(rows, cols, ri, ci, v)
    o = orc32.coo_to_csr(rows, cols, ri, ci, v)
    for a, b in zip(g, o):
        assert np.array_equal(a, b)


def test_transpose_goldens_and_involution(eng, orc32):
    rp, c, v = eng.transpose(2, 3, [0, 2, 3], [0, 2, 1], [1, -1, 1])  # test_sparse.cpp:122-130
    assert rp.tolist() == [0, 1, 2, 3] and c.tolist() == [0, 1, 0] and v.tolist() == [1, 1, -1]
    rp, c, v = eng.transpose(3, 5, [0, 0, 0, 0], [], [])  # :132-138
    assert rp.tolist() == [0] * 6 and len(c) == 0
    for seed in range(6):  # :140-147
        rng = np.random.default_rng(seed + 100)
        a = orc32.coo_to_csr(9, 14, *random_coo(rng, 9, 14, 0.25, dups=False))
        t = eng.transpose(9, 14, *a)
        assert all(np.array_equal(x, y) for x, y in zip(t, orc32.transpose(9, 14, *a)))
        tt = eng.transpose(14, 9, *t)
        assert all(np.array_equal(x, y) for x, y in zip(tt, a))


@pytest.mark.parametrize("seed", range(10))
def test_spmm_and_transpose_add_match_oracle(eng, orc32, seed):
    rng = np.random.default_rng(seed + 20)
    m, k, d = (int(rng.integers(1, 33)), int(rng.integers(1, 33)), int(rng.integers(1, 9)))
    if seed >= 8:  # longer rows (> 3 entries: the generic accumulation branch) and wide d
        m, k, d = 300, 200, 130
    a = orc32.coo_to_csr(m, k, *random_coo(rng, m, k, 0.3, dups=False))
    x = rng.uniform(-1, 1, (k, d)).astype(np.float32)
    g = rng.uniform(-1, 1, (m, d)).astype(np.float32)
    assert np.array_equal(eng.spmm(m, k, *a, x), orc32.spmm(m, k, *a, x))
    sink0 = rng.uniform(-1, 1, (k, d)).astype(np.float32)
    s_g, s_o = sink0.copy(), sink0.copy()
    eng.spmm_transpose_add(m, k, *a, g, s_g)
    orc32.spmm_transpose_add(m, k, *a, g, s_o)
    assert np.array_equal(s_g, s_o)


def test_spmm_goldens_and_errors(eng):
    a = ([0, 2, 3], [0, 2, 1], np.array([1, -1, 1], np.float32))  # test_sparse.cpp:156-163
    x = np.array([[1, 2], [3, 4], [5, 6]], np.float32)
    assert eng.spmm(2, 3, *a, x).tolist() == [[-4, -4], [3, 4]]
    z = eng.spmm(2, 3, [0, 1, 1], [1], np.array([1], np.float32), x)  # :188-196 empty row
    assert z[1].tolist() == [0, 0]
    sink = np.zeros((3, 2), np.float32)  # :245-257 A^T example
    eng.spmm_transpose_add(1, 3, [0, 2], [0, 2], np.array([1, -1], np.float32), np.ones((1, 2), np.float32), sink)
    assert sink.tolist() == [[1, 1], [0, 0], [-1, -1]]
    with pytest.raises(EngineError) as e:  # :198-204
        eng.spmm(2, 3, [0, 1, 1], [0], np.ones(1, np.float32), np.zeros((4, 2), np.float32))
    assert e.value.kind == "ShapeError" and e.value.msg == "spmm: inner dimensions 3 vs 4"
    with pytest.raises(EngineError) as e:
        eng.spmm_transpose_add(2, 3, [0, 1, 1], [0], np.ones(1, np.float32), np.zeros((3, 2), np.float32),
                               np.zeros((3, 2), np.float32))
    assert e.value.msg == "spmm_transpose: row count mismatch"


def test_incidence_through_the_generic_layer(eng, orc32):
    """build_hrt -> coo_to_csr -> spmm against the stacked table equals score residuals
    (the reference's transe_forward composition, models.cpp:11-30)."""
    rng = np.random.default_rng(4)
    n, r, m, d = 50, 6, 200, 16
    h, rel, t = rng.integers(0, n, m), rng.integers(0, r, m), rng.integers(0, n, m)
    h[:3] = t[:3]
    rows = np.repeat(np.arange(m), 3)
    cols = np.stack([h, t, n + rel], 1).ravel()
    vals = np.tile(np.array([1, -1, 1], np.float32), m)
    a = eng.coo_to_csr(m, n + r, rows, cols, vals)
    assert all(np.array_equal(x, y) for x, y in zip(a, eng.build_incidence("hrt", h, rel, t, n, r)))
    X = rng.uniform(-1, 1, (n + r, d)).astype(np.float32)
    assert np.array_equal(eng.spmm(m, n + r, *a, X), orc32.spmm(m, n + r, *a, X))
