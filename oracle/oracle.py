"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU parity oracle.

The oracle is a C++ restatement of the reference hot path (see
oracle/skge_oracle.hpp). Only tests/, __graft_entry__.smoke() and bench.py's
CPU legs (cpu_baseline, --impl reference) may import this module; the product
package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")

MODELS = {"transe": 0, "transr": 1, "transh": 2, "toruse": 3, "distmult": 4, "complex": 5, "rotate": 6}
COMPLEX = ("complex", "rotate")  # tables of interleaved (re, im) pairs: 2 * dim columns
NORMS = {"l1": 0, "l2": 1}
STATUS_NAMES = {1: "ShapeError", 2: "ConfigError", 3: "DegenerateTripleError",
                4: "TrainingError", 5: "ParseError", 7: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))
        self.msg = msg


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _ModelConfig(C.Structure):
    _fields_ = [("model", C.c_uint32), ("norm", C.c_uint32),
                ("dim_entity", C.c_int64), ("dim_relation", C.c_int64)]


class _EpochReport(C.Structure):
    _fields_ = [("epoch", C.c_int64), ("loss", C.c_double), ("t_forward_s", C.c_double),
                ("t_backward_s", C.c_double), ("t_step_s", C.c_double)]


def _store_struct(real):
    class _Store(C.Structure):
        _fields_ = [("num_entities", C.c_int64), ("num_relations", C.c_int64),
                    ("dim_entity", C.c_int64), ("dim_relation", C.c_int64),
                    ("entity", C.POINTER(real)), ("relation", C.POINTER(real)),
                    ("proj", C.POINTER(real)), ("normals", C.POINTER(real))]
    return _Store


def _train_struct(real):
    class _Train(C.Structure):
        _fields_ = [("lr", real), ("margin", real), ("epochs", C.c_int64),
                    ("batch_size", C.c_int64), ("seed", C.c_uint64),
                    ("has_scheduler", C.c_int32), ("decay_every", C.c_int64),
                    ("decay_factor", real), ("shuffle", C.c_int32),
                    ("resample_negatives", C.c_int32), ("renorm_entities", C.c_int32)]
    return _Train


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class Store:
    """Row-major numpy tables mirroring EmbeddingStoreT (embedding.hpp:15-31)."""

    def __init__(self, entity, relation, proj=None, normals=None):
        self.entity = entity
        self.relation = relation
        self.proj = proj
        self.normals = normals

    def copy(self):
        c = lambda a: None if a is None else a.copy()
        return Store(c(self.entity), c(self.relation), c(self.proj), c(self.normals))

    def zeros_like(self):
        z = lambda a: None if a is None else np.zeros_like(a)
        return Store(z(self.entity), z(self.relation), z(self.proj), z(self.normals))


class Oracle:
    def __init__(self, real: str = "f32"):
        path = os.path.join(BUILD, f"liboracle_{real}.so")
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        self.dtype = np.float32 if real == "f32" else np.float64
        self.real = C.c_float if real == "f32" else C.c_double
        self.Store = _store_struct(self.real)
        self.Train = _train_struct(self.real)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_mt19937_64_nth.restype = C.c_uint64
        L.orc_mt19937_64_nth.argtypes = [C.c_uint64, C.c_int64]
        for name in ["orc_generate_synthetic", "orc_init_store", "orc_negative_sample",
                     "orc_epoch_order", "orc_build_incidence", "orc_coo_to_csr", "orc_transpose",
                     "orc_spmm", "orc_spmm_transpose_add", "orc_score_batch", "orc_score_backward",
                     "orc_margin_ranking_loss", "orc_sgd_step", "orc_renormalize_entities",
                     "orc_train_epoch", "orc_train_batches", "orc_fit", "orc_rank_entities"]:
            getattr(L, name).restype = C.c_int
        L.orc_init_store.argtypes = [C.c_uint32, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_uint64] + [C.c_void_p] * 4
        L.orc_generate_synthetic.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64] + [C.c_void_p] * 3
        L.orc_negative_sample.argtypes = [C.c_int64] + [C.c_void_p] * 3 + [C.c_int64, C.c_int64,
                                                                          C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_epoch_order.argtypes = [C.c_int64, C.c_uint64, C.c_int, C.c_int64, C.c_void_p]
        L.orc_build_incidence.argtypes = [C.c_int, C.c_int64] + [C.c_void_p] * 3 + [C.c_int64, C.c_int64] + [C.c_void_p] * 4
        L.orc_coo_to_csr.argtypes = [C.c_int64, C.c_int64, C.c_int64] + [C.c_void_p] * 7
        L.orc_transpose.argtypes = [C.c_int64, C.c_int64] + [C.c_void_p] * 6
        L.orc_spmm.argtypes = [C.c_int64, C.c_int64] + [C.c_void_p] * 3 + [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_spmm_transpose_add.argtypes = [C.c_int64, C.c_int64] + [C.c_void_p] * 3 + [C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_margin_ranking_loss.argtypes = [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, self.real] + [C.c_void_p] * 3
        L.orc_sgd_step.argtypes = [C.c_void_p, C.c_void_p, self.real]
        L.orc_renormalize_entities.argtypes = [C.c_void_p]
        L.orc_score_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 7
        L.orc_score_backward.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 5
        L.orc_train_epoch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 6 + [
            C.c_int64, self.real, C.c_void_p]
        L.orc_train_batches.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 6 + [
            C.c_int64, self.real, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_fit.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 4
        L.orc_rank_entities.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 3 + [
            C.c_int, C.c_int64] + [C.c_void_p] * 4

    # ------------------------------------------------------------ plumbing
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    def set_num_threads(self, n: int):
        self.lib.orc_set_num_threads(int(n))

    def _f(self, a):
        return np.ascontiguousarray(a, dtype=self.dtype)

    def _store(self, s: Store):
        P = C.POINTER(self.real)
        cast = lambda a: a.ctypes.data_as(P) if a is not None else None
        for name in ("entity", "relation", "proj", "normals"):
            a = getattr(s, name)
            if a is not None:
                assert a.dtype == self.dtype and a.flags.c_contiguous, name
        return self.Store(s.entity.shape[0], s.relation.shape[0], s.entity.shape[1],
                          s.relation.shape[1], cast(s.entity), cast(s.relation),
                          cast(s.proj), cast(s.normals))

    @staticmethod
    def _cfg(model, de, dr, norm="l2"):
        return _ModelConfig(MODELS[model], NORMS[norm], de, dr)

    def _cfg_for(self, model, store, norm="l2"):
        w = 2 if model in COMPLEX else 1
        return self._cfg(model, store.entity.shape[1] // w, store.relation.shape[1] // w, norm)

    def train_config(self, lr=4e-4, margin=0.5, epochs=200, batch_size=1024, seed=0,
                     scheduler=None, shuffle=True, resample_negatives=False, renorm_entities=False):
        every, factor = scheduler if scheduler else (50, 0.5)
        return self.Train(lr, margin, epochs, batch_size, seed, 1 if scheduler else 0, every,
                          factor, int(shuffle), int(resample_negatives), int(renorm_entities))

    # ------------------------------------------------------------ API
    def mt19937_64_nth(self, seed, n):
        return int(self.lib.orc_mt19937_64_nth(seed, n))

    @staticmethod
    def split_sizes(n):
        nv = max(1, n // 20)
        nt = max(1, n // 20)
        return nt, nv, n - nt - nv

    def generate_synthetic(self, n_ent, n_rel, n_triples, seed):
        """Returns (heads, rels, tails) of all triples in generation order."""
        h, r, t = (np.empty(n_triples, np.int64) for _ in range(3))
        self._check(self.lib.orc_generate_synthetic(n_ent, n_rel, n_triples, seed, _p(h), _p(r), _p(t)))
        return h, r, t

    def synthetic_train(self, n_ent, n_rel, n_triples, seed):
        h, r, t = self.generate_synthetic(n_ent, n_rel, n_triples, seed)
        nt, nv, _ = self.split_sizes(n_triples)
        s = nt + nv
        return h[s:].copy(), r[s:].copy(), t[s:].copy()

    def init_store(self, model, n_ent, n_rel, de, dr, seed) -> Store:
        w = 2 if model in COMPLEX else 1
        e = np.empty((n_ent, w * de), self.dtype)
        r = np.empty((n_rel, w * dr), self.dtype)
        p = np.empty((n_rel, dr * de), self.dtype) if model == "transr" else None
        n = np.empty((n_rel, de), self.dtype) if model == "transh" else None
        self._check(self.lib.orc_init_store(MODELS[model], n_ent, n_rel, de, dr, seed,
                                            _p(e), _p(r), _p(p), _p(n)))
        return Store(e, r, p, n)

    def negative_sample(self, h, r, t, n_ent, n_rel, seed, avoid_self_loops=False):
        h, r, t = _i64(h), _i64(r), _i64(t)
        oh, ot = np.empty_like(h), np.empty_like(t)
        self._check(self.lib.orc_negative_sample(len(h), _p(h), _p(r), _p(t), n_ent, n_rel, seed,
                                                 int(avoid_self_loops), _p(oh), _p(ot)))
        return oh, ot

    def epoch_order(self, m, seed, epoch, shuffle=True):
        o = np.empty(m, np.int64)
        self._check(self.lib.orc_epoch_order(m, seed, int(shuffle), epoch, _p(o)))
        return o

    def build_incidence(self, kind, h, r, t, n_ent, n_rel):
        h, r, t = _i64(h), _i64(r), _i64(t)
        m = len(h)
        rp = np.empty(m + 1, np.int64)
        col = np.empty(3 * m, np.int64)
        val = np.empty(3 * m, self.dtype)
        nnz = C.c_int64()
        self._check(self.lib.orc_build_incidence({"ht": 0, "hrt": 1, "mult": 2, "mult_conj": 3}[kind], m, _p(h), _p(r), _p(t),
                                                 n_ent, n_rel, _p(rp), _p(col), _p(val), C.byref(nnz)))
        return rp, col[:nnz.value].copy(), val[:nnz.value].copy()

    def coo_to_csr(self, rows, cols, ri, ci, vi):
        ri, ci, vi = _i64(ri), _i64(ci), self._f(vi)
        rp = np.empty(rows + 1, np.int64)
        col = np.empty(max(1, len(ri)), np.int64)
        val = np.empty(max(1, len(ri)), self.dtype)
        nnz = C.c_int64()
        self._check(self.lib.orc_coo_to_csr(rows, cols, len(ri), _p(ri), _p(ci), _p(vi), _p(rp),
                                            _p(col), _p(val), C.byref(nnz)))
        return rp, col[:nnz.value].copy(), val[:nnz.value].copy()

    def transpose(self, rows, cols, rp, ci, v):
        rp, ci, v = _i64(rp), _i64(ci), self._f(v)
        orp = np.empty(cols + 1, np.int64)
        oci = np.empty(max(1, len(ci)), np.int64)
        ov = np.empty(max(1, len(ci)), self.dtype)
        self._check(self.lib.orc_transpose(rows, cols, _p(rp), _p(ci), _p(v), _p(orp), _p(oci), _p(ov)))
        return orp, oci[:len(ci)].copy(), ov[:len(ci)].copy()

    def spmm(self, rows, cols, rp, ci, v, x):
        rp, ci, v, x = _i64(rp), _i64(ci), self._f(v), self._f(x)
        out = np.empty((rows, x.shape[1]), self.dtype)
        self._check(self.lib.orc_spmm(rows, cols, _p(rp), _p(ci), _p(v), x.shape[0], x.shape[1], _p(x), _p(out)))
        return out

    def spmm_transpose_add(self, rows, cols, rp, ci, v, g, sink):
        rp, ci, v, g = _i64(rp), _i64(ci), self._f(v), self._f(g)
        assert sink.dtype == self.dtype and sink.flags.c_contiguous
        self._check(self.lib.orc_spmm_transpose_add(rows, cols, _p(rp), _p(ci), _p(v), g.shape[1], _p(g), _p(sink)))
        return sink

    def score_batch(self, model, store: Store, h, r, t, norm="l2"):
        h, r, t = _i64(h), _i64(r), _i64(t)
        de, dr = store.entity.shape[1], store.relation.shape[1]
        m = len(h)
        cfg = self._cfg_for(model, store, norm)
        scores = np.empty(m, self.dtype)
        v = np.empty((m, dr), self.dtype) if model in ("transe", "transr", "transh", "rotate") else None
        u = np.empty((m, de), self.dtype) if model in ("transr", "transh") else None
        dl = np.empty((m, de), self.dtype) if model == "toruse" else None
        st = self._store(store)
        self._check(self.lib.orc_score_batch(C.byref(cfg), C.byref(st), m, _p(h), _p(r), _p(t),
                                             _p(scores), _p(v), _p(u), _p(dl)))
        return scores, {"v": v, "u": u, "delta": dl}

    def rank_entities(self, model, store: Store, h, r, t, norm="l2", filt=None):
        """rank_entity (eval.cpp:16-63) of every query, tail then head: int64 (q, 2)."""
        h, r, t = _i64(h), _i64(r), _i64(t)
        cfg = self._cfg_for(model, store, norm)
        st = self._store(store)
        ranks = np.empty((len(h), 2), np.int64)
        if filt is None:
            fh = fr = ft = np.zeros(1, np.int64)
            nf, on = 0, 0
        else:
            fh, fr, ft = (_i64(x) for x in filt)
            nf, on = len(fh), 1
        self._check(self.lib.orc_rank_entities(C.byref(cfg), C.byref(st), len(h), _p(h), _p(r), _p(t), on, nf,
                                               _p(fh), _p(fr), _p(ft), _p(ranks)))
        return ranks

    def score_backward(self, model, store: Store, h, r, t, up, grads: Store, norm="l2"):
        h, r, t, up = _i64(h), _i64(r), _i64(t), self._f(up)
        cfg = self._cfg_for(model, store, norm)
        st, gs = self._store(store), self._store(grads)
        self._check(self.lib.orc_score_backward(C.byref(cfg), C.byref(st), len(h), _p(h), _p(r), _p(t),
                                                _p(up), C.byref(gs)))
        return grads

    def margin_ranking_loss(self, pos, neg, margin):
        pos, neg = self._f(pos), self._f(neg)
        m = len(pos)
        loss = self.real()
        dp, dn = np.empty(m, self.dtype), np.empty(m, self.dtype)
        self._check(self.lib.orc_margin_ranking_loss(m, len(neg), _p(pos), _p(neg), margin, C.byref(loss), _p(dp), _p(dn)))
        return loss.value, dp, dn

    def sgd_step(self, store: Store, grads: Store, lr):
        st, gs = self._store(store), self._store(grads)
        self._check(self.lib.orc_sgd_step(C.byref(st), C.byref(gs), lr))

    def renormalize_entities(self, store: Store):
        st = self._store(store)
        self._check(self.lib.orc_renormalize_entities(C.byref(st)))

    def train_epoch(self, model, store: Store, pos, neg, tc, epoch, lr, norm="l2"):
        (ph, pr, pt), (nh, nt) = [_i64(a) for a in pos], [_i64(a) for a in neg]
        cfg = self._cfg_for(model, store, norm)
        st = self._store(store)
        rep = _EpochReport()
        self._check(self.lib.orc_train_epoch(C.byref(cfg), C.byref(st), len(ph), _p(ph), _p(pr), _p(pt),
                                             _p(nh), _p(nt), C.byref(tc), epoch, lr, C.byref(rep)))
        return rep

    def train_batches(self, model, store: Store, pos, neg, tc, epoch, lr, b0, nb, norm="l2"):
        (ph, pr, pt), (nh, nt) = [_i64(a) for a in pos], [_i64(a) for a in neg]
        cfg = self._cfg_for(model, store, norm)
        st = self._store(store)
        secs, ls = C.c_double(), C.c_double()
        self._check(self.lib.orc_train_batches(C.byref(cfg), C.byref(st), len(ph), _p(ph), _p(pr), _p(pt),
                                               _p(nh), _p(nt), C.byref(tc), epoch, lr, b0, nb,
                                               C.byref(secs), C.byref(ls)))
        return secs.value, ls.value

    def fit(self, model, store: Store, h, r, t, tc, norm="l2"):
        h, r, t = _i64(h), _i64(r), _i64(t)
        cfg = self._cfg_for(model, store, norm)
        st = self._store(store)
        reps = (_EpochReport * max(1, tc.epochs))()
        self._check(self.lib.orc_fit(C.byref(cfg), C.byref(st), len(h), _p(h), _p(r), _p(t), C.byref(tc), reps))
        return [reps[i] for i in range(tc.epochs)]
