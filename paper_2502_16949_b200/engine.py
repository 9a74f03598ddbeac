"""ctypes binding of include/skge_b200.h (the engine's C ABI).

Method names and argument meanings follow the reference library
(/root/reference/proj/include/sparsekge/*.hpp): negative_sample, score_batch,
score_backward, margin_ranking_loss, sgd_step, renormalize_entities,
train_epoch, fit. Errors are raised as EngineError carrying the reference
exception kind (ShapeError, ConfigError, TrainingError, ...).
"""
from __future__ import annotations

import ctypes as C
import weakref
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MODELS = {"transe": 0, "transr": 1, "transh": 2, "toruse": 3, "distmult": 4, "complex": 5, "rotate": 6}
COMPLEX_TAGS = (5, 6)  # ComplEx / RotatE tables: dim interleaved (re, im) float pairs per row
NORMS = {"l1": 0, "l2": 1}
KINDS = {1: "ShapeError", 2: "ConfigError", 3: "DegenerateTripleError", 4: "TrainingError",
         5: "ParseError", 6: "CudaError"}


def lib_path() -> str:
    # SKGE_B200_LIB points at an alternative build of the same engine (A/B experiments)
    return os.environ.get("SKGE_B200_LIB") or os.path.join(HERE, "libskge_b200.so")


class EngineError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = KINDS.get(code, str(code))
        self.msg = msg
        super().__init__(f"{self.kind}: {msg}")


class ModelConfig(C.Structure):
    _fields_ = [("model", C.c_uint32), ("norm", C.c_uint32), ("dim_entity", C.c_int64),
                ("dim_relation", C.c_int64)]

    @classmethod
    def make(cls, model: str, dim_entity: int, dim_relation: int | None = None, norm: str = "l2"):
        return cls(MODELS[model], NORMS[norm], dim_entity, dim_entity if dim_relation is None else dim_relation)


class TrainConfig(C.Structure):
    _fields_ = [("lr", C.c_float), ("margin", C.c_float), ("epochs", C.c_int64), ("batch_size", C.c_int64),
                ("seed", C.c_uint64), ("has_scheduler", C.c_int32), ("decay_every", C.c_int64),
                ("decay_factor", C.c_float), ("shuffle", C.c_int32), ("resample_negatives", C.c_int32),
                ("renorm_entities", C.c_int32)]

    @classmethod
    def make(cls, lr=4e-4, margin=0.5, epochs=200, batch_size=1024, seed=0, scheduler=None, shuffle=True,
             resample_negatives=False, renorm_entities=False):
        every, factor = scheduler if scheduler else (50, 0.5)
        return cls(lr, margin, epochs, batch_size, seed, 1 if scheduler else 0, every, factor, int(shuffle),
                   int(resample_negatives), int(renorm_entities))


class EpochReport(C.Structure):
    _fields_ = [("epoch", C.c_int64), ("loss", C.c_double), ("t_forward_s", C.c_double),
                ("t_backward_s", C.c_double), ("t_step_s", C.c_double)]


_LIB = None


def load_library():
    """Loads the native engine; raises if it was not built (no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise EngineError(6, f"native engine library missing: {path} (run __graft_entry__.build())")
    L = C.CDLL(path)
    vp, i64, i32, f32 = C.c_void_p, C.c_int64, C.c_int32, C.c_float
    L.skg_last_error.restype = C.c_char_p
    L.skg_last_error.argtypes = [vp]
    L.skg_version.restype = C.c_char_p
    L.skg_num_sms.argtypes = [vp]
    L.skg_last_launch_count.restype = i64
    L.skg_last_launch_count.argtypes = [vp]
    sig = {
        "skg_create": [C.c_int, C.POINTER(vp)],
        "skg_synchronize": [vp],
        "skg_store_upload": [vp, vp, i64, i64, vp, vp, vp, vp],
        "skg_store_download": [vp, vp, vp, vp, vp],
        "skg_sgd_step": [vp, vp, vp, vp, vp, f32],
        "skg_renormalize_entities": [vp],
        "skg_set_deferred_uploads": [vp, i32],
        "skg_set_phase_timers": [vp, i32],
        "skg_upload_stats": [vp, vp, vp],
        "skg_upload_bytes": [vp, vp],
        "skg_set_triples": [vp, i64, vp, vp, vp, i64, i64],
        "skg_set_negatives": [vp, i64, vp, vp],
        "skg_negative_sample": [vp, C.c_uint64, i32, vp, vp],
        "skg_epoch_order": [vp, i64, C.c_uint64, i32, i64, vp],
        "skg_build_incidence": [vp, i32, i64, vp, vp, vp, i64, i64, vp, vp, vp, vp],
        "skg_score_batch": [vp, vp, i64, vp, vp, vp, vp, vp],
        "skg_coo_to_csr": [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp],
        "skg_csr_transpose": [vp, i64, i64, vp, vp, vp, vp, vp, vp],
        "skg_spmm": [vp, i64, i64, vp, vp, vp, i64, i64, vp, vp],
        "skg_spmm_transpose_add": [vp, i64, i64, vp, vp, vp, i64, i64, vp, vp],
        "skg_score_backward": [vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp],
        "skg_margin_ranking_loss": [vp, i64, vp, vp, f32, vp, vp, vp],
        "skg_train_epoch": [vp, vp, vp, i64, f32, vp],
        "skg_fit": [vp, vp, vp, vp],
        "skg_profile_epoch": [vp, vp, vp, i64, f32, vp, vp, vp, vp],
        "skg_profile_shuffle_ms": [vp, vp],
        "skg_nccl_unique_id": [vp],
        "skg_dp_init": [vp, vp, C.c_int, C.c_int],
        "skg_generate_synthetic": [i64, i64, i64, C.c_uint64, vp, vp, vp],
        "skg_init_store": [C.c_uint32, i64, i64, i64, i64, C.c_uint64, vp, vp, vp, vp],
        "skg_flush_l2": [vp],
        "skg_measure_gather": [vp, i64, i32, vp],
        "skg_plan_stats": [vp, i64, vp, vp, vp],
        "skg_debug_tc_gemm": [vp, i32, vp, vp, vp],
        "skg_rank_entities": [vp, vp, i64, vp, vp, vp, i32, i64, vp, vp, vp, vp],
        "skg_dp_shard": [i64, i64, i32, i32, vp],
        "skg_shard_group_init": [vp, C.c_int, i64],
        "skg_shard_group_train_epoch": [vp, C.c_int, vp, vp, i64, f32, vp],
        "skg_shard_export": [vp, C.c_int, C.c_int, i64, vp],
        "skg_shard_import": [vp, vp],
        "skg_shard_release": [vp],
        "skg_peek_checkpoint": [C.c_char_p, vp],
        "skg_save_checkpoint": [C.c_char_p, C.c_uint32, i64, i64, i64, i64, vp, vp, vp, vp],
        "skg_load_checkpoint": [C.c_char_p, C.c_uint32, vp, vp, vp, vp],
    }
    L.skg_host_last_error.restype = C.c_char_p
    L.skg_checkpoint_last_error.restype = C.c_char_p
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.skg_destroy.argtypes = [vp]
    L.skg_destroy.restype = None
    _LIB = L
    return L


_PTRS = {}  # id(array) -> (weakref, c_void_p): per-step re-uploads pass the same arrays


class _Arg:
    """A pointer argument that keeps its array alive for the duration of the call."""
    __slots__ = ("_as_parameter_", "a")

    def __init__(self, ptr, a):
        self._as_parameter_ = ptr
        self.a = a


def _p(a):
    if a is None:
        return None
    hit = _PTRS.get(id(a))
    if hit is None or hit[0]() is not a:
        if len(_PTRS) > 64:
            _PTRS.clear()
        hit = (weakref.ref(a), C.c_void_p(a.ctypes.data))
        _PTRS[id(a)] = hit
    return _Arg(hit[1], a)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


class Engine:
    """One device context (skg_ctx): device-resident store, triples and plans."""

    def __init__(self, device: int = 0):
        self.L = load_library()
        h = C.c_void_p()
        rc = self.L.skg_create(device, C.byref(h))
        if rc != 0:
            raise EngineError(rc, self.L.skg_last_error(None).decode())
        self.h = h
        self.num_sms = self.L.skg_num_sms(h)
        self.dims = None

    def close(self):
        if getattr(self, "h", None):
            self.L.skg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise EngineError(rc, self.L.skg_last_error(self.h).decode())

    # ------------------------------------------------------------ store
    def store_upload(self, cfg: ModelConfig, entity, relation, proj=None, normals=None):
        entity, relation, proj, normals = _f32(entity), _f32(relation), _f32(proj), _f32(normals)
        w = 2 if cfg.model in COMPLEX_TAGS else 1
        self.dims = (entity.shape[0], relation.shape[0], w * cfg.dim_entity, w * cfg.dim_relation,
                     proj is not None, normals is not None)
        self._check(self.L.skg_store_upload(self.h, C.byref(cfg), entity.shape[0], relation.shape[0], _p(entity),
                                            _p(relation), _p(proj), _p(normals)))

    def _empty_tables(self):
        n, r, de, dr, hp, hn = self.dims
        return (np.empty((n, de), np.float32), np.empty((r, dr), np.float32),
                np.empty((r, dr * de), np.float32) if hp else None, np.empty((r, de), np.float32) if hn else None)

    def store_download(self):
        e, r, p, n = self._empty_tables()
        self._check(self.L.skg_store_download(self.h, _p(e), _p(r), _p(p), _p(n)))
        return e, r, p, n

    def sgd_step(self, g_entity, g_relation, g_proj, g_normals, lr):
        self._check(self.L.skg_sgd_step(self.h, _p(_f32(g_entity)), _p(_f32(g_relation)), _p(_f32(g_proj)),
                                        _p(_f32(g_normals)), lr))

    def renormalize_entities(self):
        self._check(self.L.skg_renormalize_entities(self.h))

    # ------------------------------------------------------------ triples
    def set_deferred_uploads(self, enable: bool):
        """Opt-in overlapped re-upload of pinned id arrays (see skge_b200.h)."""
        self._check(self.L.skg_set_deferred_uploads(self.h, int(bool(enable))))

    def set_phase_timers(self, enable: bool):
        """PhaseTimer buckets in EpochReport (default on; see skge_b200.h)."""
        self._check(self.L.skg_set_phase_timers(self.h, int(bool(enable))))

    def upload_bytes(self):
        """Bytes DMA'd host -> device by deferred re-uploads so far (skg_upload_bytes)."""
        b = C.c_int64()
        self._check(self.L.skg_upload_bytes(self.h, C.byref(b)))
        return b.value

    def upload_stats(self):
        """(hits, misses) of deferred re-uploads: identical data kept / rolled back and retrained."""
        a, b = C.c_int64(), C.c_int64()
        self._check(self.L.skg_upload_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_triples(self, h, r, t, num_entities, num_relations):
        h, r, t = _i64(h), _i64(r), _i64(t)
        self._check(self.L.skg_set_triples(self.h, len(h), _p(h), _p(r), _p(t), num_entities, num_relations))
        self.m = len(h)

    def set_negatives(self, nh, nt):
        nh, nt = _i64(nh), _i64(nt)
        self._check(self.L.skg_set_negatives(self.h, len(nh), _p(nh), _p(nt)))

    def negative_sample(self, seed, avoid_self_loops=False):
        oh = np.empty(self.m, np.int64)
        ot = np.empty(self.m, np.int64)
        self._check(self.L.skg_negative_sample(self.h, seed, int(avoid_self_loops), _p(oh), _p(ot)))
        return oh, ot

    def epoch_order(self, m, seed, epoch, shuffle=True):
        o = np.empty(max(m, 1), np.int64)
        self._check(self.L.skg_epoch_order(self.h, m, seed, int(shuffle), epoch, _p(o)))
        return o[:m]

    # ------------------------------------------------------------ parity surface
    def build_incidence(self, layout, h, r, t, num_entities, num_relations):
        h, r, t = _i64(h), _i64(r), _i64(t)
        m = len(h)
        rp = np.empty(m + 1, np.int64)
        col = np.empty(3 * m + 1, np.int64)
        val = np.empty(3 * m + 1, np.float32)
        nnz = C.c_int64()
        self._check(self.L.skg_build_incidence(self.h, {"ht": 0, "hrt": 1, "mult": 2, "mult_conj": 3}[layout], m, _p(h), _p(r), _p(t),
                                               num_entities, num_relations, _p(rp), _p(col), _p(val),
                                               C.byref(nnz)))
        return rp, col[:nnz.value].copy(), val[:nnz.value].copy()

    def coo_to_csr(self, rows, cols, ri, ci, vi):
        """coo_to_csr (sparse.hpp:110-161) -> (row_ptr, col_idx, vals)."""
        ri, ci, vi = _i64(ri), _i64(ci), _f32(vi)
        n = len(ri)
        rp = np.empty(rows + 1, np.int64)
        col = np.empty(max(1, n), np.int64)
        val = np.empty(max(1, n), np.float32)
        nnz = C.c_int64()
        self._check(self.L.skg_coo_to_csr(self.h, rows, cols, n, _p(ri), _p(ci), _p(vi), _p(rp), _p(col), _p(val),
                                          C.byref(nnz)))
        return rp, col[:nnz.value].copy(), val[:nnz.value].copy()

    def transpose(self, rows, cols, rp, ci, v):
        """transpose (sparse.hpp:164-183) of a CSR matrix -> (row_ptr, col_idx, vals)."""
        rp, ci, v = _i64(rp), _i64(ci), _f32(v)
        nnz = int(rp[rows]) if len(rp) > rows else 0
        orp = np.empty(cols + 1, np.int64)
        oci = np.empty(max(1, nnz), np.int64)
        ov = np.empty(max(1, nnz), np.float32)
        self._check(self.L.skg_csr_transpose(self.h, rows, cols, _p(rp), _p(ci), _p(v), _p(orp), _p(oci), _p(ov)))
        return orp, oci[:nnz].copy(), ov[:nnz].copy()

    def spmm(self, rows, cols, rp, ci, v, x):
        """spmm (sparse.hpp:242-266), plus-times: A (rows x cols) times x (cols x d)."""
        rp, ci, v, x = _i64(rp), _i64(ci), _f32(v), _f32(x)
        out = np.empty((rows, x.shape[1]), np.float32)
        self._check(self.L.skg_spmm(self.h, rows, cols, _p(rp), _p(ci), _p(v), x.shape[0], x.shape[1], _p(x),
                                    _p(out)))
        return out

    def spmm_transpose_add(self, rows, cols, rp, ci, v, g, sink):
        """spmm_transpose_add (sparse.hpp:273-306): sink (cols x d) += A^T g, in place."""
        rp, ci, v, g = _i64(rp), _i64(ci), _f32(v), _f32(g)
        assert sink.dtype == np.float32 and sink.flags.c_contiguous
        self._check(self.L.skg_spmm_transpose_add(self.h, rows, cols, _p(rp), _p(ci), _p(v), g.shape[0], g.shape[1],
                                                  _p(g), _p(sink)))
        return sink

    def score_batch(self, cfg: ModelConfig, h, r, t, residual=False):
        h, r, t = _i64(h), _i64(r), _i64(t)
        m = len(h)
        scores = np.empty(max(m, 1), np.float32)
        d = cfg.dim_entity if cfg.model in (0, 3) else 2 * cfg.dim_entity if cfg.model == 6 else cfg.dim_relation
        res = np.empty((max(m, 1), d), np.float32) if residual else None  # RotatE: q rows (re, im)
        self._check(self.L.skg_score_batch(self.h, C.byref(cfg), m, _p(h), _p(r), _p(t), _p(scores), _p(res)))
        return (scores[:m], res[:m]) if residual else scores[:m]

    def score_backward(self, cfg: ModelConfig, h, r, t, upstream, grads):
        """Accumulates into grads = (entity, relation, proj|None, normals|None) in place."""
        h, r, t, up = _i64(h), _i64(r), _i64(t), _f32(upstream)
        for g in grads:
            assert g is None or (g.dtype == np.float32 and g.flags.c_contiguous)
        self._check(self.L.skg_score_backward(self.h, C.byref(cfg), len(h), _p(h), _p(r), _p(t), _p(up),
                                              *[_p(g) for g in grads]))
        return grads

    def margin_ranking_loss(self, pos, neg, margin):
        pos, neg = _f32(pos), _f32(neg)
        if len(pos) != len(neg):
            raise EngineError(1, "margin_ranking_loss: length mismatch")
        m = len(pos)
        loss = C.c_float()
        dp, dn = np.empty(max(m, 1), np.float32), np.empty(max(m, 1), np.float32)
        self._check(self.L.skg_margin_ranking_loss(self.h, m, _p(pos), _p(neg), margin, C.byref(loss), _p(dp),
                                                   _p(dn)))
        return loss.value, dp[:m], dn[:m]

    # ------------------------------------------------------------ training
    def train_epoch(self, cfg: ModelConfig, tc: TrainConfig, epoch: int, lr: float) -> EpochReport:
        rep = EpochReport()
        self._check(self.L.skg_train_epoch(self.h, C.byref(cfg), C.byref(tc), epoch, lr, C.byref(rep)))
        return rep

    def fit(self, cfg: ModelConfig, tc: TrainConfig):
        reps = (EpochReport * max(1, tc.epochs))()
        self._check(self.L.skg_fit(self.h, C.byref(cfg), C.byref(tc), reps))
        return [reps[i] for i in range(tc.epochs)]

    def profile_epoch(self, cfg: ModelConfig, tc: TrainConfig, epoch: int, lr: float):
        rep = EpochReport()
        f, b, p = C.c_double(), C.c_double(), C.c_double()
        self._check(self.L.skg_profile_epoch(self.h, C.byref(cfg), C.byref(tc), epoch, lr, C.byref(rep),
                                             C.byref(f), C.byref(b), C.byref(p)))
        return rep, f.value, b.value, p.value

    def profile_shuffle_ms(self) -> float:
        """Shuffle (epoch permutation) time of the last profile_epoch, ms."""
        v = C.c_double()
        self._check(self.L.skg_profile_shuffle_ms(self.h, C.byref(v)))
        return v.value

    def synchronize(self):
        self._check(self.L.skg_synchronize(self.h))

    def last_launch_count(self) -> int:
        return int(self.L.skg_last_launch_count(self.h))

    # ------------------------------------------------------------ data parallel
    @staticmethod
    def nccl_unique_id() -> bytes:
        L = load_library()
        buf = C.create_string_buffer(128)
        rc = L.skg_nccl_unique_id(buf)
        if rc != 0:
            raise EngineError(rc, "ncclGetUniqueId failed")
        return buf.raw

    def dp_init(self, unique_id: bytes, rank: int, world: int):
        buf = C.create_string_buffer(unique_id, 128)
        self._check(self.L.skg_dp_init(self.h, buf, rank, world))

    # ------------------------------------------------------------ row-sharded data parallel
    SHARD_HANDLE_BYTES = 128

    @staticmethod
    def _handles(engines):
        arr = (C.c_void_p * len(engines))(*[e.h.value for e in engines])
        return arr

    @staticmethod
    def shard_group_init(engines, batch_size: int):
        """One process drives every rank: engines[k] is rank k (skg_shard_group_init)."""
        L = load_library()
        rc = L.skg_shard_group_init(Engine._handles(engines), len(engines), batch_size)
        if rc != 0:
            raise EngineError(rc, L.skg_last_error(engines[0].h).decode())

    @staticmethod
    def shard_group_train_epoch(engines, cfg: ModelConfig, tc: TrainConfig, epoch: int, lr: float):
        L = load_library()
        reps = (EpochReport * len(engines))()
        rc = L.skg_shard_group_train_epoch(Engine._handles(engines), len(engines), C.byref(cfg), C.byref(tc),
                                           epoch, lr, reps)
        if rc != 0:
            msgs = [L.skg_last_error(e.h).decode() for e in engines]
            raise EngineError(rc, next((m for m in msgs if m), ""))
        return [reps[i] for i in range(len(engines))]

    def shard_export(self, rank: int, world: int, batch_size: int) -> bytes:
        """This rank's IPC handle (one process per GPU); all-gather it, then shard_import."""
        buf = C.create_string_buffer(self.SHARD_HANDLE_BYTES)
        self._check(self.L.skg_shard_export(self.h, rank, world, batch_size, buf))
        return buf.raw

    def shard_import(self, handles):
        blob = b"".join(handles)
        buf = C.create_string_buffer(blob, len(blob))
        self._check(self.L.skg_shard_import(self.h, buf))

    def shard_release(self):
        self._check(self.L.skg_shard_release(self.h))

    # ------------------------------------------------------------ measurement hooks
    def measure_gather(self, table_bytes: int, row_floats: int) -> float:
        """Random-row gather GB/s over a table of table_bytes (L2-resident when it fits)."""
        g = C.c_double()
        self._check(self.L.skg_measure_gather(self.h, table_bytes, row_floats, C.byref(g)))
        return g.value

    def flush_l2(self):
        self._check(self.L.skg_flush_l2(self.h))

    def rank_entities(self, cfg, h, r, t, filt=None):
        """rank_entity (eval.cpp:16-63) for every query: int64 (q, 2) = [tail rank, head rank];
        filt = (heads, relations, tails) of the known-true triples selects the filtered protocol."""
        h, r, t = _i64(h), _i64(r), _i64(t)
        ranks = np.empty((len(h), 2), np.int64)
        if filt is None:
            z = np.zeros(1, np.int64)
            self._check(self.L.skg_rank_entities(self.h, C.byref(cfg), len(h), _p(h), _p(r), _p(t), 0, 0,
                                                 _p(z), _p(z), _p(z), _p(ranks)))
        else:
            fh, fr, ft = (_i64(x) for x in filt)
            self._check(self.L.skg_rank_entities(self.h, C.byref(cfg), len(h), _p(h), _p(r), _p(t), 1, len(fh),
                                                 _p(fh), _p(fr), _p(ft), _p(ranks)))
        return ranks

    def debug_tc_gemm(self, mode: int, A, B):
        A, B = _f32(A), _f32(B)
        D = np.empty((128, 128), np.float32)
        self._check(self.L.skg_debug_tc_gemm(self.h, mode, _p(A), _p(B), _p(D)))
        return D

    def plan_stats(self, batch: int):
        s, e, r = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.L.skg_plan_stats(self.h, batch, C.byref(s), C.byref(e), C.byref(r)))
        return s.value, e.value, r.value


def dp_shard(m: int, batch_size: int, world: int, rank: int):
    """Host-only shard geometry of the data-parallel engine (no GPU needed)."""
    L = load_library()
    out = np.zeros(5, np.int64)
    rc = L.skg_dp_shard(m, batch_size, world, rank, _p(out))
    if rc != 0:
        raise EngineError(rc, "dp_shard: bad arguments")
    return dict(S=int(out[0]), i0_last=int(out[1]), s_last=int(out[2]), Mg=int(out[3]), nb=int(out[4]))


def _host_check(L, rc):
    if rc != 0:
        raise EngineError(rc, L.skg_host_last_error().decode())


def split_sizes(n: int):
    """data_io.cpp:189-190: test n/20, valid n/20, rest train."""
    nv = max(1, n // 20)
    nt = max(1, n // 20)
    return nt, nv, n - nt - nv


def generate_synthetic(n_entities: int, n_relations: int, n_triples: int, seed: int):
    """Reference lattice generator (host, once per job); returns the train split."""
    L = load_library()
    h, r, t = (np.empty(n_triples, np.int64) for _ in range(3))
    _host_check(L, L.skg_generate_synthetic(n_entities, n_relations, n_triples, seed, _p(h), _p(r), _p(t)))
    nt, nv, _ = split_sizes(n_triples)
    s = nt + nv
    return h[s:].copy(), r[s:].copy(), t[s:].copy()


def init_store(model: str, n_entities: int, n_relations: int, de: int, dr: int, seed: int):
    """init_store (embedding.cpp:129-163) on the host; returns fp32 tables."""
    L = load_library()
    w = 2 if MODELS[model] in COMPLEX_TAGS else 1
    e = np.empty((n_entities, w * de), np.float32)
    r = np.empty((n_relations, w * dr), np.float32)
    p = np.empty((n_relations, dr * de), np.float32) if model == "transr" else None
    n = np.empty((n_relations, de), np.float32) if model == "transh" else None
    _host_check(L, L.skg_init_store(MODELS[model], n_entities, n_relations, de, dr, seed, _p(e), _p(r), _p(p), _p(n)))
    return e, r, p, n


# ---- checkpoints (embedding.cpp:200-251, SKGECKPT v1) ----------------------
class CheckpointHeader(C.Structure):  # embedding.hpp:134-140
    _fields_ = [("model", C.c_uint32), ("num_entities", C.c_int64), ("num_relations", C.c_int64),
                ("dim_entity", C.c_int64), ("dim_relation", C.c_int64)]


class RunSummary(C.Structure):
    _fields_ = [("engine", C.c_char_p), ("dataset_source", C.c_char_p), ("entities", C.c_int64),
                ("relations", C.c_int64), ("train", C.c_int64), ("valid", C.c_int64), ("test", C.c_int64),
                ("dropped_valid", C.c_int64), ("dropped_test", C.c_int64), ("threads", C.c_int32),
                ("epochs_run", C.c_int64), ("final_loss", C.c_double), ("t_forward_s", C.c_double),
                ("t_backward_s", C.c_double), ("t_step_s", C.c_double), ("checkpoint_path", C.c_char_p)]


class RunLog:
    """train_log.jsonl / loss.log / summary.json writers of `kge train` (kge.cpp:181-247)."""

    def __init__(self, out_dir: str):
        self.L = load_library()
        for name, args in {"skg_run_log_open": [C.c_char_p, C.c_void_p],
                           "skg_run_log_epoch": [C.c_void_p, C.c_void_p],
                           "skg_run_log_summary": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]}.items():
            getattr(self.L, name).argtypes = args
            getattr(self.L, name).restype = C.c_int
        self.L.skg_run_log_close.argtypes = [C.c_void_p]
        self.L.skg_run_log_close.restype = None
        self.L.skg_run_log_last_error.restype = C.c_char_p
        self.h = C.c_void_p()
        self._check(self.L.skg_run_log_open(out_dir.encode(), C.byref(self.h)))

    def _check(self, rc):
        if rc != 0:
            raise EngineError(rc, self.L.skg_run_log_last_error().decode())

    def epoch(self, rep: EpochReport):
        self._check(self.L.skg_run_log_epoch(self.h, C.byref(rep)))

    def summary(self, cfg: ModelConfig, tc: TrainConfig, info: RunSummary):
        self._check(self.L.skg_run_log_summary(self.h, C.byref(cfg), C.byref(tc), C.byref(info)))

    def close(self):
        if self.h:
            self.L.skg_run_log_close(self.h)
            self.h = None


def _ckpt_check(L, rc):
    if rc != 0:
        raise EngineError(rc, L.skg_checkpoint_last_error().decode())


def peek_checkpoint(path: str) -> CheckpointHeader:
    L = load_library()
    h = CheckpointHeader()
    _ckpt_check(L, L.skg_peek_checkpoint(path.encode(), C.byref(h)))
    return h


def save_checkpoint(path: str, model: str, entity, relation, proj=None, normals=None):
    """save_checkpoint(path, model, store): fp32 host tables written as f64 (the reference's 32-bit build)."""
    L = load_library()
    e, r = _f32(entity), _f32(relation)
    p = None if proj is None else _f32(proj)
    n = None if normals is None else _f32(normals)
    w = 2 if MODELS[model] in COMPLEX_TAGS else 1
    _ckpt_check(L, L.skg_save_checkpoint(path.encode(), MODELS[model], e.shape[0], r.shape[0], e.shape[1] // w,
                                         r.shape[1] // w, _p(e), _p(r), _p(p), _p(n)))


def load_checkpoint(path: str, expected: str):
    """load_checkpoint<Real>(path, expected) -> (entity, relation, proj, normals) fp32 tables."""
    L = load_library()
    h = peek_checkpoint(path)
    w = 2 if h.model in COMPLEX_TAGS else 1
    e = np.empty((h.num_entities, w * h.dim_entity), np.float32)
    r = np.empty((h.num_relations, w * h.dim_relation), np.float32)
    p = np.empty((h.num_relations, h.dim_relation * h.dim_entity), np.float32) if h.model == 1 else None
    n = np.empty((h.num_relations, h.dim_entity), np.float32) if h.model == 2 else None
    _ckpt_check(L, L.skg_load_checkpoint(path.encode(), MODELS[expected], _p(e), _p(r), _p(p), _p(n)))
    return e, r, p, n
