"""SKGECKPT v1 checkpoints (embedding.cpp:200-251) through the engine's C ABI.

Host-only file I/O (no GPU): the reference's own checkpoint tests
(test_embedding.cpp:220-329) restated — exact round trip of every table,
the fixed byte layout, malformed-input rejection and tag validation.
"""
import os
import struct

import numpy as np
import pytest

from paper_2502_16949_b200.engine import (EngineError, init_store, load_checkpoint, peek_checkpoint,
                                          save_checkpoint)


@pytest.mark.parametrize("model,de,dr", [("transe", 5, 5), ("transr", 5, 3), ("transh", 4, 4), ("toruse", 6, 6),
                                         ("distmult", 4, 4), ("complex", 3, 3), ("rotate", 5, 5)])
def test_round_trip_exact(tmp_path, model, de, dr):  # test_embedding.cpp:220-245
    e, r, p, n = init_store(model, 7, 3, de, dr, 42)
    path = str(tmp_path / f"ckpt_{model}.bin")
    save_checkpoint(path, model, e, r, p, n)
    h = peek_checkpoint(path)
    assert (h.model, h.num_entities, h.num_relations, h.dim_entity, h.dim_relation) == (
        {"transe": 0, "transr": 1, "transh": 2, "toruse": 3, "distmult": 4, "complex": 5, "rotate": 6}[model],
        7, 3, de, dr)
    e2, r2, p2, n2 = load_checkpoint(path, model)
    assert np.array_equal(e, e2) and np.array_equal(r, r2)
    assert (p is None and p2 is None) or np.array_equal(p, p2)
    assert (n is None and n2 is None) or np.array_equal(n, n2)


def test_fixed_byte_layout(tmp_path):  # test_embedding.cpp:257-283
    path = str(tmp_path / "ckpt_layout.bin")
    save_checkpoint(path, "transe", np.array([[1.0, 2.0]], np.float32), np.array([[-3.5, 0.25]], np.float32))
    b = open(path, "rb").read()
    assert len(b) == 8 + 4 + 4 + 4 * 8 + 4 * 8
    assert b[:8] == b"SKGECKPT"
    assert struct.unpack("<II", b[8:16]) == (1, 0)
    assert struct.unpack("<4Q", b[16:48]) == (1, 1, 2, 2)
    assert struct.unpack("<4d", b[48:80]) == (1.0, 2.0, -3.5, 0.25)


def test_malformed_inputs(tmp_path):  # test_embedding.cpp:285-320
    path = str(tmp_path / "ckpt_bad.bin")
    open(path, "wb").write(b"NOTACKPT" + b"x" * 32)
    with pytest.raises(EngineError) as ei:
        peek_checkpoint(path)
    assert ei.value.kind == "ParseError"
    e, r, p, n = init_store("transe", 4, 2, 3, 3, 9)
    save_checkpoint(path, "transe", e, r)
    with pytest.raises(EngineError) as ei:  # wrong model on load
        load_checkpoint(path, "transr")
    assert ei.value.kind == "ConfigError" and "expected transr" in ei.value.msg
    b = open(path, "rb").read()
    open(path, "wb").write(b[:-7])  # truncated payload
    with pytest.raises(EngineError) as ei:
        load_checkpoint(path, "transe")
    assert ei.value.kind == "ParseError"
    open(path, "wb").write(b + b"junk")  # trailing bytes
    with pytest.raises(EngineError) as ei:
        load_checkpoint(path, "transe")
    assert "trailing bytes" in ei.value.msg
    with pytest.raises(EngineError):
        peek_checkpoint(str(tmp_path / "ckpt_missing.bin"))


def test_save_validates_tables(tmp_path):  # test_embedding.cpp:322-329
    e, r, _, _ = init_store("transe", 3, 2, 4, 4, 1)
    path = str(tmp_path / "ckpt_mismatch.bin")
    with pytest.raises(EngineError) as ei:
        save_checkpoint(path, "transr", e, r)
    assert ei.value.kind == "ConfigError"
    assert not os.path.exists(path) or os.path.getsize(path) == 0


def test_complex_payload_layout(tmp_path):  # test_embedding.cpp:246-256: interleaved (re, im) doubles
    e, r, _, _ = init_store("rotate", 6, 2, 5, 5, 77)
    assert e.shape == (6, 10) and r.shape == (2, 10)
    path = str(tmp_path / "ckpt_rotate.bin")
    save_checkpoint(path, "rotate", e, r)
    b = open(path, "rb").read()
    assert len(b) == 8 + 4 + 4 + 4 * 8 + 8 * (6 * 10 + 2 * 10)
    v = np.frombuffer(b[48:48 + 8 * 60], np.float64).reshape(6, 10)
    assert np.array_equal(v.astype(np.float32), e)
    with pytest.raises(EngineError) as ei:
        load_checkpoint(path, "complex")
    assert ei.value.kind == "ConfigError"
