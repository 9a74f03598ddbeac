"""CPU checks of the native boundary: the C-ABI library loads and exports every
entry point include/skge_b200.h declares (no compute without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "skge_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(skg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("skg_create", "skg_negative_sample", "skg_build_incidence", "skg_score_batch",
                 "skg_score_backward", "skg_margin_ranking_loss", "skg_sgd_step", "skg_train_epoch", "skg_fit"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2502_16949_b200.engine import lib_path, load_library
    if not os.path.exists(lib_path()):
        pytest.fail("libskge_b200.so not built (run __graft_entry__.build())")
    lib = load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2502_16949_b200 import Engine, EngineError
    with pytest.raises(EngineError) as e:
        Engine(0)
    assert e.value.kind == "CudaError"


@pytest.mark.parametrize("name", ["shim_drop_in", "ref_cases"])
def test_cpp_shim_compiles(name):
    """The reference-signature C++ shim (include/skge_b200.hpp) compiles against the ABI, with
    a reference-style caller and with the adapted reference unit-test case bodies."""
    import subprocess
    import tempfile
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "shim")
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", out,
                        "-L", os.path.join(ROOT, "paper_2502_16949_b200"), "-lskge_b200",
                        f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2502_16949_b200')}"], check=True)


def test_torch_imports_after_engine_library():
    """libskge_b200.so links the libnccl.so.2 PyTorch ships, so loading the
    engine first must not break a later `import torch` (shared soname)."""
    import subprocess
    import sys
    from paper_2502_16949_b200.engine import lib_path
    code = ("import ctypes, sys; ctypes.CDLL(sys.argv[1]); import torch; "
            "print(torch.cuda.nccl.version() if hasattr(torch.cuda, 'nccl') else 'no-nccl')")
    out = subprocess.run([sys.executable, "-c", code, lib_path()], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]


def test_mt_jump_ahead_continues_the_reference_stream():
    """Host part of the chunked MT19937-64 generator (mt_jump.cpp): states advanced by
    x^J mod f (Berlekamp-Massey characteristic polynomial) continue std::mt19937_64."""
    import ctypes as C
    from paper_2502_16949_b200.engine import load_library
    L = load_library()
    L.skg_debug_mt_jump_selftest.restype = C.c_int32
    L.skg_debug_mt_jump_selftest.argtypes = [C.c_uint64, C.c_int64]
    for seed, jump in [(5489, 1), (1, 312), (7, 312 * 1000 + 5), (0x9E3779B97F4A7C15, 8_000_000)]:
        assert L.skg_debug_mt_jump_selftest(seed, jump) == 1, (seed, jump)
