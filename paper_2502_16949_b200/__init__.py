"""B200-native SparseTransX training engine (arXiv 2502.16949), sm_100a only.

The product is the in-tree C-ABI library ``libskge_b200.so`` (CUDA kernels +
C++ host orchestration, see include/skge_b200.h). This package is a thin
ctypes binding of that ABI used by the test-suite and bench.py; it has no
compute of its own and raises if the native library is missing.
"""
from .engine import (Engine, EngineError, ModelConfig, TrainConfig, EpochReport, lib_path,  # noqa: F401
                     load_library, MODELS, NORMS)

__all__ = ["Engine", "EngineError", "ModelConfig", "TrainConfig", "EpochReport", "lib_path",
           "load_library", "MODELS", "NORMS"]
