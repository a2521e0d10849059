"""B200-native self-assisted speculative decoding for CPU-offloaded MoE (arxiv/paper_2604_10152).

The product is the sm_100a library ``lib/libspecmoe_b200.so`` (kernels + C++ engine + C ABI,
include/specmoe_b200.h); ``engine`` is its Python host mirror.
"""
from .engine import (BF16, F32, GEMM_AUTO, GEMM_SIMT, GEMM_TCGEN05, SWIGLU3, TANH2, Engine, EngineError,  # noqa: F401
                     ModelSpec, RunCfg)
from .prompts import make_prompts  # noqa: F401
