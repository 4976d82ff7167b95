"""paper_2402_07033_b200 — B200-native MoE-layer hot path of Fiddler (arXiv 2402.07033).

The product is two native libraries built in-tree under ``_build/``:

* ``libmoe_b200.so``      — the C-ABI (``include/moe_b200.h``) over hand-written
  sm_100a kernels (router/top-k, TMA-ring streaming decode, permutation,
  combine/residual, weights init);
* ``libmoe_orch_b200.so`` — the drop-in C++ ``moe_orch`` API
  (``include/moe_orch/*.hpp``) implemented on top of that C-ABI.

This Python module is a thin ctypes front-end used by the tests and
``bench.py``.  There is no CPU fallback: loading fails loudly if the CUDA
library was not built, and every compute call fails with MOE_ERR_NO_DEVICE
without an sm_100 GPU.
"""
from .capi import (  # noqa: F401
    DTYPE_BF16,
    DTYPE_F32,
    Ctx,
    MoeError,
    Shape,
    Weights,
    declared_symbols,
    ep_shard_map_coselect,
    get_option,
    lib,
    lib_path,
    options,
    replica_plan,
    set_option,
    set_trace_path,
)
