"""B200-native batched NTT engine for the hot path of arXiv 2402.00675.

The compute lives in ``libnttk_gpu.so`` (sm_100a kernels behind the C ABI in
include/nttk_gpu.h); ``nttk`` mirrors the reference ``nttk`` C++ interface on top of it,
and ``shard`` splits batches across the GPUs of one node.
"""
from . import nttk  # noqa: F401
from .nttk import (  # noqa: F401
    ButterflyKind, ContractViolation, CudaError, NttParams, Ordering, Redc, Spectrum, Tree,
    all_butterfly_kinds, build_params, butterfly_kind_from_string, cyclic_convolution_via_ntt,
    intt_inverse, ntt_forward, ntt_forward_inplace, pointwise_multiply, preset,
)

__version__ = "0.1.0"
