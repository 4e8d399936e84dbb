"""B200-native HybriMoE MoE-layer hot path.

Drop-in for the reference simulator's API (``moesim.core / costs /
scheduling / caching / prefetch / engine / tracegen``) backed by the native
library ``libhybrimoe.so``: a bit-exact C++ decision core plus sm_100a CUDA
kernels and a host runtime that execute the decided plan for real.
"""
__version__ = "0.1.0"
