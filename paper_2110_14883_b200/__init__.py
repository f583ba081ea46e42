"""B200-native multi-dimensional tensor-parallel linear layer (arXiv 2110.14883, Colossal-AI).

The product is the C-ABI library libtp_b200.so (include/tp_b200.h): hand-written
sm_100a tcgen05/TMEM/TMA GEMMs, HBM-bound layout kernels, and the 1D / 2D / 2.5D / 3D
schedules over NCCL (or the in-process transport). `api` is its thin ctypes binding.
Importing `api` fails loudly if the library was not built; there is no CPU fallback.
"""
__all__ = ["api", "build"]
