"""paper_2409_03856_b200 — B200-native Sirius decode hot path (arXiv 2409.03856).

libsirius.so (CUDA, sm_100a) behind the C ABI in include/sirius.h; `sirius` is the ctypes binding
with the same entry-point names, `driver` the host loop of Algorithm 1.
"""
__all__ = ["sirius", "driver"]
