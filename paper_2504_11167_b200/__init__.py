"""B200-native LR-SPIKE preconditioned Krylov solver (arXiv 2504.11167 hot path).

Layers:
  include/lrspike_capi.h      extern "C" boundary (liblrspike_cuda.so, CUDA sm_100a)
  include/lrspike/*.hpp       C++ drop-in API, namespace lrspike (liblrspike.so)
  paper_2504_11167_b200.api   Python mirror of the same operations over the C-ABI (ctypes)
"""

__all__ = ["api", "configs"]
