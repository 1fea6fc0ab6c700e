"""B200-native (sm_100a) active-view scoring rasterizer for DAV-GSWT (arXiv 2602.15355).

The hot path (project -> bin/sort -> composite -> score -> select) runs in the
CUDA kernels of libgsr.so behind the C ABI of include/gsr.h; ``gsr`` is the
thin ctypes binding, ``pipeline`` sequences the calls for a set of candidate
views, ``distributed`` shards views across GPUs.  No CPU fallback: importing
this package without a built libgsr.so raises ImportError.
"""
from . import gsr  # noqa: F401  (loads libgsr.so or fails loudly)
from .gsr import CAM_DTYPE, Context, Gaussians, GsrError, Lod  # noqa: F401

__all__ = ["gsr", "CAM_DTYPE", "Context", "Gaussians", "GsrError", "Lod"]
