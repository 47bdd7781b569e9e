"""B200-native coupled MLMC level sampler (arXiv 1612.07717 hot path).

The product is ``libablmc_b200.so`` (sm_100a CUDA kernels behind the C ABI in
``include/ablmc_b200.h``); :mod:`.ablmc` mirrors the reference's API over it.
"""
from . import capi  # noqa: F401

__all__ = ["capi", "ablmc"]
