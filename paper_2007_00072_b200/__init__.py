"""B200-native (sm_100a) data-movement-optimised BERT encoder layer (arXiv 2007.00072).

The compute path is libencoder.so (include/encoder.h, csrc/): fused BSB / BDRLN / BAD /
AIB / BEI kernels and their backwards, cuBLAS contractions.  This package is the thin
ctypes binding (`ops`, `layer`), the data-parallel helpers (`dp`) and the byte/flop
tally (`tally`).  There is no CPU fallback: loading the binding without the built
library raises.
"""
from . import _abi  # noqa: F401

__all__ = ["ops", "layer", "dp", "tally"]
