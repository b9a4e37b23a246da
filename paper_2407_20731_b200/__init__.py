"""B200-native in-situ lossy compression of spectral-element fields (arXiv 2407.20731).

The hot path -- per-element 3-D discrete Legendre transform, exact energy
truncation, mask + packed-value encoding, inverse transform with L2/Linf error
report -- runs in hand-written sm_100a kernels behind the C ABI of
include/isf_lossy.h; this package is the Python mirror of the reference's task
interface.  See DESIGN.md.
"""
from .lossy import (  # noqa: F401
    CompressedBlock, CompressionReport, ErrorCode, ErrorNorm, ErrorReport, Field, IsfError,
    LossyConfig, LossyPlan, compression_ratio, decompress_with_error, get_plan, lossy_compress,
    lossy_compress_frame, lossy_decompress,
)
from ._native import LIB_PATH, EXPORTS  # noqa: F401
