"""B200-native LSS sequence-distributed self-attention (arXiv 2311.02382).

Drop-in for the attention half of the reference's layer API (seqpar.model /
seqpar.sharded): hand-written sm_100a kernels in liblss.so (C ABI in
include/lss.h), driven from Python with torch used for device memory,
streams and torch.distributed (NCCL) only.
"""

from .errors import (CommAborted, CommTimeout, DegenerateRowError, NativeError, NumericsError,
                     PartitionError, ShapeError, UnsupportedError)

__all__ = [
    "CommAborted", "CommTimeout", "DegenerateRowError", "NativeError", "NumericsError",
    "PartitionError", "ShapeError", "UnsupportedError",
]
