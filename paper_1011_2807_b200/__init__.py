"""paper_1011_2807_b200 -- B200-native hot path of the sparse KNN join of arxiv 1011.2807.

The product is ``libknnjoin.so`` (C ABI, ``include/knnjoin.h``).  This package is its thin Python binding:
argument marshalling only, with the same entry-point names.  PyTorch supplies device memory, streams and
(in ``dist``) process groups.  There is no CPU fallback: if the library is missing, importing the binding
raises.
"""
from ._binding import (  # noqa: F401
    BINARY,
    FP32,
    INT8,
    DeviceCSR,
    Index,
    KnnJoinError,
    knnjoin_build_index,
    knnjoin_certify,
    knnjoin_index_stats,
    knnjoin_last_error,
    knnjoin_merge,
    knnjoin_query,
    knnjoin_validate_csr,
    knnjoin_version,
    library_path,
)
