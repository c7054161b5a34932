"""B200-native GpSense subgraph-matching hot path (arxiv 1807.08804, thesis Ch. 3).

The product is libgpsense.so (include/gpsense.h); `gpsense` is its thin ctypes
binding.  Importing this package loads the CUDA library and raises if it has not
been built -- there is no CPU fallback.
"""
from .gpsense import (  # noqa: F401
    GPS_ANY,
    GPS_FREE,
    Context,
    GpsError,
    Graph,
    default_opts,
)

__all__ = ["Context", "Graph", "GpsError", "default_opts", "GPS_ANY", "GPS_FREE"]
