"""B200-native forward/backward operators of fan-beam coded-aperture X-ray
coherent-scatter imaging (arXiv 1603.06400) -- Python side of libcacsi.so.

The product is the C-ABI library (include/cacsi.h, csrc/); this package only
builds it (build.py) and marshals arguments to it (binding.py).
"""
from .binding import CacsiError, Geometry, GeometryDesc, geometry_create, lib, status_string  # noqa: F401
