"""B200-native FCDP parameter-movement hot path (arxiv 2602.06499).

libfcdp.so (built from csrc/ by build.py) holds the C++ control plane (a
drop-in re-implementation of the reference `shardsim` API) and the sm_100a
data plane.  This package is its Python face:

    shardsim   - the reference control-plane API, same names and errors
    _capi      - ctypes binding of include/fcdp.h
"""
from . import _capi  # noqa: F401

__version__ = "0.1.0"
