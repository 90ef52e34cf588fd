"""B200-native FCDP parameter-movement hot path (arxiv 2602.06499).

libfcdp.so (built from csrc/ by build.py) holds the C++ control plane (a
drop-in re-implementation of the reference `shardsim` API) and the sm_100a
data plane.  This package is its Python face:

    shardsim   - the reference control-plane API, same names and errors
    _capi      - ctypes binding of include/fcdp.h
"""
import os as _os

# One hardware work queue per CUDA stream.  The engine's streams carry
# cross-rank waits (cuStreamWaitValue32); if two streams aliased onto one
# queue (the default is 8 queues), a wait on one would stall the other and
# could close a cycle across ranks.  Must be set before the CUDA context exists.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import _capi  # noqa: E402,F401

__version__ = "0.1.0"
