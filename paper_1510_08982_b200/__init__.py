"""B200-native (sm_100a) FTCS heat-equation hot path of arXiv 1510.08982.

Synchronous and bounded-stale asynchronous FTCS updates behind the reference's
solver API (see include/heat_b200.h for the C-ABI, ``heat`` for the Python
mirror of namespace heat).  Build the CUDA library with
``python -m paper_1510_08982_b200.build``.
"""
from .heat import *  # noqa: F401,F403
from . import heat  # noqa: F401
