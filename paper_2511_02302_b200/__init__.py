"""paper_2511_02302_b200 -- B200-native (sm_100a) FP8-Flow-MoE hot path (arXiv 2511.02302).

The product is the C-ABI library ``libfp8flow.so`` (include/fp8flow.h, sources in csrc/); this
package holds its thin ctypes binding (``fp8flow``), the in-tree build script and the
expert-group sharding helpers used by bench.py.  It never imports the test oracle.
"""
from . import fp8flow  # noqa: F401
from .fp8flow import *  # noqa: F401,F403
