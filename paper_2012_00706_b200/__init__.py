"""B200-native hot path of the mixed-precision interpolative decomposition (arXiv 2012.00706).

libmpid.so (csrc/, C ABI in include/mpid.h) holds every kernel of the path;
`mpid` is the thin ctypes binding.  Build with `python -m paper_2012_00706_b200.build`.
"""
from . import mpid  # noqa: F401
