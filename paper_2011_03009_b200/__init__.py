"""B200-native volume-potential harmonic solver (arXiv 2011.03009), drop-in for the
reference's ``namespace fus`` hot path.  Numerics: libfusg.so (sm_100a CUDA kernels behind
the C-ABI in include/fusg.h).  ``fus`` mirrors the reference's C++ API."""
from . import fus  # noqa: F401
from ._lib import LIB_PATH, FusgError  # noqa: F401
