"""B200-native maximal biclique enumeration (cuMBE, arXiv 2401.05039 hot path).

The product is libmbe.so (include/mbe.h): hand-written sm_100a CUDA kernels
behind a C ABI.  This package holds its ctypes binding (``_lib``), the build
script (``build``), the seeded synthetic input generators (``inputs``, no
method arithmetic) and the multi-GPU driver (``dist``).  Importing the package
does not load the library; the first call does, and fails loudly if it is
missing (no CPU fallback).
"""
from ._lib import (  # noqa: F401
    EXPORTED_SYMBOLS,
    MBE_ARENA_GROW,
    MBE_NO_RS,
    ClaimCounter,
    MBE_NO_ANTICHAIN,
    MBE_NO_STEAL,
    MBE_NO_TWIN,
    MBE_STEAL_HALF,
    MBE_STEAL_ONE,
    MBE_STATS,
    MBEError,
    MBEGraph,
    Result,
    load_library,
    make_config,
    make_output,
    mbe_enumerate,
    mbe_format_listing,
    mbe_free,
    mbe_get_info,
    mbe_last_error_detail,
    mbe_load_csr,
    mbe_release_workspaces,
    mbe_strerror,
)
