"""B200-native FHP lattice-gas engine (drop-in for the reference's fhp::advance path).

Native pieces: paper_1208_2428_b200/lib/libfhpg.so (sm_100a kernels + C ABI,
include/fhpg.h) and the C++ host layer (paper_1208_2428_b200/host). This
package is the thin Python binding used by tests and bench.py.
"""
from .engine import (Engine, FhpgError, FhpgInvalidArgument, bernoulli_threshold,  # noqa: F401
                     build_table, load_library, state_digest, validate_table)
