"""B200-native coverage-feedback core of hetfuzz / cuFuzz (arXiv 2603.12485).

The package is a thin host layer over ``libhfz.so`` (hand-written sm_100a CUDA
behind the C-ABI of ``include/hfz.h``).  It mirrors the reference's Python
surface (``proj/python/bindings.cpp:310-350``): ``MAP_SIZE``, ``HOST_SLOTS``,
``havoc_mutant``, ``splice_mutant``, ``deterministic_mutants`` keep their names
and argument meaning, and batched calls are added beside them.

Importing the package loads the shared library and fails loudly if it has not
been built; there is no CPU fallback anywhere in the product path.
"""
from ._lib import HfzError, LIB_PATH, lib  # noqa: F401  (loads libhfz.so or raises)
from .api import (Context, SigSet, dispatch_batch, GAMMA, HOST_SLOTS, MAP_SIZE, MAX_INPUT_BYTES, i64_to_u64,  # noqa: F401
                  record_bytes, rng_jump, rng_split, u64_to_i64)
from .binding import (TargetError, deterministic_mutants, havoc_mutant, splice_mutant,  # noqa: F401
                      feedback_batch, feedback_batch_sparse, feedback_batch_compact, havoc_batch,
                      default_context, signatures, replay_signatures)

__all__ = ["Context", "MAP_SIZE", "HOST_SLOTS", "MAX_INPUT_BYTES", "havoc_mutant", "splice_mutant",
           "deterministic_mutants", "feedback_batch", "feedback_batch_sparse", "feedback_batch_compact", "havoc_batch", "default_context", "signatures", "replay_signatures",
           "record_bytes", "rng_jump", "rng_split", "HfzError", "TargetError"]
