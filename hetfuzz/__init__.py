"""``import hetfuzz`` for hosts written against the reference's Python package
(proj/python/hetfuzz/__init__.py:3-18): the stateless entry points of the coverage-feedback path,
computed on the B200 through ``paper_2603_12485_b200`` (libhfz.so) -- no reference build needed.

Same names, argument meaning and return types as ``hetfuzz._core`` (proj/python/bindings.cpp):

    MAP_SIZE, HOST_SLOTS                                   bindings.cpp:316-317
    TargetError (a ValueError)                             bindings.cpp:314
    havoc_mutant(data, seed) -> bytes                      bindings.cpp:220-223
    splice_mutant(a, b, seed) -> bytes                     bindings.cpp:225-229
    deterministic_mutants(data) -> list[bytes]             bindings.cpp:213-218

and, for the hot-path OUTPUTS of the two calls that need the simulator (out of scope here):

    signatures(map) -> {"nonzero_slots", "full_sig", "simple_sig"}      the keys run_input returns (:199-202)
    replay_signatures(maps) -> {"full_sigs", "simple_sigs", ...}        the keys replay_sequence returns (:278-284)

where a map is one execution's raw record or its (slot, count) pairs.  The campaign-level functions
(run_campaign, run_input, replay_sequence, showmap, bench, compare_kernel, targets, seeded_key_hex) drive
the reference's runtime simulator; they are available from the reference's own module built against this
repository's headers (oracle/build_dropin.sh) and raise here with that pointer.
"""
from paper_2603_12485_b200 import (HOST_SLOTS, MAP_SIZE, TargetError, deterministic_mutants, havoc_batch,  # noqa: F401
                                   havoc_mutant, replay_signatures, signatures, splice_mutant)

__all__ = ["HOST_SLOTS", "MAP_SIZE", "TargetError", "deterministic_mutants", "havoc_mutant", "splice_mutant",
           "signatures", "replay_signatures", "havoc_batch"]

_NEEDS_RUNTIME = ("run_campaign", "run_input", "replay_sequence", "showmap", "bench", "compare_kernel", "targets",
                  "seeded_key_hex")


def __getattr__(name):
    if name in _NEEDS_RUNTIME:
        raise AttributeError(
            f"hetfuzz.{name} drives the reference's runtime simulator, which this package does not rebuild; build the "
            "reference's module against this repository's headers (oracle/build_dropin.sh, INTEGRATION.md section 1) "
            "or use signatures() / replay_signatures() for the hot-path outputs of a map you already hold")
    raise AttributeError(f"module 'hetfuzz' has no attribute {name!r}")
