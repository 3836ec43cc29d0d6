"""ctypes binding of the C-ABI in include/hfz.h (libhfz.so, built in-tree by
``__graft_entry__.build()`` / ``make -C paper_2603_12485_b200/csrc``).

There is no fallback: if the shared library is missing or a symbol is absent
the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhfz.so")

HFZ_OK, HFZ_EINVAL, HFZ_ECUDA, HFZ_ENOMEM, HFZ_ECAP, HFZ_ENCCL = range(6)

_vp = C.c_void_p
_u64 = C.c_uint64
_u32 = C.c_uint32

# name -> (restype, argtypes); mirrors include/hfz.h one to one
PROTOTYPES = {
    "hfz_version": (C.c_int, []),
    "hfz_last_error": (C.c_char_p, []),
    "hfz_ctx_create": (C.c_int, [C.POINTER(_vp), C.c_int, _u32, _vp]),
    "hfz_ctx_destroy": (C.c_int, [_vp]),
    "hfz_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "hfz_ctx_sync": (C.c_int, [_vp]),
    "hfz_ctx_map_slots": (_u32, [_vp]),
    "hfz_record_bytes": (_u64, [_u32]),
    "hfz_ctx_set_option": (C.c_int, [_vp, C.c_char_p, C.c_int64]),
    "hfz_ctx_launch_count": (_u64, [_vp]),
    "hfz_ctx_get_stat": (C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_double)]),
    "hfz_feedback_batch": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfz_feedback_batch_host": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfz_feedback_batch_sparse": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfz_feedback_batch_sparse_host": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfz_feedback_batch_compact_host": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfz_feedback_batch_packed_host": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfz_feedback_batch_packed_host_v": (C.c_int, [_vp, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfz_expand_sparse": (C.c_int, [_vp, _vp, _vp, _u64, _vp]),
    "hfz_host_alloc": (C.c_int, [C.POINTER(_vp), _u64]),
    "hfz_host_free": (C.c_int, [_vp]),
    "hfz_feedback_scan": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfz_feedback_resolve": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _vp, _u32, _u32, _vp]),
    "hfz_feedback_resolve_peers": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _vp, _u32, _u32, _vp]),
    "hfz_peer_alloc": (C.c_int, [_vp, _u64, C.POINTER(_vp), _vp]),
    "hfz_peer_open": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "hfz_peer_close": (C.c_int, [_vp, _vp]),
    "hfz_peer_free": (C.c_int, [_vp, _vp]),
    "hfz_virgin_merge": (C.c_int, [_vp, _vp, _vp, _vp, _u32]),
    "hfz_feedback_resolve_allgather": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _u32, _u32, _vp]),
    "hfz_edge_record_batch": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _u64, _u64, _vp, _vp]),
    "hfz_edge_record_batch_lists": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _u32, _vp]),
    "hfz_host_edge_record_batch": (C.c_int, [_vp, _vp, _vp, _u64, _vp]),
    "hfz_havoc_max_out": (_u64, [_u64]),
    "hfz_havoc_batch": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp]),
    "hfz_splice_batch": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "hfz_deterministic_count": (_u64, [_vp, _u64]),
    "hfz_deterministic_batch": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _u64]),
    "hfz_havoc_batch_host": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp]),
    "hfz_splice_batch_host": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "hfz_deterministic_host": (C.c_int, [_vp, _vp, _u64, _vp, _u64]),
    "hfz_havoc_serial_host": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "hfz_havoc_serial_plan": (C.c_int, [_vp, _vp, _u64, _vp, _vp]),
    "hfz_sigset_create": (C.c_int, [_vp, _u64, C.POINTER(_vp)]),
    "hfz_sigset_destroy": (C.c_int, [_vp]),
    "hfz_sigset_size": (C.c_int, [_vp, C.POINTER(_u64)]),
    "hfz_sigset_seen_insert": (C.c_int, [_vp, _vp, _vp, _u64, _vp]),
    "hfz_dispatch_batch": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _u64, C.c_int, _vp, _vp, _vp]),
    "hfz_rng_jump": (_u64, [_u64, _u64]),
    "hfz_rng_next": (_u64, [C.POINTER(_u64)]),
    "hfz_rng_below": (_u64, [C.POINTER(_u64), _u64]),
    "hfz_rng_split": (_u64, [C.POINTER(_u64), _u64]),
}


class HfzError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hfz error {code}: {msg}")
        self.code = code


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2603_12485_b200/csrc` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)  # AttributeError if the symbol is not exported
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


def check(rc: int) -> None:
    if rc != HFZ_OK:
        raise HfzError(rc, (lib.hfz_last_error() or b"").decode("utf-8", "replace"))
