"""ctypes/numpy front-end of the CPU oracles.  TEST INFRASTRUCTURE ONLY.

Two checkers live behind this module:

* ``Port``  -- ``oracle/libhfz_oracle.so``, the plain-C restatement
  (``oracle/hfz_oracle.c``), map size is a run-time parameter.
* ``Ref``   -- ``oracle/_ref/libhetfuzz_ref*.so``, the UNMODIFIED reference
  compiled from ``/root/reference/proj/src`` by ``oracle/build_ref.sh``
  (fixed map size per build: 65,536 or the patched 262,144).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GAMMA = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1

_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)


def _p(a, t):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


def record_bytes(S: int) -> int:
    """Raw bytes of one exec's map: H u8 host counters + H u32 device counters."""
    return (S // 2) * 5


def build(ref: bool = True) -> None:
    """Compile the C restatement and, when /root/reference exists, the reference."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref:
        subprocess.run([os.path.join(HERE, "build_ref.sh")], check=True)


class _FeedbackMixin:
    def feedback_batch(self, raw, n_exec, S, virgin, edge_counts, want_classed=False):
        """Ordered fold (src/engine.cpp:471-478).  Mutates virgin/edge_counts.
        Returns dict(admit, sig_full, sig_simple, nnz[, classed])."""
        raw = np.ascontiguousarray(raw, dtype=np.uint8).reshape(-1)
        assert raw.size == n_exec * record_bytes(S)
        assert virgin.dtype == np.uint8 and virgin.size == S
        assert edge_counts.dtype == np.uint64 and edge_counts.size == 2
        admit = np.zeros(n_exec, np.uint8)
        sf = np.zeros(n_exec, np.uint64)
        ss = np.zeros(n_exec, np.uint64)
        nnz = np.zeros(n_exec, np.uint32)
        classed = np.zeros((n_exec, S), np.uint8) if want_classed else None
        self._feedback(raw, n_exec, S, virgin, edge_counts, classed, admit, sf, ss, nnz)
        out = dict(admit=admit, sig_full=sf, sig_simple=ss, nnz=nnz)
        if want_classed:
            out["classed"] = classed
        return out


class _BatchMixin:
    """Range calls for the CPU legs of bench.py and full-size checks: ctypes releases the GIL, so one
    call per host thread runs in parallel."""

    def havoc_range(self, in_bytes, in_off, first, count, state, out, out_off, out_len):
        """Slots [first, first+count): state (u64[n]) advanced in place, out/out_len filled."""
        f = self.lib.orc_havoc_batch if self.kind == "port" else self.lib.ref_havoc_batch
        rc = f(_p(in_bytes, _u8p), _p(in_off, _u64p), first, count, _p(state, _u64p), _p(out, _u8p),
               _p(out_off, _u64p), _p(out_len, _u64p))
        assert rc == 0, rc

    def edge_record_range(self, tr, first, count, S, raw, ev):
        """Execs [first, first+count) of trace batch `tr` (dict of contiguous arrays in
        hfz_edge_record_batch layout) -> device halves of raw (records) and warp events."""
        args = [_p(tr["launch_off"], _u64p), _p(tr["dims"], _u32p), _p(tr["thread_off"], _u64p),
                _p(tr["ev_off"], _u64p), _p(tr["sites"], _u32p), first, count]
        if self.kind == "port":
            rc = self.lib.orc_edge_record_range(*args, S, _p(raw, _u8p), _p(ev, _u64p))
        else:
            assert S == self.S
            rc = self.lib.ref_edge_record_range(*args, _p(raw, _u8p), _p(ev, _u64p))
        assert rc == 0, rc


class Port(_FeedbackMixin, _BatchMixin):
    """Plain-C restatement (kind "port")."""

    kind = "port"

    def __init__(self):
        path = os.path.join(HERE, "libhfz_oracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_classify_host.restype = C.c_uint8
        L.orc_classify_host.argtypes = [C.c_uint64]
        L.orc_classify_device.restype = C.c_uint8
        L.orc_classify_device.argtypes = [C.c_uint64]
        L.orc_device_edge_index.restype = C.c_uint32
        L.orc_device_edge_index.argtypes = [C.c_uint32] * 3
        L.orc_feedback_batch.restype = C.c_int
        L.orc_feedback_batch.argtypes = [_u8p, C.c_uint64, C.c_uint32, _u8p, _u64p, _u8p, _u8p,
                                         _u64p, _u64p, _u32p]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_next.argtypes = [_u64p]
        L.orc_rng_below.restype = C.c_uint64
        L.orc_rng_below.argtypes = [_u64p, C.c_uint64]
        L.orc_rng_split.restype = C.c_uint64
        L.orc_rng_split.argtypes = [_u64p, C.c_uint64]
        L.orc_havoc_max_out.restype = C.c_uint64
        L.orc_havoc_max_out.argtypes = [C.c_uint64]
        L.orc_havoc.restype = C.c_int
        L.orc_havoc.argtypes = [_u8p, C.c_uint64, _u64p, _u8p, _u64p]
        L.orc_splice.restype = C.c_int
        L.orc_splice.argtypes = [_u8p, C.c_uint64, _u8p, C.c_uint64, _u64p, _u8p, _u64p]
        L.orc_deterministic.restype = C.c_uint64
        L.orc_deterministic.argtypes = [_u8p, C.c_uint64, _u8p]
        L.orc_host_edge_record.restype = C.c_int
        L.orc_host_edge_record.argtypes = [_u16p, C.c_uint64, C.c_uint32, _u8p, _u64p]
        L.orc_edge_record_exec.restype = C.c_int
        L.orc_edge_record_exec.argtypes = [_u32p, C.c_uint32, _u64p, _u32p, C.c_uint32, _u32p, _u64p]
        L.orc_edge_record_batch.restype = C.c_int
        L.orc_edge_record_batch.argtypes = [_u64p, _u32p, _u64p, _u64p, _u32p, C.c_uint64,
                                            C.c_uint32, _u8p, _u64p]
        L.orc_havoc_batch.restype = C.c_int
        L.orc_havoc_batch.argtypes = [_u8p, _u64p, C.c_uint64, C.c_uint64, _u64p, _u8p, _u64p, _u64p]
        L.orc_edge_record_range.restype = C.c_int
        L.orc_edge_record_range.argtypes = [_u64p, _u32p, _u64p, _u64p, _u32p, C.c_uint64, C.c_uint64,
                                            C.c_uint32, _u8p, _u64p]
        L.orc_rank_delta.restype = C.c_int
        L.orc_rank_delta.argtypes = [_u8p, C.c_uint64, C.c_uint32, _u8p, _u8p]

    # -- ladders / indices
    def classify_host(self, c):
        return self.lib.orc_classify_host(c & MASK64)

    def classify_device(self, c):
        return self.lib.orc_classify_device(c & MASK64)

    def device_edge_index(self, prev, cur, H=32768):
        return self.lib.orc_device_edge_index(prev, cur, H)

    def map_sizes(self):
        return None  # any power of two

    def _feedback(self, raw, n, S, virgin, counts, classed, admit, sf, ss, nnz):
        rc = self.lib.orc_feedback_batch(_p(raw, _u8p), n, S, _p(virgin, _u8p), _p(counts, _u64p),
                                         _p(classed, _u8p), _p(admit, _u8p), _p(sf, _u64p),
                                         _p(ss, _u64p), _p(nnz, _u32p))
        assert rc == 0

    def rank_delta(self, raw, n_exec, S, v0):
        raw = np.ascontiguousarray(raw, dtype=np.uint8).reshape(-1)
        out = np.zeros(S, np.uint8)
        self.lib.orc_rank_delta(_p(raw, _u8p), n_exec, S, _p(np.ascontiguousarray(v0), _u8p),
                                _p(out, _u8p))
        return out

    # -- rng
    def rng_next(self, state):
        s = C.c_uint64(state)
        v = self.lib.orc_rng_next(C.byref(s))
        return v, s.value

    def rng_below(self, state, n):
        s = C.c_uint64(state)
        v = self.lib.orc_rng_below(C.byref(s), n)
        return v, s.value

    def rng_split(self, state, tag):
        s = C.c_uint64(state)
        child = self.lib.orc_rng_split(C.byref(s), tag)
        return child, s.value

    # -- mutators
    def havoc(self, data: bytes, state: int):
        """-> (mutant bytes, end state, draws)"""
        inp = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        out = np.zeros(len(data) + 64 * 16 + 32, np.uint8)
        s = C.c_uint64(state)
        n = C.c_uint64(0)
        rc = self.lib.orc_havoc(_p(inp, _u8p), len(data), C.byref(s), _p(out, _u8p), C.byref(n))
        assert rc == 0
        draws = ((s.value - state) & MASK64) * pow(GAMMA, -1, 1 << 64) & MASK64
        return out[: n.value].tobytes(), s.value, draws

    def splice(self, a: bytes, b: bytes, state: int):
        ia = np.frombuffer(a, np.uint8).copy() if len(a) else np.zeros(1, np.uint8)
        ib = np.frombuffer(b, np.uint8).copy() if len(b) else np.zeros(1, np.uint8)
        out = np.zeros(len(a) + len(b) + 1, np.uint8)
        s = C.c_uint64(state)
        n = C.c_uint64(0)
        self.lib.orc_splice(_p(ia, _u8p), len(a), _p(ib, _u8p), len(b), C.byref(s),
                            _p(out, _u8p), C.byref(n))
        return out[: n.value].tobytes(), s.value

    def deterministic(self, data: bytes):
        inp = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        cnt = self.lib.orc_deterministic(_p(inp, _u8p), len(data), None)
        out = np.zeros(max(1, cnt * len(data)), np.uint8)
        self.lib.orc_deterministic(_p(inp, _u8p), len(data), _p(out, _u8p))
        L = len(data)
        return [out[i * L:(i + 1) * L].tobytes() for i in range(cnt)]

    # -- edge recording
    def host_edge_record(self, sites, H=32768):
        sites = np.ascontiguousarray(sites, dtype=np.uint16)
        half = np.zeros(H, np.uint8)
        viol = C.c_uint64(0)
        self.lib.orc_host_edge_record(_p(sites, _u16p), sites.size, H, _p(half, _u8p), C.byref(viol))
        return half, viol.value

    def edge_record_exec(self, dims, ev_off, sites, H=32768, counters=None):
        """dims: (n_launch,6) u32; ev_off: (n_threads+1,) u64; sites u32.
        -> (counters[H] u32, warp_events)"""
        dims = np.ascontiguousarray(dims, dtype=np.uint32).reshape(-1, 6)
        ev_off = np.ascontiguousarray(ev_off, dtype=np.uint64)
        sites = np.ascontiguousarray(sites, dtype=np.uint32)
        if sites.size == 0:
            sites = np.zeros(1, np.uint32)
        if counters is None:
            counters = np.zeros(H, np.uint32)
        ev = C.c_uint64(0)
        rc = self.lib.orc_edge_record_exec(_p(dims, _u32p), dims.shape[0], _p(ev_off, _u64p),
                                           _p(sites, _u32p), H, _p(counters, _u32p), C.byref(ev))
        assert rc == 0
        return counters, ev.value

    def edge_record_batch(self, launch_off, dims, thread_off, ev_off, sites, n_exec, S, raw=None):
        launch_off = np.ascontiguousarray(launch_off, dtype=np.uint64)
        dims = np.ascontiguousarray(dims, dtype=np.uint32)
        thread_off = np.ascontiguousarray(thread_off, dtype=np.uint64)
        ev_off = np.ascontiguousarray(ev_off, dtype=np.uint64)
        sites = np.ascontiguousarray(sites, dtype=np.uint32)
        if sites.size == 0:
            sites = np.zeros(1, np.uint32)
        if raw is None:
            raw = np.zeros(n_exec * record_bytes(S), np.uint8)
        ev = np.zeros(n_exec, np.uint64)
        rc = self.lib.orc_edge_record_batch(_p(launch_off, _u64p), _p(dims, _u32p),
                                            _p(thread_off, _u64p), _p(ev_off, _u64p),
                                            _p(sites, _u32p), n_exec, S, _p(raw, _u8p), _p(ev, _u64p))
        assert rc == 0
        return raw, ev


class Ref(_FeedbackMixin, _BatchMixin):
    """The compiled, unmodified reference (kind "reference")."""

    kind = "reference"

    @staticmethod
    def path(S=65536):
        name = "libhetfuzz_ref.so" if S == 65536 else f"libhetfuzz_ref_{S}.so"
        return os.path.join(HERE, "_ref", name)

    @classmethod
    def available(cls, S=65536):
        return os.path.exists(cls.path(S))

    def __init__(self, S=65536):
        self.S = S
        L = self.lib = C.CDLL(self.path(S))
        L.ref_map_size.restype = C.c_uint32
        assert L.ref_map_size() == S
        L.ref_classify_host.restype = C.c_uint8
        L.ref_classify_host.argtypes = [C.c_uint64]
        L.ref_classify_device.restype = C.c_uint8
        L.ref_classify_device.argtypes = [C.c_uint64]
        L.ref_device_edge_index.restype = C.c_uint32
        L.ref_device_edge_index.argtypes = [C.c_uint32] * 2
        L.ref_maps_create.restype = C.c_void_p
        L.ref_maps_create.argtypes = [_u8p, C.c_uint64]
        L.ref_maps_free.argtypes = [C.c_void_p]
        L.ref_feedback_run.restype = C.c_int
        L.ref_feedback_run.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, _u8p, _u64p, _u8p, _u8p,
                                       _u64p, _u64p, _u32p]
        L.ref_rng_next.restype = C.c_uint64
        L.ref_rng_next.argtypes = [_u64p]
        L.ref_rng_below.restype = C.c_uint64
        L.ref_rng_below.argtypes = [_u64p, C.c_uint64]
        L.ref_rng_split.restype = C.c_uint64
        L.ref_rng_split.argtypes = [_u64p, C.c_uint64]
        L.ref_host_edge_record.restype = C.c_int
        L.ref_host_edge_record.argtypes = [_u16p, C.c_uint64, _u8p, _u64p]
        L.ref_edge_record_exec.restype = C.c_int
        L.ref_edge_record_exec.argtypes = [_u32p, C.c_uint32, _u64p, _u32p, _u32p, _u64p]
        L.ref_edge_record_range.restype = C.c_int
        L.ref_edge_record_range.argtypes = [_u64p, _u32p, _u64p, _u64p, _u32p, C.c_uint64, C.c_uint64, _u8p, _u64p]
        self.has_engine = hasattr(L, "ref_havoc")
        if self.has_engine:
            L.ref_havoc_batch.restype = C.c_int
            L.ref_havoc_batch.argtypes = [_u8p, _u64p, C.c_uint64, C.c_uint64, _u64p, _u8p, _u64p, _u64p]
            L.ref_havoc.restype = C.c_int
            L.ref_havoc.argtypes = [_u8p, C.c_uint64, _u64p, _u8p, _u64p]
            L.ref_splice.restype = C.c_int
            L.ref_splice.argtypes = [_u8p, C.c_uint64, _u8p, C.c_uint64, _u64p, _u8p, _u64p]
            L.ref_deterministic.restype = C.c_uint64
            L.ref_deterministic.argtypes = [_u8p, C.c_uint64, _u8p]

    def classify_host(self, c):
        return self.lib.ref_classify_host(c & MASK64)

    def classify_device(self, c):
        return self.lib.ref_classify_device(c & MASK64)

    def device_edge_index(self, prev, cur, H=None):
        return self.lib.ref_device_edge_index(prev, cur)

    # maps handle API (construction outside timed regions)
    def maps_create(self, raw, n_exec):
        raw = np.ascontiguousarray(raw, dtype=np.uint8).reshape(-1)
        assert raw.size == n_exec * record_bytes(self.S)
        return self.lib.ref_maps_create(_p(raw, _u8p), n_exec)

    def maps_free(self, h):
        self.lib.ref_maps_free(h)

    def feedback_run(self, h, first, count, virgin, counts, outs=None):
        """outs: optional dict(admit, sig_full, sig_simple, nnz, classed) of arrays."""
        o = outs or {}
        return self.lib.ref_feedback_run(h, first, count, _p(virgin, _u8p), _p(counts, _u64p),
                                         _p(o.get("classed"), _u8p), _p(o.get("admit"), _u8p),
                                         _p(o.get("sig_full"), _u64p), _p(o.get("sig_simple"), _u64p),
                                         _p(o.get("nnz"), _u32p))

    def _feedback(self, raw, n, S, virgin, counts, classed, admit, sf, ss, nnz):
        assert S == self.S
        h = self.maps_create(raw, n)
        try:
            rc = self.lib.ref_feedback_run(h, 0, n, _p(virgin, _u8p), _p(counts, _u64p),
                                           _p(classed, _u8p), _p(admit, _u8p), _p(sf, _u64p),
                                           _p(ss, _u64p), _p(nnz, _u32p))
            assert rc == 0
        finally:
            self.maps_free(h)

    def rng_next(self, state):
        s = C.c_uint64(state)
        v = self.lib.ref_rng_next(C.byref(s))
        return v, s.value

    def rng_below(self, state, n):
        s = C.c_uint64(state)
        v = self.lib.ref_rng_below(C.byref(s), n)
        return v, s.value

    def rng_split(self, state, tag):
        s = C.c_uint64(state)
        child = self.lib.ref_rng_split(C.byref(s), tag)
        return child, s.value

    def havoc(self, data: bytes, state: int):
        inp = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        out = np.zeros(len(data) + 64 * 16 + 32, np.uint8)
        s = C.c_uint64(state)
        n = C.c_uint64(0)
        rc = self.lib.ref_havoc(_p(inp, _u8p), len(data), C.byref(s), _p(out, _u8p), C.byref(n))
        assert rc == 0
        draws = ((s.value - state) & MASK64) * pow(GAMMA, -1, 1 << 64) & MASK64
        return out[: n.value].tobytes(), s.value, draws

    def splice(self, a: bytes, b: bytes, state: int):
        ia = np.frombuffer(a, np.uint8).copy() if len(a) else np.zeros(1, np.uint8)
        ib = np.frombuffer(b, np.uint8).copy() if len(b) else np.zeros(1, np.uint8)
        out = np.zeros(len(a) + len(b) + 1, np.uint8)
        s = C.c_uint64(state)
        n = C.c_uint64(0)
        self.lib.ref_splice(_p(ia, _u8p), len(a), _p(ib, _u8p), len(b), C.byref(s),
                            _p(out, _u8p), C.byref(n))
        return out[: n.value].tobytes(), s.value

    def deterministic(self, data: bytes):
        inp = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        cnt = self.lib.ref_deterministic(_p(inp, _u8p), len(data), None)
        out = np.zeros(max(1, cnt * len(data)), np.uint8)
        self.lib.ref_deterministic(_p(inp, _u8p), len(data), _p(out, _u8p))
        L = len(data)
        return [out[i * L:(i + 1) * L].tobytes() for i in range(cnt)]

    def host_edge_record(self, sites, H=None):
        sites = np.ascontiguousarray(sites, dtype=np.uint16)
        half = np.zeros(self.S // 2, np.uint8)
        viol = C.c_uint64(0)
        self.lib.ref_host_edge_record(_p(sites, _u16p), sites.size, _p(half, _u8p), C.byref(viol))
        return half, viol.value

    def edge_record_exec(self, dims, ev_off, sites, H=None, counters=None):
        assert counters is None, "the reference runtime always starts from zero counters"
        dims = np.ascontiguousarray(dims, dtype=np.uint32).reshape(-1, 6)
        ev_off = np.ascontiguousarray(ev_off, dtype=np.uint64)
        sites = np.ascontiguousarray(sites, dtype=np.uint32)
        if sites.size == 0:
            sites = np.zeros(1, np.uint32)
        counters = np.zeros(self.S // 2, np.uint32)
        ev = C.c_uint64(0)
        rc = self.lib.ref_edge_record_exec(_p(dims, _u32p), dims.shape[0], _p(ev_off, _u64p),
                                           _p(sites, _u32p), _p(counters, _u32p), C.byref(ev))
        assert rc == 0, rc
        return counters, ev.value


def best_checker(S=65536):
    """The reference when its build for S exists, else the C restatement."""
    return Ref(S) if Ref.available(S) else Port()
