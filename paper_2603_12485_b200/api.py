"""Host-side wrapper of the C-ABI (include/hfz.h) over torch device tensors.

PyTorch is plumbing only (device memory, streams, torch.distributed); every
computation below is a call into libhfz.so.  Method names follow the reference's
vocabulary (classify_trace / has_new_bits / trace_signature ->
``feedback_batch``; ``havoc_mutant`` -> ``havoc_batch``; DeviceThreadCtx::edge ->
``edge_record_batch``).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

MAP_SIZE = 65536          # kMapSize, include/hetfuzz/coverage.hpp:13
HOST_SLOTS = MAP_SIZE // 2  # kHostSlots, coverage.hpp:14
MAX_INPUT_BYTES = 1 << 20   # kMaxInputBytes, engine.hpp:17
GAMMA = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def record_bytes(S: int = MAP_SIZE) -> int:
    return int(lib.hfz_record_bytes(S))


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    assert t.is_contiguous()
    return C.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor, device, dtype=None):
    assert t.is_cuda and t.device == device, f"tensor must live on {device}"
    if dtype is not None:
        assert t.dtype == dtype, f"expected {dtype}, got {t.dtype}"
    return t


class Context:
    """One hfz_ctx: one host thread driving one GPU (SPEC.md:124-125 threading contract)."""

    def __init__(self, device: int | torch.device = 0, map_slots: int = MAP_SIZE):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2603_12485_b200 needs a CUDA device; there is no CPU fallback")
        self.device = torch.device("cuda", device if isinstance(device, int) else device.index or 0)
        self.S = int(map_slots)
        self.H = self.S // 2
        self.rec = record_bytes(self.S)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            check(lib.hfz_ctx_create(C.byref(h), self.device.index, self.S, C.c_void_p(stream)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hfz_ctx_destroy(self._h)
            self._h = None

    __del__ = close

    def _sync_stream(self):
        check(lib.hfz_ctx_set_stream(self._h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def set_option(self, key: str, value: int):
        check(lib.hfz_ctx_set_option(self._h, key.encode(), int(value)))

    def get_stat(self, key: str) -> float:
        v = C.c_double(0)
        check(lib.hfz_ctx_get_stat(self._h, key.encode(), C.byref(v)))
        return float(v.value)

    @property
    def launch_count(self) -> int:
        return int(lib.hfz_ctx_launch_count(self._h))

    def synchronize(self):
        self._sync_stream()
        check(lib.hfz_ctx_sync(self._h))

    # ---- allocation helpers -------------------------------------------------
    def new_virgin(self) -> torch.Tensor:
        return torch.zeros(self.S, dtype=torch.uint8, device=self.device)

    def new_edge_counts(self) -> torch.Tensor:
        return torch.zeros(2, dtype=torch.int64, device=self.device)

    # ---- K2 -----------------------------------------------------------------
    def feedback_batch(self, raw: torch.Tensor, virgin: torch.Tensor, edge_counts: torch.Tensor,
                       want_classed: bool = False, want_nnz: bool = True, out: dict | None = None):
        """Fold `raw` (n_exec records) into `virgin` in exec order.  Returns a dict of device
        tensors: admit (u8), sig_full / sig_simple (int64 bit patterns of the u64
        signatures), nnz (int32), optionally classed (n_exec x S u8)."""
        _dev(raw, self.device, torch.uint8)
        _dev(virgin, self.device, torch.uint8)
        _dev(edge_counts, self.device, torch.int64)
        n = raw.numel() // self.rec
        assert raw.numel() == n * self.rec and virgin.numel() == self.S and edge_counts.numel() == 2
        o = out or {}
        if "admit" not in o:
            o["admit"] = torch.empty(n, dtype=torch.uint8, device=self.device)
            o["sig_full"] = torch.empty(n, dtype=torch.int64, device=self.device)
            o["sig_simple"] = torch.empty(n, dtype=torch.int64, device=self.device)
        if want_nnz and "nnz" not in o:
            o["nnz"] = torch.empty(n, dtype=torch.int32, device=self.device)
        if want_classed and "classed" not in o:
            o["classed"] = torch.empty((n, self.S), dtype=torch.uint8, device=self.device)
        self._sync_stream()
        check(lib.hfz_feedback_batch(self._h, _ptr(raw), n, _ptr(virgin), _ptr(edge_counts),
                                     _ptr(o.get("classed")) if want_classed else None,
                                     _ptr(o["admit"]), _ptr(o["sig_full"]), _ptr(o["sig_simple"]),
                                     _ptr(o.get("nnz")) if want_nnz else None))
        return o

    def feedback_scan(self, raw, virgin_v0, want_classed=False, out: dict | None = None):
        """Rank-local half of the sharded step: signatures, nnz and this rank's novelty delta."""
        _dev(raw, self.device, torch.uint8)
        n = raw.numel() // self.rec
        o = out or {}
        if "sig_full" not in o:
            o["sig_full"] = torch.empty(n, dtype=torch.int64, device=self.device)
            o["sig_simple"] = torch.empty(n, dtype=torch.int64, device=self.device)
            o["nnz"] = torch.empty(n, dtype=torch.int32, device=self.device)
        if "delta" not in o:
            o["delta"] = torch.empty(self.S, dtype=torch.uint8, device=self.device)
        if want_classed and "classed" not in o:
            o["classed"] = torch.empty((n, self.S), dtype=torch.uint8, device=self.device)
        self._sync_stream()
        check(lib.hfz_feedback_scan(self._h, _ptr(raw), n, _ptr(virgin_v0),
                                    _ptr(o.get("classed")) if want_classed else None,
                                    _ptr(o["sig_full"]), _ptr(o["sig_simple"]), _ptr(o["nnz"]),
                                    _ptr(o["delta"])))
        return o

    def feedback_resolve(self, raw, virgin, edge_counts, deltas, n_ranks, rank, admit=None):
        """Second half: exact Admit codes against P_rank and the ordered virgin merge."""
        n = raw.numel() // self.rec
        if admit is None:
            admit = torch.empty(n, dtype=torch.uint8, device=self.device)
        assert deltas.numel() == n_ranks * self.S
        self._sync_stream()
        check(lib.hfz_feedback_resolve(self._h, _ptr(raw), n, _ptr(virgin), _ptr(edge_counts),
                                       _ptr(deltas), n_ranks, rank, _ptr(admit)))
        return admit

    def feedback_resolve_peers(self, raw, virgin, edge_counts, delta_tensors, rank, admit=None):
        """feedback_resolve reading every rank's delta in place: delta_tensors[q] is rank q's delta
        (a tensor, or the device address as an int: own or peer-mapped memory visible from this device)."""
        n = raw.numel() // self.rec
        if admit is None:
            admit = torch.empty(n, dtype=torch.uint8, device=self.device)
        ptrs = (C.c_void_p * len(delta_tensors))(*[t if isinstance(t, int) else t.data_ptr() for t in delta_tensors])
        self._sync_stream()
        check(lib.hfz_feedback_resolve_peers(self._h, _ptr(raw), n, _ptr(virgin), _ptr(edge_counts), ptrs,
                                             len(delta_tensors), rank, _ptr(admit)))
        return admit

    # ---- peer-visible buffers (CUDA IPC) for the collective-free exchange ----
    def peer_alloc(self, nbytes: int):
        """(device address, 64-byte handle) of a zero-filled device buffer other PROCESSES can map (peer_open)."""
        p = C.c_void_p()
        h = (C.c_uint8 * 64)()
        check(lib.hfz_peer_alloc(self._h, int(nbytes), C.byref(p), h))
        return int(p.value), bytes(h)

    def peer_open(self, handle: bytes) -> int:
        p = C.c_void_p()
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        check(lib.hfz_peer_open(self._h, buf, C.byref(p)))
        return int(p.value)

    def peer_close(self, ptr: int):
        check(lib.hfz_peer_close(self._h, C.c_void_p(ptr)))

    def peer_free(self, ptr: int):
        check(lib.hfz_peer_free(self._h, C.c_void_p(ptr)))

    def device_view(self, ptr: int, nbytes: int) -> torch.Tensor:
        """uint8 tensor over device memory the library owns (no copy, no ownership)."""
        class _Raw:
            __cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False), "version": 2}
        return torch.as_tensor(_Raw(), device=self.device)

    def virgin_merge(self, virgin, edge_counts, deltas, n_ranks):
        self._sync_stream()
        check(lib.hfz_virgin_merge(self._h, _ptr(virgin), _ptr(edge_counts), _ptr(deltas), n_ranks))

    def feedback_batch_host(self, raw: np.ndarray, virgin: np.ndarray, edge_counts: np.ndarray,
                            want_classed: bool = False):
        """Same fold through HOST buffers (numpy, ideally pinned): the e2e path of bench.py."""
        n = raw.size // self.rec
        assert raw.dtype == np.uint8 and raw.size == n * self.rec
        assert virgin.dtype == np.uint8 and virgin.size == self.S
        assert edge_counts.dtype == np.uint64 and edge_counts.size == 2
        admit = np.empty(n, np.uint8)
        sf = np.empty(n, np.uint64)
        ss = np.empty(n, np.uint64)
        nnz = np.empty(n, np.uint32)
        classed = np.empty((n, self.S), np.uint8) if want_classed else None
        vp = lambda a: None if a is None else C.c_void_p(a.ctypes.data)
        self._sync_stream()
        check(lib.hfz_feedback_batch_host(self._h, vp(raw), n, vp(virgin), vp(edge_counts), vp(classed),
                                          vp(admit), vp(sf), vp(ss), vp(nnz)))
        o = dict(admit=admit, sig_full=sf, sig_simple=ss, nnz=nnz)
        if want_classed:
            o["classed"] = classed
        return o

    # ---- sparse ingest ------------------------------------------------------
    def feedback_batch_sparse(self, entries: torch.Tensor, entry_off: torch.Tensor, virgin: torch.Tensor,
                              edge_counts: torch.Tensor, want_classed: bool = False, out: dict | None = None):
        """feedback_batch fed with per-exec touched-slot lists: `entries` is an (N, 2) int32 device
        tensor of (slot, count) bit patterns, `entry_off` an int64 device tensor of n_exec+1 offsets."""
        _dev(entries, self.device, torch.int32)
        _dev(entry_off, self.device, torch.int64)
        n = entry_off.numel() - 1
        o = out or {}
        if "admit" not in o:
            o["admit"] = torch.empty(n, dtype=torch.uint8, device=self.device)
            o["sig_full"] = torch.empty(n, dtype=torch.int64, device=self.device)
            o["sig_simple"] = torch.empty(n, dtype=torch.int64, device=self.device)
            o["nnz"] = torch.empty(n, dtype=torch.int32, device=self.device)
        if want_classed and "classed" not in o:
            o["classed"] = torch.empty((n, self.S), dtype=torch.uint8, device=self.device)
        self._sync_stream()
        check(lib.hfz_feedback_batch_sparse(self._h, _ptr(entries), _ptr(entry_off), n, _ptr(virgin),
                                            _ptr(edge_counts), _ptr(o.get("classed")) if want_classed else None,
                                            _ptr(o["admit"]), _ptr(o["sig_full"]), _ptr(o["sig_simple"]),
                                            _ptr(o["nnz"])))
        return o

    def feedback_batch_sparse_host(self, entries: np.ndarray, entry_off: np.ndarray, virgin: np.ndarray,
                                   edge_counts: np.ndarray, want_classed: bool = False):
        """Same through HOST buffers: entries (N, 2) uint32, entry_off (n_exec+1) uint64 (numpy,
        ideally views of pinned memory): the sparse e2e path of bench.py."""
        n = entry_off.size - 1
        assert entries.dtype == np.uint32 and entries.flags.c_contiguous and entries.size % 2 == 0
        assert entry_off.dtype == np.uint64 and entry_off.flags.c_contiguous and n >= 0
        assert virgin.dtype == np.uint8 and virgin.size == self.S
        assert edge_counts.dtype == np.uint64 and edge_counts.size == 2
        admit = np.empty(n, np.uint8)
        sf = np.empty(n, np.uint64)
        ss = np.empty(n, np.uint64)
        nnz = np.empty(n, np.uint32)
        classed = np.empty((n, self.S), np.uint8) if want_classed else None
        vp = lambda a: None if a is None else C.c_void_p(a.ctypes.data)
        self._sync_stream()
        check(lib.hfz_feedback_batch_sparse_host(self._h, vp(entries), vp(entry_off), n, vp(virgin),
                                                 vp(edge_counts), vp(classed), vp(admit), vp(sf), vp(ss),
                                                 vp(nnz)))
        o = dict(admit=admit, sig_full=sf, sig_simple=ss, nnz=nnz)
        if want_classed:
            o["classed"] = classed
        return o

    def feedback_batch_compact_host(self, compact: np.ndarray, compact_off: np.ndarray, wide: np.ndarray | None,
                                    wide_off: np.ndarray | None, virgin: np.ndarray, edge_counts: np.ndarray,
                                    want_classed: bool = False):
        """Touched-slot lists at 4 bytes per pair (maps of <= 65,536 slots): compact = uint32 words
        slot | count << 16 for counts below 65,536, wide = (M, 2) uint32 (slot, count) pairs for the
        larger device counters (None when there are none); one uint64 offsets array per list."""
        n = compact_off.size - 1
        assert compact.dtype == np.uint32 and compact.flags.c_contiguous
        assert compact_off.dtype == np.uint64 and compact_off.flags.c_contiguous
        if wide_off is not None:
            assert wide is not None and wide.dtype == np.uint32 and wide.flags.c_contiguous
            assert wide_off.dtype == np.uint64 and wide_off.size == n + 1 and wide_off.flags.c_contiguous
        assert virgin.dtype == np.uint8 and virgin.size == self.S
        assert edge_counts.dtype == np.uint64 and edge_counts.size == 2
        admit = np.empty(n, np.uint8)
        sf = np.empty(n, np.uint64)
        ss = np.empty(n, np.uint64)
        nnz = np.empty(n, np.uint32)
        classed = np.empty((n, self.S), np.uint8) if want_classed else None
        vp = lambda a: None if a is None else C.c_void_p(a.ctypes.data)
        self._sync_stream()
        check(lib.hfz_feedback_batch_compact_host(self._h, vp(compact), vp(compact_off),
                                                  vp(wide) if wide_off is not None else None, vp(wide_off), n,
                                                  vp(virgin), vp(edge_counts), vp(classed), vp(admit), vp(sf), vp(ss),
                                                  vp(nnz)))
        o = dict(admit=admit, sig_full=sf, sig_simple=ss, nnz=nnz)
        if want_classed:
            o["classed"] = classed
        return o

    def feedback_batch_packed_host(self, host3: np.ndarray, host3_off: np.ndarray, dev17: np.ndarray,
                                   dev17_off: np.ndarray, virgin: np.ndarray, edge_counts: np.ndarray,
                                   want_classed: bool = False):
        """Touched-slot lists of 65,536-slot maps at 3 bytes per host-half slot (uint8 triples slot lo, slot hi,
        count; every exec padded to a multiple of four entries) and 4 bytes per device-half slot (uint32 words
        (slot - 32768) | min(count, 65536) << 15); one uint64 offsets array (in entries) per list."""
        n = host3_off.size - 1
        assert host3.dtype == np.uint8 and host3.flags.c_contiguous and host3.ctypes.data % 4 == 0
        assert dev17.dtype == np.uint32 and dev17.flags.c_contiguous
        for off in (host3_off, dev17_off):
            assert off.dtype == np.uint64 and off.size == n + 1 and off.flags.c_contiguous
        assert virgin.dtype == np.uint8 and virgin.size == self.S
        assert edge_counts.dtype == np.uint64 and edge_counts.size == 2
        admit = np.empty(n, np.uint8)
        sf = np.empty(n, np.uint64)
        ss = np.empty(n, np.uint64)
        nnz = np.empty(n, np.uint32)
        classed = np.empty((n, self.S), np.uint8) if want_classed else None
        vp = lambda a: None if a is None else C.c_void_p(a.ctypes.data)
        self._sync_stream()
        check(lib.hfz_feedback_batch_packed_host(self._h, vp(host3), vp(host3_off), vp(dev17), vp(dev17_off), n,
                                                 vp(virgin), vp(edge_counts), vp(classed), vp(admit), vp(sf), vp(ss),
                                                 vp(nnz)))
        o = dict(admit=admit, sig_full=sf, sig_simple=ss, nnz=nnz)
        if want_classed:
            o["classed"] = classed
        return o

    def expand_sparse(self, entries: torch.Tensor, entry_off: torch.Tensor, raw: torch.Tensor | None = None):
        """Touched-slot lists -> dense raw records on the device."""
        n = entry_off.numel() - 1
        if raw is None:
            raw = torch.empty(n * self.rec, dtype=torch.uint8, device=self.device)
        self._sync_stream()
        check(lib.hfz_expand_sparse(self._h, _ptr(entries), _ptr(entry_off), n, _ptr(raw)))
        return raw

    # ---- K1 -----------------------------------------------------------------
    def edge_record_batch(self, launch_off, dims, thread_off, ev_off, sites, n_exec, raw=None,
                          want_events=True):
        """Device basic-block traces -> device half of each raw record (+ warp_edge_events)."""
        for t in (launch_off, thread_off, ev_off):
            _dev(t, self.device, torch.int64)
        _dev(dims, self.device, torch.int32)
        _dev(sites, self.device, torch.int32)
        if raw is None:
            raw = torch.zeros(n_exec * self.rec, dtype=torch.uint8, device=self.device)
        ev = torch.empty(n_exec, dtype=torch.int64, device=self.device) if want_events else None
        n_launch = thread_off.numel() - 1
        self._sync_stream()
        check(lib.hfz_edge_record_batch(self._h, _ptr(launch_off), _ptr(dims), _ptr(thread_off),
                                        _ptr(ev_off), _ptr(sites), n_exec, n_launch, _ptr(raw),
                                        _ptr(ev)))
        return raw, ev

    def edge_record_batch_lists(self, launch_off, dims, thread_off, ev_off, sites, n_exec, cap=6144, raw=None,
                                want_events=True, out=None):
        """Device basic-block traces -> per-exec touched-slot lists at a fixed stride of `cap` pairs (the
        form feedback_batch_sparse folds; entry_off = arange(n_exec + 1) * cap), optionally the dense
        records too (`raw`).  Returns (entries (n_exec * cap, 2) int32, n_slots int32 [-1 = not listed],
        entry_off int64, warp_edge_events)."""
        for t in (launch_off, thread_off, ev_off):
            _dev(t, self.device, torch.int64)
        _dev(dims, self.device, torch.int32)
        _dev(sites, self.device, torch.int32)
        o = out or {}
        if "entries" not in o:
            o["entries"] = torch.empty((n_exec * cap, 2), dtype=torch.int32, device=self.device)
            o["n_slots"] = torch.empty(n_exec, dtype=torch.int32, device=self.device)
            o["entry_off"] = torch.arange(n_exec + 1, dtype=torch.int64, device=self.device) * cap
            o["events"] = torch.empty(n_exec, dtype=torch.int64, device=self.device) if want_events else None
        n_launch = thread_off.numel() - 1
        self._sync_stream()
        check(lib.hfz_edge_record_batch_lists(self._h, _ptr(launch_off), _ptr(dims), _ptr(thread_off), _ptr(ev_off),
                                              _ptr(sites), n_exec, n_launch, _ptr(raw) if raw is not None else None,
                                              _ptr(o["events"]) if o["events"] is not None else None,
                                              _ptr(o["entries"]), cap, _ptr(o["n_slots"])))
        return o

    def host_edge_record_batch(self, site_off, sites, n_exec, raw=None):
        _dev(site_off, self.device, torch.int64)
        _dev(sites, self.device, torch.int16)
        if raw is None:
            raw = torch.zeros(n_exec * self.rec, dtype=torch.uint8, device=self.device)
        self._sync_stream()
        check(lib.hfz_host_edge_record_batch(self._h, _ptr(site_off), _ptr(sites), n_exec, _ptr(raw)))
        return raw

    # ---- K3 -----------------------------------------------------------------
    def havoc_batch(self, in_bytes, in_off, rng_state, want_draws=True, out=None):
        """Batched havoc_mutant.  in_off / rng_state are int64 device tensors (u64 bit
        patterns); rng_state is advanced in place.  Returns (out_bytes, out_off, out_len, draws):
        slot j's mutant is out_bytes[out_off[j] : out_off[j] + out_len[j]].  `out` = the tuple a
        previous call with the same in_off returned: its buffers are reused (no allocation, no
        host synchronisation to size them)."""
        _dev(in_bytes, self.device, torch.uint8)
        _dev(in_off, self.device, torch.int64)
        _dev(rng_state, self.device, torch.int64)
        n = in_off.numel() - 1
        if out is not None:
            out_bytes, out_off, out_len, draws = out
            self._sync_stream()
            check(lib.hfz_havoc_batch(self._h, _ptr(in_bytes), _ptr(in_off), n, _ptr(rng_state),
                                      _ptr(out_bytes), _ptr(out_off), _ptr(out_len), _ptr(draws)))
            return out
        lens = in_off[1:] - in_off[:-1]
        caps = torch.clamp(lens + 1024, max=MAX_INPUT_BYTES)
        caps = (caps + 15) // 16 * 16  # keep every slot 16-byte aligned
        out_off = torch.zeros(n + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(caps, 0, out=out_off[1:])
        total = int(out_off[-1].item()) if n else 0
        out_bytes = torch.empty(max(total, 16), dtype=torch.uint8, device=self.device)
        out_len = torch.empty(n, dtype=torch.int64, device=self.device)
        draws = torch.empty(n, dtype=torch.int32, device=self.device) if want_draws else None
        self._sync_stream()
        check(lib.hfz_havoc_batch(self._h, _ptr(in_bytes), _ptr(in_off), n, _ptr(rng_state),
                                  _ptr(out_bytes), _ptr(out_off), _ptr(out_len), _ptr(draws)))
        return out_bytes, out_off, out_len, draws

    def havoc_serial_plan(self, in_off, stream_state):
        """Serial-stream mode: `stream_state` (1-element int64 device tensor) is the campaign's single
        Rng; returns the per-slot start states for havoc_batch and advances stream_state past all
        n mutants (Campaign::fuzz_entry, src/engine.cpp:561-562)."""
        n = in_off.numel() - 1
        states = torch.empty(n, dtype=torch.int64, device=self.device)
        self._sync_stream()
        check(lib.hfz_havoc_serial_plan(self._h, _ptr(in_off), n, _ptr(stream_state), _ptr(states)))
        return states

    def splice_batch(self, in_bytes, in_off, a_idx, b_idx, rng_state):
        _dev(in_bytes, self.device, torch.uint8)
        n = a_idx.numel()
        lens = in_off[1:] - in_off[:-1]
        caps = torch.clamp(lens[a_idx.long()] + lens[b_idx.long()], max=MAX_INPUT_BYTES)
        caps = (caps + 15) // 16 * 16
        out_off = torch.zeros(n + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(caps, 0, out=out_off[1:])
        total = int(out_off[-1].item()) if n else 0
        out_bytes = torch.empty(max(total, 16), dtype=torch.uint8, device=self.device)
        out_len = torch.empty(n, dtype=torch.int64, device=self.device)
        self._sync_stream()
        check(lib.hfz_splice_batch(self._h, _ptr(in_bytes), _ptr(in_off), _ptr(a_idx), _ptr(b_idx), n,
                                   _ptr(rng_state), _ptr(out_bytes), _ptr(out_off), _ptr(out_len)))
        return out_bytes, out_off, out_len

    def deterministic_mutants(self, data: bytes):
        """deterministic_mutants of one input, materialised on the device; returns (count, tensor
        of shape (count, len))."""
        L = len(data)
        host = np.frombuffer(data, np.uint8).copy() if L else np.zeros(1, np.uint8)
        cnt = int(lib.hfz_deterministic_count(C.c_void_p(host.ctypes.data), L))
        if cnt == 0 or L == 0:
            return cnt, torch.empty((cnt, L), dtype=torch.uint8, device=self.device)
        dev_in = torch.from_numpy(host).to(self.device)
        out = torch.empty((cnt, L), dtype=torch.uint8, device=self.device)
        self._sync_stream()
        check(lib.hfz_deterministic_batch(self._h, _ptr(dev_in), L, C.c_void_p(host.ctypes.data),
                                          _ptr(out), cnt))
        return cnt, out


class SigSet:
    """Device-resident std::set<uint64_t> stand-in with count()-then-insert() batch semantics."""

    def __init__(self, ctx: Context, capacity: int = 1 << 22):
        self.ctx = ctx
        h = C.c_void_p()
        check(lib.hfz_sigset_create(ctx._h, capacity, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.hfz_sigset_destroy(self._h)
            self._h = None

    __del__ = close

    def __len__(self):
        v = C.c_uint64(0)
        check(lib.hfz_sigset_size(self._h, C.byref(v)))
        return int(v.value)

    def seen_insert(self, sigs: torch.Tensor) -> torch.Tensor:
        seen = torch.empty(sigs.numel(), dtype=torch.uint8, device=sigs.device)
        self.ctx._sync_stream()
        check(lib.hfz_sigset_seen_insert(self.ctx._h, self._h, _ptr(sigs), sigs.numel(), _ptr(seen)))
        return seen


STRATEGIES = {"all-trace": 0, "unique-trace": 1, "simple-trace": 2, "coverage-increase": 3}


def dispatch_batch(ctx: Context, full_set: SigSet, simple_set: SigSet, sig_full, sig_simple, admit,
                   strategy: str = "simple-trace"):
    """engine.cpp:474-478 + should_sanitize for a whole batch: (full_seen, simple_seen, sanitize)."""
    n = admit.numel()
    fs = torch.empty(n, dtype=torch.uint8, device=admit.device)
    ss = torch.empty(n, dtype=torch.uint8, device=admit.device)
    sz = torch.empty(n, dtype=torch.uint8, device=admit.device)
    ctx._sync_stream()
    check(lib.hfz_dispatch_batch(ctx._h, full_set._h, simple_set._h, _ptr(sig_full), _ptr(sig_simple),
                                 _ptr(admit), n, STRATEGIES[strategy], _ptr(fs), _ptr(ss), _ptr(sz)))
    return fs, ss, sz


# ---- scalar Rng helpers (host arithmetic, rng.hpp) ------------------------------------

def rng_jump(state: int, k: int) -> int:
    return int(lib.hfz_rng_jump(state & MASK64, k & MASK64))


def rng_split(state: int, tag: int):
    s = C.c_uint64(state & MASK64)
    child = int(lib.hfz_rng_split(C.byref(s), tag & MASK64))
    return child, int(s.value)


def u64_to_i64(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)


def i64_to_u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)
