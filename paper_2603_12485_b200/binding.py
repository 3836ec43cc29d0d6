"""Drop-in for the stateless entry points of the reference's pybind11 module
``hetfuzz._core`` (proj/python/bindings.cpp): same names, argument meaning and
error behaviour, computed on the GPU.

    havoc_mutant(data: bytes, seed: int) -> bytes          bindings.cpp:220-223, :336-337
    splice_mutant(a: bytes, b: bytes, seed: int) -> bytes  bindings.cpp:225-229, :338-339
    deterministic_mutants(data: bytes) -> list[bytes]      bindings.cpp:213-218, :334-335

Each call creates a fresh ``Rng(seed)`` exactly like the reference.  The batched
variants are what a fuzzer should call; the single-item ones are batch-of-one
device calls (latency-bound, kept for API parity).
"""
from __future__ import annotations

import numpy as np
import torch

from . import api

_default = {}


class TargetError(ValueError):
    """bindings.cpp:314 maps hetfuzz::TargetError to ValueError."""


def default_context(device: int = 0, map_slots: int = api.MAP_SIZE) -> api.Context:
    key = (device, map_slots)
    if key not in _default:
        _default[key] = api.Context(device, map_slots)
    return _default[key]


def _check_seed(seed: int) -> int:
    if not isinstance(seed, int) or seed < 0 or seed > api.MASK64:
        raise TypeError("seed must be an unsigned 64-bit integer")  # pybind11 raises TypeError too
    return seed


def havoc_batch(inputs, seeds, device: int = 0):
    """inputs: list[bytes]; seeds: list[int] (slot j uses a fresh Rng(seeds[j])).
    Returns (list[bytes], end_states list[int], draws list[int])."""
    ctx = default_context(device)
    n = len(inputs)
    lens = np.array([len(b) for b in inputs], np.int64)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    blob = np.frombuffer(b"".join(inputs), np.uint8) if off[-1] else np.zeros(0, np.uint8)
    d_in = torch.from_numpy(np.concatenate([blob, np.zeros(16, np.uint8)])).to(ctx.device)
    d_off = torch.from_numpy(off).to(ctx.device)
    d_state = torch.from_numpy(api.u64_to_i64(np.array(seeds, np.uint64))).to(ctx.device)
    out_bytes, out_off, out_len, draws = ctx.havoc_batch(d_in, d_off, d_state)
    ob = out_bytes.cpu().numpy()
    oo = out_off.cpu().numpy()
    ol = out_len.cpu().numpy()
    res = [ob[oo[j]:oo[j] + ol[j]].tobytes() for j in range(n)]
    return res, [int(x) for x in api.i64_to_u64(d_state)], [int(x) for x in draws.cpu().numpy()]


def havoc_mutant(data: bytes, seed: int) -> bytes:
    return havoc_batch([bytes(data)], [_check_seed(seed)])[0][0]


def splice_mutant(a: bytes, b: bytes, seed: int) -> bytes:
    ctx = default_context()
    a, b = bytes(a), bytes(b)
    off = np.array([0, len(a), len(a) + len(b)], np.int64)
    blob = np.frombuffer(a + b + bytes(16), np.uint8)
    d_in = torch.from_numpy(blob.copy()).to(ctx.device)
    d_off = torch.from_numpy(off).to(ctx.device)
    ai = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    bi = torch.ones(1, dtype=torch.int32, device=ctx.device)
    st = torch.from_numpy(api.u64_to_i64(np.array([_check_seed(seed)], np.uint64))).to(ctx.device)
    ob, oo, ol = ctx.splice_batch(d_in, d_off, ai, bi, st)
    n = int(ol[0].item())
    return ob[:n].cpu().numpy().tobytes()


def deterministic_mutants(data: bytes):
    ctx = default_context()
    cnt, out = ctx.deterministic_mutants(bytes(data))
    host = out.cpu().numpy()
    return [host[i].tobytes() for i in range(cnt)]


def feedback_batch(raw: np.ndarray, virgin: np.ndarray, edge_counts: np.ndarray, device: int = 0,
                   want_classed: bool = False, map_slots: int = api.MAP_SIZE):
    """Host-buffer feedback fold (classify_trace + trace_signature x2 + has_new_bits per exec,
    src/engine.cpp:471-478).  Mutates virgin / edge_counts like has_new_bits mutates VirginMap."""
    return default_context(device, map_slots).feedback_batch_host(raw, virgin, edge_counts, want_classed)


def feedback_batch_sparse(entries: np.ndarray, entry_off: np.ndarray, virgin: np.ndarray,
                          edge_counts: np.ndarray, device: int = 0, want_classed: bool = False,
                          map_slots: int = api.MAP_SIZE):
    """The same fold fed with per-exec touched-slot lists: entries (N, 2) uint32 of (slot, count),
    entry_off (n_exec+1) uint64.  ~10 KB per exec over PCIe instead of a 163,840-byte record."""
    return default_context(device, map_slots).feedback_batch_sparse_host(entries, entry_off, virgin,
                                                                         edge_counts, want_classed)


def feedback_batch_compact(compact: np.ndarray, compact_off: np.ndarray, wide, wide_off, virgin: np.ndarray,
                           edge_counts: np.ndarray, device: int = 0, want_classed: bool = False):
    """Touched-slot lists at 4 bytes per pair (65,536-slot maps): compact uint32 words
    slot | count << 16, plus (M, 2) wide pairs for counts >= 65,536 (or None, None)."""
    return default_context(device, api.MAP_SIZE).feedback_batch_compact_host(compact, compact_off, wide, wide_off,
                                                                             virgin, edge_counts, want_classed)


def _as_pairs(m, map_slots):
    """One execution's map in any of the accepted forms -> (entries (N, 2) uint32 of (slot, count))."""
    if isinstance(m, (bytes, bytearray, memoryview)):
        m = np.frombuffer(bytes(m), np.uint8)
    a = np.asarray(m)
    H = map_slots // 2
    if a.dtype == np.uint8 and a.size == api.record_bytes(map_slots):      # dense raw record
        host = a[:H]
        dev = a[H:].view(np.uint32)
        hs = np.nonzero(host)[0]
        ds = np.nonzero(dev)[0]
        out = np.empty((hs.size + ds.size, 2), np.uint32)
        out[:hs.size, 0] = hs
        out[:hs.size, 1] = host[hs]
        out[hs.size:, 0] = ds + H
        out[hs.size:, 1] = dev[ds]
        return out
    a = np.ascontiguousarray(a, dtype=np.uint32)
    if a.ndim == 2 and a.shape[1] == 2:                                  # (slot, count) pairs, any order
        return a
    raise TypeError("a map is a dense raw record (bytes / uint8 array of map_slots/2*5 bytes) or an (N, 2) array "
                    "of (slot, count) pairs")


def replay_signatures(maps, device: int = 0, map_slots: int = api.MAP_SIZE):
    """The hot-path part of the reference's ``replay_sequence`` (bindings.cpp:268-286, which returns
    ``full_sigs`` / ``simple_sigs`` of the executed inputs): the same two lists for maps the caller
    already holds -- the simulator that produces them is out of scope here.  Each map is a dense raw
    record or an (N, 2) array of (slot, count) pairs.  Also returns ``nonzero_slots`` per map."""
    pairs = [_as_pairs(m, map_slots) for m in maps]
    off = np.zeros(len(pairs) + 1, np.uint64)
    np.cumsum([p.shape[0] for p in pairs], out=off[1:])
    ent = np.concatenate(pairs) if pairs else np.zeros((0, 2), np.uint32)
    if ent.shape[0] == 0:
        ent = np.zeros((1, 2), np.uint32)
    o = default_context(device, map_slots).feedback_batch_sparse_host(
        np.ascontiguousarray(ent), off, np.zeros(map_slots, np.uint8), np.zeros(2, np.uint64))
    return {"full_sigs": [int(x) for x in o["sig_full"]], "simple_sigs": [int(x) for x in o["sig_simple"]],
            "nonzero_slots": [int(x) for x in o["nnz"]]}


def signatures(m, device: int = 0, map_slots: int = api.MAP_SIZE):
    """The hot-path outputs of the reference's ``run_input`` (bindings.cpp:199-202) for a map the caller
    already holds: ``{"nonzero_slots", "full_sig", "simple_sig"}`` -- classify_trace + both trace_signature
    calls on the GPU."""
    r = replay_signatures([m], device, map_slots)
    return {"nonzero_slots": r["nonzero_slots"][0], "full_sig": r["full_sigs"][0], "simple_sig": r["simple_sigs"][0]}
