"""Synthetic workloads of the shapes BASELINE.json names.

Everything here is counter-based splitmix64 (the reference's Rng,
include/hetfuzz/rng.hpp:15-21: state after k draws = seed + k*gamma), so every
draw is addressable in parallel by numpy.  The recipes are this repo's own --
the reference ships no workload generator -- and are documented in DESIGN.md.

Raw record layout of one exec (see include/hfz.h):
    [H x u8 host counters][H x u32 device counters],  H = S/2.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

HOST_TABLE = np.array([1, 2, 3, 5, 9, 20, 40, 200], np.uint32)          # one value per host rung
DEV_TABLE = np.array([1, 2, 100, 600, 5000, 20000, 70000], np.uint32)   # one value per device rung


def record_bytes(S: int) -> int:
    return (S // 2) * 5


def sm64(seed, k):
    """k-th (0-based) output of splitmix64 seeded with `seed`; vectorised over k/seed."""
    with np.errstate(over="ignore"):
        z = np.asarray(seed, np.uint64) + (np.asarray(k, np.uint64) + np.uint64(1)) * GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def below32(x, n):
    """Map 64-bit draws to [0, n) for n < 2**32 (top-32-bit multiply; generator-only)."""
    return ((np.asarray(x, np.uint64) >> np.uint64(32)) * np.uint64(n)) >> np.uint64(32)


def _split_views(raw, n_exec, S):
    H = S // 2
    rec = raw.reshape(n_exec, record_bytes(S))
    host = rec[:, :H]
    dev = rec[:, H:].view(np.uint32)  # (n_exec, H)
    return host, dev


def maps_iid(n_exec: int, S: int = 65536, density: float = 0.02, seed: int = 42, first: int = 0):
    """Mode (i): per exec ~density*S slots drawn iid over the whole map (duplicates
    collapse, last value wins).  Host value 1+below(40), device count 1+below(100000).
    Every map is a novelty candidate for a long time -- the stress case."""
    H = S // 2
    nnz = max(1, int(round(density * S)))
    raw = np.zeros(n_exec * record_bytes(S), np.uint8)
    host, dev = _split_views(raw, n_exec, S)
    e = (np.arange(n_exec, dtype=np.uint64) + np.uint64(first))[:, None]
    k = np.arange(nnz, dtype=np.uint64)[None, :]
    es = sm64(np.uint64(seed), e)                      # per-exec stream seed
    idx = below32(sm64(es, 2 * k), S).astype(np.int64)
    val = sm64(es, 2 * k + np.uint64(1))
    hv = (np.uint64(1) + below32(val, 40)).astype(np.uint8)
    dv = (np.uint64(1) + below32(val, 100000)).astype(np.uint32)
    rows = np.broadcast_to(np.arange(n_exec)[:, None], idx.shape)
    mh = idx < H
    host[rows[mh], idx[mh]] = hv[mh]
    md = ~mh
    dev[rows[md], idx[md] - H] = dv[md]
    return raw


def maps_campaign(n_exec: int, S: int = 65536, density: float = 0.02, seed: int = 43,
                  first: int = 0, p_extra: int = 256, p_rare: int = 512):
    """Mode (ii), campaign-like: a fixed 'program' E of ~density*S
    slots; each exec hits each slot of E with prob 9/10; the count comes from the
    slot's favourite rung with prob 97/100, else from the single alternate rung
    (fav+1); with prob 1/p_extra one extra random slot is hit once (NewEdges
    source); with prob 1/p_rare one slot of E takes the rare rung (fav+3)
    (NewCounts source).  `first` offsets the exec index so shards of one big batch
    can be generated independently."""
    H = S // 2
    nE = max(1, int(round(density * S)))
    raw = np.zeros(n_exec * record_bytes(S), np.uint8)
    host, dev = _split_views(raw, n_exec, S)
    j = np.arange(nE, dtype=np.uint64)
    prog = np.uint64(seed)
    E = below32(sm64(prog, 2 * j), S).astype(np.int64)              # may contain duplicates
    fav = below32(sm64(prog, 2 * j + np.uint64(1)), 7).astype(np.int64)
    is_host = E < H
    ntab = np.where(is_host, 8, 7)

    e = (np.arange(n_exec, dtype=np.uint64) + np.uint64(first))[:, None]
    es = sm64(prog ^ np.uint64(0xD1B54A32D192ED03), e)
    d = sm64(es, j[None, :])                                         # one draw per (exec, slot)
    hit = below32(d, 10) < 9
    alt = below32(sm64(es ^ np.uint64(0xA17), j[None, :]), 100) >= 97
    rung = np.where(alt, (fav[None, :] + 1) % ntab[None, :], fav[None, :])

    dx = sm64(es[:, 0], np.uint64(nE) + np.arange(4, dtype=np.uint64)[:, None]).T  # (n_exec,4)
    rare_on = below32(dx[:, 0], p_rare) == 0 if p_rare else np.zeros(n_exec, bool)
    rare_j = below32(dx[:, 1], nE).astype(np.int64)
    rr = np.nonzero(rare_on)[0]
    rung[rr, rare_j[rr]] = (fav[rare_j[rr]] + 3) % ntab[rare_j[rr]]
    hit[rr, rare_j[rr]] = True

    rows = np.broadcast_to(np.arange(n_exec)[:, None], hit.shape)
    cols = np.broadcast_to(E[None, :], hit.shape)
    mh = hit & is_host[None, :]
    host[rows[mh], cols[mh]] = HOST_TABLE[rung[mh]].astype(np.uint8)
    md = hit & ~is_host[None, :]
    dev[rows[md], cols[md] - H] = DEV_TABLE[rung[md]]

    extra_on = below32(dx[:, 2], p_extra) == 0 if p_extra else np.zeros(n_exec, bool)
    xs = below32(dx[:, 3], S).astype(np.int64)
    for r in np.nonzero(extra_on)[0]:
        s = xs[r]
        if s < H:
            if host[r, s] == 0:
                host[r, s] = 1
        elif dev[r, s - H] == 0:
            dev[r, s - H] = 1
    return raw


def maps_edge_cases(S: int = 65536):
    """Edge vectors of SURVEY 8d config 1: all-zero map, full-density map, counts
    at every rung boundary +-1, host 255 / wrapped values, device 0xffffffff."""
    H = S // 2
    recs = []

    def new():
        r = np.zeros(record_bytes(S), np.uint8)
        return r, r[:H], r[H:].view(np.uint32)

    r, h, d = new()
    recs.append(r)                                     # all-zero
    r, h, d = new()
    h[:] = (np.arange(H) % 255 + 1).astype(np.uint8)   # full density
    d[:] = (np.arange(H, dtype=np.uint32) * np.uint32(2654435761)) | np.uint32(1)
    recs.append(r)
    r, h, d = new()                                    # every rung boundary +-1
    hb = [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 127, 128, 129, 254, 255]
    db = [1, 2, 3, 4, 511, 512, 513, 4095, 4096, 4097, 16383, 16384, 16385, 65535, 65536,
          65537, 0x7FFFFFFF, 0xFFFFFFFE, 0xFFFFFFFF]
    h[np.arange(len(hb)) * 37 % H] = hb
    d[np.arange(len(db)) * 41 % H] = np.array(db, np.uint32)
    recs.append(r)
    r, h, d = new()                                    # only the last slot of each half
    h[H - 1] = 255
    d[H - 1] = 0xFFFFFFFF
    recs.append(r)
    r, h, d = new()                                    # only the first slot of each half
    h[0] = 1
    d[0] = 1
    recs.append(r)
    r, h, d = new()                                    # one dense 16-byte vector + lone slots
    h[512:528] = np.arange(1, 17, dtype=np.uint8)
    d[100:104] = [1, 2, 3, 70000]
    h[H // 2 + 5] = 3
    recs.append(r)
    return np.concatenate(recs), len(recs)


def to_sparse(raw: np.ndarray, n_exec: int, S: int = 65536, shuffle_seed: int | None = 1):
    """Dense records -> per-exec touched-slot lists for the sparse ingest calls: returns
    (entries (N, 2) uint32 of (slot, count), entry_off (n_exec+1) uint64).  The pairs of an exec
    are put in a seeded random order (touch order is arbitrary); shuffle_seed=None keeps them
    ascending."""
    H = S // 2
    host, dev = _split_views(raw, n_exec, S)
    hr, hc = np.nonzero(host)
    dr, dc = np.nonzero(dev)
    rows = np.concatenate([hr, dr])
    slots = np.concatenate([hc, dc + H]).astype(np.uint32)
    cnts = np.concatenate([host[hr, hc].astype(np.uint32), dev[dr, dc]])
    if shuffle_seed is None:
        order = np.lexsort((slots, rows))
    else:
        key = sm64(np.uint64(shuffle_seed), np.arange(rows.size, dtype=np.uint64))
        order = np.lexsort((key, rows))
    entries = np.empty((rows.size, 2), np.uint32)
    entries[:, 0] = slots[order]
    entries[:, 1] = cnts[order]
    off = np.zeros(n_exec + 1, np.uint64)
    np.cumsum(np.bincount(rows, minlength=n_exec), out=off[1:])
    return entries, off


def to_compact(raw: np.ndarray, n_exec: int, S: int = 65536, shuffle_seed: int | None = 1):
    """Dense records -> the compact list form (S <= 65,536): (compact uint32 words slot | count << 16,
    compact_off, wide (M, 2) uint32 pairs for counts >= 65,536, wide_off)."""
    assert S <= 65536
    entries, off = to_sparse(raw, n_exec, S, shuffle_seed)
    rows = np.repeat(np.arange(n_exec), np.diff(off).astype(np.int64))
    big = entries[:, 1] >= 65536
    compact = (entries[~big, 0] | (entries[~big, 1] << np.uint32(16))).astype(np.uint32)
    wide = np.ascontiguousarray(entries[big])
    coff = np.zeros(n_exec + 1, np.uint64)
    woff = np.zeros(n_exec + 1, np.uint64)
    np.cumsum(np.bincount(rows[~big], minlength=n_exec), out=coff[1:])
    np.cumsum(np.bincount(rows[big], minlength=n_exec), out=woff[1:])
    return np.ascontiguousarray(compact), coff, wide, woff


def to_packed(raw: np.ndarray, n_exec: int, S: int = 65536, shuffle_seed: int | None = 1):
    """Dense records -> the packed list form of hfz_feedback_batch_packed_host (S = 65,536): (host3 uint8 bytes, three
    per host-half slot -- slot lo, slot hi, count -- every exec padded with zero entries to a multiple of four,
    host3_off in entries; dev17 uint32 words (slot - H) | min(count, 65536) << 15, dev17_off)."""
    assert S == 65536
    H = S // 2
    entries, off = to_sparse(raw, n_exec, S, shuffle_seed)
    rows = np.repeat(np.arange(n_exec), np.diff(off).astype(np.int64))
    is_host = entries[:, 0] < H
    nh = np.bincount(rows[is_host], minlength=n_exec).astype(np.int64)
    nh_pad = (nh + 3) // 4 * 4
    hoff = np.zeros(n_exec + 1, np.uint64)
    np.cumsum(nh_pad, out=hoff[1:])
    host3 = np.zeros((int(hoff[-1]), 3), np.uint8)
    hrows = rows[is_host]
    within = np.arange(hrows.size) - np.repeat(np.cumsum(nh) - nh, nh)  # index of each host entry inside its exec
    dst = hoff[:-1].astype(np.int64)[hrows] + within
    hs = entries[is_host]
    host3[dst, 0] = hs[:, 0] & 0xFF
    host3[dst, 1] = hs[:, 0] >> 8
    host3[dst, 2] = hs[:, 1]
    ds = entries[~is_host]
    dev17 = ((ds[:, 0] - np.uint32(H)) | (np.minimum(ds[:, 1], np.uint32(65536)) << np.uint32(15))).astype(np.uint32)
    doff = np.zeros(n_exec + 1, np.uint64)
    np.cumsum(np.bincount(rows[~is_host], minlength=n_exec), out=doff[1:])
    return np.ascontiguousarray(host3.reshape(-1)), hoff, np.ascontiguousarray(dev17), doff


# ---- havoc seeds (config 4) ---------------------------------------------------

def havoc_inputs(n: int, seed: int = 45, lo: int = 1024, hi: int = 4096):
    """n inputs of length lo + below(hi-lo+1), bytes below(256).  Returns (bytes u8, offsets u64[n+1])."""
    i = np.arange(n, dtype=np.uint64)
    lens = (np.uint64(lo) + below32(sm64(np.uint64(seed), i), hi - lo + 1)).astype(np.uint64)
    off = np.zeros(n + 1, np.uint64)
    np.cumsum(lens, out=off[1:])
    total = int(off[-1])
    data = (sm64(np.uint64(seed) ^ np.uint64(0xABCDEF), np.arange((total + 7) // 8, dtype=np.uint64))
            .view(np.uint8)[:total].copy())
    return data, off


# ---- device basic-block traces (config 3) ---------------------------------------

def _bb_paths(S0, keys, ids, succ, n_sites, max_len):
    """Path of every key: (lens int64, steps (len(keys), max_len) int16 site indices)."""
    ks = sm64(S0 ^ np.uint64(0x77), keys)
    lens = (np.uint64(1) + below32(sm64(ks, 0), max_len)).astype(np.int64)
    cur = below32(sm64(ks, 1), n_sites).astype(np.int64)
    steps = np.zeros((keys.size, max_len), np.int16)
    for s in range(max_len):
        steps[:, s] = cur
        cur = succ[cur, below32(sm64(ks, 2 + s), 2).astype(np.int64)]
    return lens, steps


def bb_traces(n_exec: int, seed: int = 44, n_launch: int = 4, grid=(16, 1, 1), block=(256, 1, 1),
              n_sites: int = 512, max_len: int = 24, divergent_den: int = 16, chunk_execs: int = 64):
    """Per exec `n_launch` launches of grid x block threads.  Each thread walks a random
    CFG over `n_sites` site ids (ids = 32-bit truncations of splitmix64 draws): a warp
    shares one path (coherent) unless it is one of the 1/divergent_den fully divergent
    warps, in which case every lane has its own path.  A path of length 1+below(max_len)
    follows succ[site][below(2)] from a start site, so loops revisit sites.
    Returns dict(launch_off, dims, thread_off, ev_off, sites) in hfz_edge_record_batch layout.
    (Paths are a function of a per-warp or per-thread key, so they are computed once per
    coherent warp and expanded to its lanes; execs are generated `chunk_execs` at a time.)"""
    assert n_sites < 32768
    tpb = block[0] * block[1] * block[2]
    blocks = grid[0] * grid[1] * grid[2]
    wpb = (tpb + 31) // 32
    threads = tpb * blocks
    S0 = np.uint64(seed)
    ids = (sm64(S0, np.arange(n_sites, dtype=np.uint64)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    succ = below32(sm64(S0 ^ np.uint64(0x5151), np.arange(2 * n_sites, dtype=np.uint64)),
                   n_sites).astype(np.int64).reshape(n_sites, 2)
    # a few self/short loops so the k-th-visit rule is exercised
    succ[::7, 0] = np.arange(n_sites)[::7]

    n_l = n_exec * n_launch
    tl = np.arange(tpb)
    warp_of_tl = tl // 32
    cols = np.arange(max_len)[None, :]
    site_chunks, len_chunks = [], []
    l_step = max(1, chunk_execs * n_launch)
    for l0 in range(0, n_l, l_step):
        l1 = min(n_l, l0 + l_step)
        L = np.arange(l0, l1, dtype=np.uint64)[:, None, None]
        B = np.arange(blocks, dtype=np.uint64)[None, :, None]
        W = np.arange(wpb, dtype=np.uint64)[None, None, :]
        wkey = ((L * np.uint64(blocks) + B) * np.uint64(wpb) + W).reshape(-1)      # one per simulated warp
        div = below32(sm64(S0 ^ np.uint64(0xD1), wkey), divergent_den) == 0
        wlens, wsteps = _bb_paths(S0, wkey, ids, succ, n_sites, max_len)
        # thread -> row of the path table: its warp's row unless the warp is divergent
        n_w = wkey.size
        warp_of_thread = (np.arange(n_w // wpb)[:, None] * wpb + warp_of_tl[None, :]).reshape(-1)
        row = warp_of_thread.copy()
        tdiv = div[warp_of_thread]
        if tdiv.any():
            T = np.broadcast_to(tl.astype(np.uint64)[None, :], (n_w // wpb, tpb)).reshape(-1)[tdiv]
            tkey = (wkey[warp_of_thread[tdiv]] << np.uint64(10)) ^ T ^ np.uint64(1 << 40)
            tlens, tsteps = _bb_paths(S0, tkey, ids, succ, n_sites, max_len)
            row[tdiv] = n_w + np.arange(tkey.size)
            wlens = np.concatenate([wlens, tlens])
            wsteps = np.concatenate([wsteps, tsteps])
        lens = wlens[row]
        keep = cols < lens[:, None]
        site_chunks.append(ids[wsteps[row][keep]])
        len_chunks.append(lens)
    lens = np.concatenate(len_chunks) if len_chunks else np.zeros(0, np.int64)
    ev_off = np.zeros(lens.size + 1, np.uint64)
    np.cumsum(lens.astype(np.uint64), out=ev_off[1:])
    sites = np.concatenate(site_chunks) if site_chunks else np.zeros(0, np.uint32)
    dims = np.tile(np.array([*grid, *block], np.uint32), (n_l, 1))
    launch_off = (np.arange(n_exec + 1, dtype=np.uint64) * np.uint64(n_launch))
    thread_off = (np.arange(n_l + 1, dtype=np.uint64) * np.uint64(threads))
    return dict(launch_off=launch_off, dims=dims, thread_off=thread_off, ev_off=ev_off,
                sites=sites.astype(np.uint32))
