// hfz_edge.cu -- K1 edge record: batched device basic-block traces -> warp-granular saturating
// edge counters in the device half of each raw map; plus the host-edge record stage.
//
// Reference semantics (paths under /root/reference/proj):
//   DeviceThreadCtx::Impl::edge   src/hdvm.cpp:415-431   (first-lane-to-reach-visit-k rule)
//   Runtime::bump_counter         src/hdvm.cpp:362-366   (saturating u32)
//   thread / warp enumeration     src/hdvm.cpp:556-603   (gtid flattening :597-600, warp_global :602)
//   device_edge_index             include/hetfuzz/coverage.hpp:88-91
//   merge_device_into_map         src/coverage.cpp:99-105
//   host_edge_update/host_increment  include/hetfuzz/coverage.hpp:24-32,79-84
//
// The reference runs the simulated threads one after another; event (lane L, site s, k-th
// visit of s by L in this launch) bumps a counter iff k > max_{L' < L, same warp} count_{L'}(s),
// at slot (prev_L ^ s) % H with lane L's own running prev (= previous site >> 1, carried
// across launches per flattened gtid).  That rule is separable per site, so here:
//   * one CTA owns one execution; its counters live in SHARED memory (warp bumps are
//     shared-memory atomics, flushed to HBM once per exec -- no global atomic per hit): a dense
//     table of packed 16-bit counters for up to 32,768 device slots, a hashed dirty-slot table
//     (slot -> u32 count, the reference's own dirty list of src/hdvm.cpp:356-366 as an open-
//     addressing table) for larger maps such as the 131,072 device slots of a 262,144-slot map;
//   * a real warp replays one simulated warp, real lane L <-> simulated lane L:
//       fast path   all active lanes walk the same site sequence (the SIMT common case):
//                   only the lowest lane can ever bump, every event of it does;
//       general     the simulated lanes are replayed in order (that is the rule), but each
//                   lane's events are spread over the 32 real lanes (coalesced loads):
//                   __match_any gives the visit number within the chunk, a per-warp
//                   shared-memory table site -> (max count of lower lanes, count of the current
//                   lane) gives M_L(s); visits with k > M_L(s) bump in parallel.  If a warp has
//                   more distinct sites than the table holds, the site space is partitioned by
//                   hash prefix (the rule is separable per site) and the replay repeats per
//                   partition, splitting on overflow.
#include <stdio.h>
#include <string.h>

#include "hfz_common.cuh"

// Dev diagnostic (make EXTRA=-DHFZ_EDGE_PROF): cycles per phase, summed over the lane 0s of the table-owning
// (row 0) and the other (row 1) warps; read back with hfz_dbg_edge_prof (scripts/probe_k1k3.py edge).
#ifdef HFZ_EDGE_PROF
__device__ unsigned long long g_edge_prof[2][16];
#define PROF_DECL long long _pt = clock64()
#define PROF(prof, cat)                                                                \
  do {                                                                                 \
    const long long _pn = clock64();                                                   \
    if (lane == 0 && (prof)) atomicAdd((prof) + (cat), (unsigned long long)(_pn - _pt)); \
    _pt = _pn;                                                                         \
  } while (0)
#else
#define PROF_DECL
#define PROF(prof, cat)
#endif

namespace {

constexpr int kEdgeWarps = 32;
constexpr uint32_t kRows = 256;        // site table rows
// One table serves either general-path variant:
//   transposed replay: keys u64[kRows] + per-row byte matrix [kRows][32]  (2 KB + 8 KB)
//   partitioned replay (fallback): keys u64, m u32, c u32, stamp u32       (5 KB)
// Only non-coherent simulated warps need one, and 24 tables do not fit beside the counters: the
// first kPool warps of the CTA each OWN a table for the whole kernel; the other warps hand a
// non-coherent simulated warp they popped over to the owners through a small queue in shared memory
// (atomics only).  No table ever changes hands, so there is no lock for compute-sanitizer's
// racecheck to misread (the pool of borrowed tables this replaces was a spin lock on a free-mask).
constexpr uint32_t kTabBytes = kRows * (8 + 32) + 64;
constexpr int kPool = 16;
constexpr uint32_t kDeferCap = 64;  // queue slots (simulated warp index + 1; 0 = empty)
constexpr uint32_t kSmemSlots = 32768; // device slots whose counters fit in shared memory
constexpr uint32_t kMaxBlockThreads = 1024;         // hdvm.hpp:167
constexpr uint64_t kMaxLaunchThreads = 1ull << 22;  // hdvm.hpp:168

struct EdgeParams {
  const uint64_t* launch_off;
  const uint32_t* dims;
  const uint64_t* thread_off;
  const uint64_t* ev_off;
  const uint32_t* sites;
  uint64_t n_exec;
  uint32_t H;
  uint64_t rec_bytes;
  uint8_t* raw;
  uint64_t* warp_events;
  uint32_t* prev_scratch;    // [gridDim.x][prev_stride]
  uint64_t prev_stride;
  const uint32_t* exec_list; // NULL: execs 0 .. n_exec - 1; else the n_exec execs listed (any order)
};

// bijective 32-bit mixer: distinct sites have distinct hashes, so a partition of depth 32 holds one site
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ bool launch_valid(const uint32_t* d) {
  if (!d[0] || !d[1] || !d[2] || !d[3] || !d[4] || !d[5]) return false;
  const uint64_t tpb = (uint64_t)d[3] * d[4] * d[5];
  if (tpb > kMaxBlockThreads) return false;
  const uint64_t blocks = (uint64_t)d[0] * d[1] * d[2];
  return blocks * tpb <= kMaxLaunchThreads;  // blocks <= 2^22 here, no overflow
}

// saturating bump (hdvm.cpp:362-366).  A wrapped add is repaired by the thread that wrapped it;
// once a counter has wrapped its final value is always 0xffffffff.
__device__ __forceinline__ void bump(uint32_t* c) {
  if (atomicAdd(c, 1u) == 0xffffffffu) atomicExch(c, 0xffffffffu);
}

// Where an exec's counters live while it is replayed.
//   packed  shared memory, TWO 16-bit counters per 32-bit word (64 KB for 32,768 slots instead of
//           128 KB: room for more warps and tables).  A counter that comes near 16 bits raises
//           *overflow; the exec is then replayed once more with wide counters.
//   hashed  shared memory, open-addressing table slot -> saturating u32 count (kHashCap rows,
//           64 KB) for maps whose device half does not fit shared memory even packed: an exec
//           touches a few thousand distinct slots (~2 % of the map), so the table holds the
//           dirty slots only and the flush is zero-fill + scatter.  More than kHashLimit
//           distinct slots raise *overflow; the exec is then replayed with wide counters.
//   wide    saturating u32 counters in the exec's output record (global atomics): the replay
//           after an overflow, nothing else.
// kNear leaves more headroom than the CTA has threads, so no concurrent burst of bumps can
// carry into the neighbouring counter before one of them has seen the flag condition.
constexpr uint32_t kNear = 0xf000;
constexpr uint32_t kHashBits = 13, kHashCap = 1u << kHashBits;  // 8,192 rows x (u32 key + u32 count) = 64 KB
constexpr uint32_t kHashLimit = kHashCap * 3 / 4;               // distinct slots before the exec is replayed wide
constexpr uint32_t kHashEmpty = 0xffffffffu;                     // slot ids are < 2^23
enum { kCntWide = 0, kCntPacked = 1, kCntHashed = 2 };
struct Counters {
  uint32_t* base;      // packed: H/2 words; hashed: keys[kHashCap] then counts[kHashCap]; wide: the record's device half
  int mode;
  uint32_t* overflow;
  uint32_t* used;      // hashed: rows taken
  __device__ __forceinline__ void bump_slot(uint32_t slot) const {
    if (mode == kCntPacked) {
      const uint32_t sh = (slot & 1u) * 16u;
      const uint32_t old = atomicAdd(base + (slot >> 1), 1u << sh);
      if (((old >> sh) & 0xffffu) >= kNear) *overflow = 1u;
    } else if (mode == kCntHashed) {
      if (*reinterpret_cast<volatile uint32_t*>(overflow)) return;  // the exec is replayed anyway; keeps the table from filling up
      volatile uint32_t* keys = base;
      uint32_t r = (slot * 0x9e3779b1u) >> (32 - kHashBits);
      for (;;) {
        const uint32_t cur = keys[r];
        if (cur == slot) break;
        if (cur == kHashEmpty) {
          const uint32_t old = atomicCAS(base + r, kHashEmpty, slot);
          if (old == kHashEmpty) {
            if (atomicAdd(used, 1u) >= kHashLimit) *overflow = 1u;
            break;
          }
          if (old == slot) break;
        }
        r = (r + 1) & (kHashCap - 1);
      }
      bump(base + kHashCap + r);
    } else {
      bump(base + slot);
    }
  }
};

// Where the replay paths put a bump.  emit() is called by all 32 lanes together (f = this lane bumps).
//   CounterSink  the per-exec kernel: straight into the exec's counters (n = this lane's bumps)
//   ListSink     the flat kernel: appended to the simulated warp's bump list in global scratch, one
//                ballot per call instead of an atomic per bump (n = bumps of the warp so far, warp-uniform)
struct CounterSink {
  Counters c;
  uint32_t n;
  __device__ __forceinline__ void emit(bool f, uint32_t slot, int) {
    if (f) {
      c.bump_slot(slot);
      ++n;
    }
  }
};
struct ListSink {
  uint32_t* out;
  uint32_t n;
  __device__ __forceinline__ void emit(bool f, uint32_t slot, int lane) {
    const uint32_t m = __ballot_sync(0xffffffffu, f);
    if (f) out[n + __popc(m & ((1u << lane) - 1u))] = slot;
    n += __popc(m);
  }
};

struct WarpTable {
  unsigned long long* keys;  // [kRows]  0 = empty, else (1<<32 | site)
  uint32_t* m;               // [kRows]  max visit count of this site among LOWER simulated lanes
  uint32_t* c;               // [kRows]  visits by the simulated lane `stamp` so far
  uint32_t* stamp;           // [kRows]  simulated lane that owns c (lazy merge into m)
  uint32_t* used;            // [1]
};

// find-or-insert; returns the row or kRows when the table is full
__device__ __forceinline__ uint32_t table_insert(WarpTable& t, uint32_t site, uint32_t h) {
  const unsigned long long want = (1ull << 32) | site;
  uint32_t r = h & (kRows - 1);
  for (uint32_t probe = 0; probe < kRows; ++probe) {
    const unsigned long long cur = t.keys[r];
    if (cur == want) return r;
    if (cur == 0) {
      const unsigned long long old = atomicCAS(&t.keys[r], 0ull, want);
      if (old == 0) {
        atomicAdd(t.used, 1u);
        return r;
      }
      if (old == want) return r;
    }
    r = (r + 1) & (kRows - 1);
  }
  return kRows;
}

// General path for one simulated warp.  e0/n_ev/prev0 are per real lane = per simulated lane.
// Bumps go to the sink.
template <class Sink>
__device__ __forceinline__ void general_path(WarpTable& tab, const uint32_t* sites, uint64_t e0,
                                             uint32_t n_ev, uint32_t prev0, Sink& sink,
                                             uint32_t hmask, int lane) {
  const uint32_t lane_le = 0xffffffffu >> (31 - lane);
  const uint32_t ev_total = __reduce_add_sync(0xffffffffu, n_ev);
  // initial depth: the expected events per partition fit the table even if all were distinct
  // sites (a replay costs the same however few of its events belong to the partition, so start
  // as shallow as possible; a partition that does overflow is found by the dry run and split)
  uint32_t d0 = 0;
  while (d0 < 26 && (ev_total >> d0) > kRows - 32) ++d0;
  uint32_t stk_prefix[36], stk_depth[36];
  for (uint32_t root = 0; root < (1u << d0); ++root) {
    int sp = 1;
    stk_prefix[0] = root;
    stk_depth[0] = d0;
    while (sp > 0) {
      --sp;
      const uint32_t prefix = stk_prefix[sp], depth = stk_depth[sp];
      // events of this partition (an upper bound of its distinct sites): no table can overflow
      // when they fit, otherwise a dry run inserts the sites to find out
      uint32_t mine_cnt = n_ev;
      if (depth) {
        mine_cnt = 0;
        for (uint32_t i = 0; i < n_ev; ++i) mine_cnt += (mix32(sites[e0 + i]) >> (32 - depth)) == prefix;
      }
      const uint32_t part_events = __reduce_add_sync(0xffffffffu, mine_cnt);
      if (part_events == 0) continue;
      for (uint32_t i = lane; i < kRows; i += 32) {
        tab.keys[i] = 0;
        tab.stamp[i] = 0xffffffffu;  // row never touched in this partition: m = c = 0
      }
      if (lane == 0) *tab.used = 0;
      __syncwarp();
      if (part_events > kRows - 16) {
        bool full = false;
        for (uint32_t i = 0; i < n_ev && !full; ++i) {
          const uint32_t s = sites[e0 + i];
          const uint32_t h = mix32(s);
          if (depth && (h >> (32 - depth)) != prefix) continue;
          full = table_insert(tab, s, h) == kRows;
        }
        __syncwarp();
        if (__any_sync(0xffffffffu, full) || (*tab.used > kRows - 16 && depth < 32)) {
          stk_prefix[sp] = prefix * 2 + 1;
          stk_depth[sp] = depth + 1;
          stk_prefix[sp + 1] = prefix * 2;
          stk_depth[sp + 1] = depth + 1;
          sp += 2;
          continue;
        }
      }
      // replay the simulated lanes in order; lane L's events are spread over the real lanes
      for (int L = 0; L < 32; ++L) {
        const uint32_t nL = __shfl_sync(0xffffffffu, n_ev, L);
        if (nL == 0) continue;
        const uint64_t eL = __shfl_sync(0xffffffffu, e0, L);
        uint32_t carry = __shfl_sync(0xffffffffu, prev0, L);  // prev of the chunk's first event
        for (uint32_t c0 = 0; c0 < nL; c0 += 32) {
          const bool act = c0 + lane < nL;
          const uint32_t s = act ? sites[eL + c0 + lane] : 0u;
          const uint32_t h = mix32(s);
          const bool mine = act && (!depth || (h >> (32 - depth)) == prefix);
          uint32_t up = __shfl_up_sync(0xffffffffu, s, 1);
          const uint32_t pv = lane ? (up >> 1) : carry;
          carry = __shfl_sync(0xffffffffu, s, 31) >> 1;  // only used when the chunk is full
          const unsigned long long key = mine ? ((1ull << 32) | s) : (unsigned long long)lane;
          const uint32_t grp = __match_any_sync(0xffffffffu, key);
          uint32_t row = 0, mm = 0, cc = 0;
          bool bf = false;
          if (mine) {
            row = table_insert(tab, s, h);  // cannot fail: checked by the dry run / event bound
            const uint32_t owner = tab.stamp[row];
            if (owner == (uint32_t)L) {
              mm = tab.m[row];
              cc = tab.c[row];
            } else if (owner != 0xffffffffu) {  // counts of an earlier lane: fold into the max
              mm = max(tab.m[row], tab.c[row]);
            }
            bf = cc + __popc(grp & lane_le) > mm;
          }
          sink.emit(bf, (pv ^ s) & hmask, lane);
          __syncwarp();
          if (mine && (grp & (0u - grp)) == (1u << lane)) {  // one writer per site
            tab.m[row] = mm;
            tab.c[row] = cc + __popc(grp);
            tab.stamp[row] = (uint32_t)L;
          }
          __syncwarp();
        }
      }
    }
  }
}

// Transposed general path for one simulated warp.
//   phase 1  the warp's events (contiguous in the trace: lane 0's, then lane 1's, ...) are dealt out
//            32 at a time, one per REAL lane -- coalesced loads, and a warp whose lanes walked paths
//            of different lengths still keeps every real lane busy.  The simulated lane L of an event
//            is found by a 5-step shuffle search over the lanes' end offsets; the event is counted in
//            a nibble matrix cnt[row(site)][L] (shared-memory atomics on the word that holds the nibble);
//   row pass c_L(s) -> d_L(s) = max(0, c_L(s) - max_{L' < L} c_{L'}(s)): the number of bumps lane L
//            owes for site s (its visits k = M_L(s)+1 .. c_L(s)); exclusive prefix max over the 32
//            lanes of a row with SIMD byte ops, saturating byte subtract;
//   phase 2  the events are dealt out again, from the END of the warp's range backwards, and the
//            d_L(s) bumps go to the last d_L(s) visits of s by L -- exactly the visits with
//            k > M_L(s): inside a round __match_any groups the visits of one (L, s), the j-th from the
//            end bumps iff j < d, and the group's first lane takes min(d, size) off the nibble before
//            the next (earlier) round reads it.  The slot uses that visit's own prev.  Bumps commute
//            (saturating adds), so their order is free.
// Table: 128 buckets x 4 site keys, then (kTRows + 1) rows of 16 bytes of nibbles; byte b of a row
// holds lane b (low nibble) and lane b + 16 (high nibble).  A lookup reads a whole bucket with one
// 128-bit load (1.2 probes on average at the ~55 % load of a fully divergent warp; linear probing
// over single keys needed ~8 warp-level steps until the slowest lane had found its row).
// Returns false (nothing bumped) when the table fills up, a lane visits a site more than 15 times
// or the warp has 2^31 events or more: the caller then runs the partitioned replay, which has none
// of these limits.
constexpr uint32_t kTRows = 512;
constexpr uint32_t kTBuckets = kTRows / 4;
constexpr uint32_t kTEmpty = 0xffffffffu;  // key of a free row; the site 0xffffffff gets row kTRows
static_assert((kTRows + 1) * (4 + 16) <= kTabBytes, "transposed table must fit a pool table");

template <class Sink>
__device__ __forceinline__ bool transposed_path(uint8_t* tab, const uint32_t* sites, uint64_t e0, uint32_t n_ev,
                                                bool active, uint32_t prev0, Sink& sink, uint32_t hmask,
                                                int lane, unsigned long long* prof = nullptr) {
  PROF_DECL;
  uint32_t* keys = reinterpret_cast<uint32_t*>(tab);                    // [kTRows + 1], buckets of 4
  uint32_t* cnt = reinterpret_cast<uint32_t*>(tab + (kTRows + 4) * 4);  // [kTRows + 1][4], 16-byte aligned
  for (uint32_t i = lane; i < kTRows + 1; i += 32) keys[i] = kTEmpty;
  uint4* clr = reinterpret_cast<uint4*>(cnt);
  for (uint32_t i = lane; i < kTRows + 1; i += 32) clr[i] = make_uint4(0, 0, 0, 0);
  // the warp's event range [first, first + N); rel_end = end of this lane's events inside it
  // (non-decreasing over the lanes: the inactive lanes of a partial warp are its last ones)
  const uint64_t first = __shfl_sync(0xffffffffu, e0, 0);
  const uint64_t my_end = active ? e0 + n_ev - first : 0;
  uint64_t n64 = my_end;
  for (int d = 16; d; d >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, n64, d);
    n64 = o > n64 ? o : n64;
  }
  __syncwarp();
  if (n64 >= (1ull << 31)) return false;
  const uint32_t N = (uint32_t)n64;
  const uint32_t rel_end = active ? (uint32_t)my_end : N;
  const uint32_t* ev = sites + first;
  PROF(prof, 5);
  auto sim_lane = [&](uint32_t g) -> uint32_t {  // lanes whose events end at or before g
    uint32_t L = 0;
#pragma unroll
    for (uint32_t step = 16; step; step >>= 1) {
      const uint32_t pe = __shfl_sync(0xffffffffu, rel_end, (int)(L + step - 1));
      L += pe <= g ? step : 0u;
    }
    return L & 31u;  // (a lane past the range computes 32: it is off anyway)
  };
  auto cell_word = [](uint32_t L) { return (L & 15u) >> 2; };
  auto cell_shift = [](uint32_t L) { return (L & 3u) * 8u + (L >> 4) * 4u; };
  // find (insert = false) or find-or-insert, called by the WHOLE warp (on = this lane has a site to
  // look up): the probe loop is warp-synchronous -- it runs until no lane is pending, so the lanes
  // leave it together (a per-lane loop with early returns left the warp split for everything after it).
  // Returns the row, kTRows for the site 0xffffffff, kTRows + 1 when the table is full / the key absent.
  const uint4* keys4 = reinterpret_cast<const uint4*>(keys);
  auto find = [&](uint32_t s, bool on, bool insert) -> uint32_t {
    uint32_t b = (s * 0x9e3779b1u) >> (32 - 7);  // multiplicative hash: the top 7 bits pick one of 128 buckets
    static_assert(kTBuckets == 128, "hash shift assumes 128 buckets");
    uint32_t res = kTRows + 1, probes = 0;
    bool pending = on;
    if (on && s == kTEmpty) {
      res = kTRows;
      pending = false;
    }
    while (__any_sync(0xffffffffu, pending)) {
      if (pending) {
        uint4 k;  // (volatile: other lanes insert between two looks at a bucket)
        asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(k.x), "=r"(k.y), "=r"(k.z), "=r"(k.w)
                     : "r"(hfz_smem_u32(keys4 + b)));
        int j = k.x == s ? 0 : (k.y == s ? 1 : (k.z == s ? 2 : (k.w == s ? 3 : -1)));
        bool advance = false;
        if (j < 0) {
          if (insert) {
            const int f = k.x == kTEmpty ? 0 : (k.y == kTEmpty ? 1 : (k.z == kTEmpty ? 2 : (k.w == kTEmpty ? 3 : -1)));
            if (f < 0) {
              advance = true;  // bucket full of other keys
            } else {
              const uint32_t old = atomicCAS(&keys[b * 4 + f], kTEmpty, s);
              if (old == kTEmpty || old == s) j = f;  // else: another key took the slot -- read the bucket again
            }
          } else {
            advance = true;  // lookups are for keys phase 1 inserted: the key sits in a later bucket
          }
        }
        if (j >= 0) {
          res = b * 4 + (uint32_t)j;
          pending = false;
        } else if (advance) {
          b = (b + 1) & (kTBuckets - 1);
          pending = ++probes < kTBuckets;
        }
      }
    }
    return res;
  };
  bool bad = false;
  for (uint32_t g0 = 0; g0 < N; g0 += 32) {
    const uint32_t g = g0 + lane;
    const bool on = g < N && !bad;
    const uint32_t s = g < N ? ev[g] : 0u;
    const uint32_t L = sim_lane(g);
    const uint32_t r = find(s, on, true);
    if (on) {
      if (r > kTRows) {
        bad = true;
      } else {
        const uint32_t sh = cell_shift(L);
        const uint32_t old = atomicAdd(&cnt[r * 4 + cell_word(L)], 1u << sh);
        bad = ((old >> sh) & 15u) == 15u;  // nibble overflow: the table is abandoned
      }
    }
    __syncwarp();
  }
  const bool any_bad = __any_sync(0xffffffffu, bad);
  __syncwarp();  // table reads above are ordered before whatever reuses the table next
  PROF(prof, 6);
  if (any_bad) return false;
  // rows -> owed bumps.  Lane order inside a row: low nibbles of words 0..3 (lanes 0..15), then the
  // high nibbles (lanes 16..31).  Each real lane takes every 32nd row.  Nearly every visited row of a
  // divergent warp is one of two cheap kinds -- ONE visiting lane (d = c: nothing to do), or all
  // visiting lanes with the SAME count c (only the lowest of them owes bumps, c of them) -- and is
  // rewritten in place by its lane.  Rows whose visitors differ in their counts are rare; taking
  // them on inside the per-lane loop made every lane of the warp step through the 240-instruction
  // prefix-max each time one lane needed it (a quarter of the kernel's instructions), so they
  // are flagged by ballot and done by the WHOLE warp: lane L holds c_L, five shuffle steps give the
  // exclusive prefix max, and the new nibbles are gathered with four warp-wide ORs.
  auto nzn = [](uint32_t v) { return (v | (v >> 1) | (v >> 2) | (v >> 3)) & 0x11111111u; };
  const uint32_t my_word = cell_word((uint32_t)lane), my_shift = cell_shift((uint32_t)lane);
  for (uint32_t r0 = 0; r0 < kTRows + 1; r0 += 32) {
    const uint32_t r = r0 + lane;
    bool general = false;
    if (r < kTRows + 1) {
      const uint4 x = reinterpret_cast<uint4*>(cnt)[r];
      const uint32_t any = x.x | x.y | x.z | x.w;
      const uint32_t n0 = nzn(x.x), n1 = nzn(x.y), n2 = nzn(x.z), n3 = nzn(x.w);
      if (any != 0u && __popc(n0) + __popc(n1) + __popc(n2) + __popc(n3) > 1) {
        // the lowest visiting lane's nibble: low nibbles of words 0..3 first, then the high ones
        const uint32_t l0 = n0 & 0x01010101u, l1 = n1 & 0x01010101u, l2 = n2 & 0x01010101u, l3 = n3 & 0x01010101u;
        const bool low = (l0 | l1 | l2 | l3) != 0u;
        const uint32_t c0 = low ? l0 : n0, c1 = low ? l1 : n1, c2 = low ? l2 : n2, c3 = low ? l3 : n3;  // candidates (flag bits)
        const int wsel = c0 ? 0 : (c1 ? 1 : (c2 ? 2 : 3));
        const uint32_t cw = wsel == 0 ? c0 : (wsel == 1 ? c1 : (wsel == 2 ? c2 : c3));
        const uint32_t xw = wsel == 0 ? x.x : (wsel == 1 ? x.y : (wsel == 2 ? x.z : x.w));
        const uint32_t pos = (uint32_t)__ffs(cw) - 1u;  // bit 0 of the lowest visiting lane's nibble
        const uint32_t c = (xw >> pos) & 15u;           // its count
        // same count everywhere?  every visited nibble equals c <=> x == flags * c
        if (x.x == n0 * c && x.y == n1 * c && x.z == n2 * c && x.w == n3 * c) {
          uint4 d4 = make_uint4(0, 0, 0, 0);
          const uint32_t keep = c << pos;
          d4.x = wsel == 0 ? keep : 0u;
          d4.y = wsel == 1 ? keep : 0u;
          d4.z = wsel == 2 ? keep : 0u;
          d4.w = wsel == 3 ? keep : 0u;
          reinterpret_cast<uint4*>(cnt)[r] = d4;
        } else {
          general = true;
        }
      }
    }
    uint32_t todo = __ballot_sync(0xffffffffu, general);
    while (todo) {  // warp-uniform
      const uint32_t rr = r0 + (uint32_t)__ffs(todo) - 1;
      todo &= todo - 1;
      uint32_t* row = &cnt[rr * 4];
      const uint32_t c = (row[my_word] >> my_shift) & 15u;  // c_L of this lane
      uint32_t pm = c;  // inclusive prefix max over the lanes
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, pm, dd);
        if (lane >= dd) pm = max(pm, o);
      }
      uint32_t ex = __shfl_up_sync(0xffffffffu, pm, 1);
      if (lane == 0) ex = 0;
      const uint32_t dv = c > ex ? c - ex : 0u;
      const uint32_t mine = dv << my_shift;
      __syncwarp();  // every lane has read its nibble
      const uint32_t w0 = __reduce_or_sync(0xffffffffu, my_word == 0 ? mine : 0u);
      const uint32_t w1 = __reduce_or_sync(0xffffffffu, my_word == 1 ? mine : 0u);
      const uint32_t w2 = __reduce_or_sync(0xffffffffu, my_word == 2 ? mine : 0u);
      const uint32_t w3 = __reduce_or_sync(0xffffffffu, my_word == 3 ? mine : 0u);
      if (lane == 0) *reinterpret_cast<uint4*>(row) = make_uint4(w0, w1, w2, w3);
    }
  }
  __syncwarp();
  PROF(prof, 7);
  const uint32_t lanes_above = lane == 31 ? 0u : (0xffffffffu << (lane + 1));
  for (uint32_t hi = N; hi > 0; hi = hi > 32 ? hi - 32 : 0) {
    const int32_t g = (int32_t)hi - 32 + lane;  // higher lane = later event
    const bool on = g >= 0;
    const uint32_t s = on ? ev[g] : 0u;
    const uint32_t L = sim_lane(on ? (uint32_t)g : 0u);
    const uint32_t r = find(s, on, false);  // present since phase 1
#ifdef HFZ_EDGE_DEBUG
    if (on && r > kTRows) printf("phase 2: site %08x not found (blk %d)\n", s, blockIdx.x);
#endif
    const uint32_t end_below = __shfl_sync(0xffffffffu, rel_end, (int)((L - 1) & 31u));  // (every lane shuffles)
    const uint32_t lane_start = L ? end_below : 0u;
    const uint32_t lane_prev0 = __shfl_sync(0xffffffffu, prev0, (int)L);
    const unsigned long long key = on ? (((unsigned long long)L << 32) | s) : (0xffffffff00000000ull | (uint32_t)lane);
    const uint32_t grp = __match_any_sync(0xffffffffu, key);
    uint32_t* c = &cnt[(on ? r : kTRows) * 4 + cell_word(L)];
    const uint32_t sh = cell_shift(L);
    const uint32_t d = on ? ((*reinterpret_cast<volatile uint32_t*>(c) >> sh) & 15u) : 0u;
    __syncwarp();  // every nibble of this round is read before any is lowered
    bool bf = false;
    uint32_t bslot = 0;
    if (on && d) {
      if ((uint32_t)__popc(grp & lanes_above) < d) {  // one of the last d visits of s by L still open
        const uint32_t pv = (uint32_t)g > lane_start ? (ev[g - 1] >> 1) : lane_prev0;
        bslot = (pv ^ s) & hmask;
        bf = true;
      }
      if ((grp & (0u - grp)) == (1u << lane)) {  // the group's first lane lowers the nibble for the earlier rounds
        const uint32_t m = (uint32_t)__popc(grp);
        atomicSub(c, (m < d ? m : d) << sh);
      }
    }
    sink.emit(bf, bslot, lane);
    __syncwarp();
  }
  __syncwarp();
  PROF(prof, 8);
  return true;
}


// Divergent warps with SHORT paths (every lane at most kShortPath events -- the usual basic-block
// trace of one kernel launch): real lane L keeps simulated lane L's events in registers.
// Visit (L, s, k) bumps iff no lower lane reaches a k-th visit of s, i.e. iff L is the LOWEST lane
// holding the pair (s, k) -- a first-occurrence test:
//   pass 1  step i of every lane at once: k = 1 + earlier events of the lane at the same site
//           (register compares), then find-or-insert (s, k) in an open-addressing table of 1,024
//           64-bit entries {site, k << 8 | lowest lane} (claimed by one 64-bit CAS, lane by atomicMin);
//   pass 2  the visit bumps iff the entry's lane is its own; slot from its own prev (the event before).
// One table operation per event, no per-site count matrix, no row pass, no second lookup (the row
// found in pass 1 is kept, 10 bits per event).  Returns false without bumping when a lane has more
// than kShortPath events: the caller then takes the transposed replay, which has no such limit.
constexpr int kShortPath = 24;
constexpr uint32_t kShortRows = 1024;  // >= 32 x kShortPath distinct (s, k) pairs at 75 % load
static_assert(kShortRows * 8 <= kTabBytes, "short-path table must fit a site table");

template <class Sink>
__device__ __forceinline__ bool short_divergent_path(uint8_t* tab, const uint32_t* sites, uint64_t e0, uint32_t n_ev,
                                                     uint32_t prev0, Sink& sink, uint32_t hmask, int lane) {
  const uint32_t n_max = __reduce_max_sync(0xffffffffu, n_ev);
  if (n_max > (uint32_t)kShortPath) return false;
  unsigned long long* ent = reinterpret_cast<unsigned long long*>(tab);
  constexpr unsigned long long kFree = ~0ull;
  {
    uint4* clr = reinterpret_cast<uint4*>(tab);
#pragma unroll
    for (uint32_t i = 0; i < kShortRows * 8 / 16 / 32; ++i) clr[i * 32 + lane] = make_uint4(~0u, ~0u, ~0u, ~0u);
  }
  uint32_t ev[kShortPath];
  const uint32_t* mine = sites + e0;
#pragma unroll
  for (int i = 0; i < kShortPath; ++i) ev[i] = (uint32_t)i < n_ev ? mine[i] : 0u;
  uint32_t rows[kShortPath / 3];  // three 10-bit rows per word
#pragma unroll
  for (int i = 0; i < kShortPath / 3; ++i) rows[i] = 0;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kShortPath; ++i) {
    if ((uint32_t)i < n_max) {  // warp-uniform
      const bool on = (uint32_t)i < n_ev;
      const uint32_t s = ev[i];
      uint32_t k = 1;
#pragma unroll
      for (int j = 0; j < i; ++j) k += ev[j] == s ? 1u : 0u;
      uint32_t r = (s * 0x9e3779b1u + k * 0x85ebca6bu) >> 22;
      static_assert(kShortRows == 1024, "hash shift assumes 1,024 rows");
      const unsigned long long want = ((unsigned long long)((k << 8) | 0xffu) << 32) | s;  // a claim: lane field open
      bool pending = on;
      while (__any_sync(0xffffffffu, pending)) {  // warp-synchronous probes: the lanes leave together
        if (pending) {
          unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(ent + r);
          if (cur == kFree) cur = atomicCAS(ent + r, kFree, want);
          // ours if the row was free (now claimed) or holds (s, k) already; the lane byte is ignored
          if (cur == kFree || ((cur ^ want) & 0xffffff00ffffffffull) == 0ull) pending = false;
          else r = (r + 1) & (kShortRows - 1);
        }
      }
      if (on) atomicMin(reinterpret_cast<uint32_t*>(ent + r) + 1, (k << 8) | (uint32_t)lane);
      rows[i / 3] |= r << (10 * (i % 3));
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kShortPath; ++i) {
    if ((uint32_t)i < n_max) {
      const bool on = (uint32_t)i < n_ev;
      const uint32_t r = (rows[i / 3] >> (10 * (i % 3))) & 1023u;
      const uint32_t y = reinterpret_cast<const uint32_t*>(ent + r)[1];
      const uint32_t pv = i ? ev[i > 0 ? i - 1 : 0] >> 1 : prev0;
      sink.emit(on && (y & 0xffu) == (uint32_t)lane, (pv ^ ev[i]) & hmask, lane);
    }
  }
  __syncwarp();
  return true;
}

// exact a / b for a < 2^23, b >= 1: float quotient is within 1 of the true one
__device__ __forceinline__ uint32_t div_small(uint32_t a, uint32_t b, float rb) {
  uint32_t q = (uint32_t)((float)a * rb);
  const uint32_t r = a - q * b;
  if ((int32_t)r < 0) --q;             // overshoot by one
  else if (r >= b) ++q;                // undershoot by one
  return q;
}

// bytes of shared memory the exec's counters take in mode MODE
__host__ __device__ constexpr size_t counters_smem(int mode, uint32_t H) {
  return mode == kCntPacked ? (size_t)H * 2 : (mode == kCntHashed ? (size_t)kHashCap * 8 : 0);
}

template <int MODE>
__global__ void __launch_bounds__(kEdgeWarps * 32, 1) hfz_k_edge_record(const EdgeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);  // packed: H / 2 words; hashed: keys + counts
  uint8_t* pool = smem + counters_smem(MODE, p.H);
  const int lane = threadIdx.x & 31;
  __shared__ unsigned long long s_events;
  __shared__ uint32_t s_next;
  __shared__ uint32_t s_defer[kDeferCap];  // non-coherent simulated warps waiting for a table-owning warp
  __shared__ uint32_t s_dhead, s_dtail;    // tickets taken by consumers / producers
  __shared__ uint32_t s_left;              // non-owner warps that have left the pop loop of this pass
  __shared__ uint32_t s_overflow;  // a packed counter came near 16 bits / the hashed table is nearly full: replay with wide counters
  __shared__ uint32_t s_used;      // rows of the hashed table in use
  const bool owner = (threadIdx.x >> 5) < (uint32_t)kPool;
  const uint32_t n_nonowners = kEdgeWarps - kPool;
#ifdef HFZ_EDGE_PROF
  __shared__ unsigned long long s_prof[2][16];
  if (threadIdx.x < 32) s_prof[threadIdx.x >> 4][threadIdx.x & 15] = 0;
  unsigned long long* prof = s_prof[owner ? 0 : 1];
  const long long t_kernel = clock64();
  __syncthreads();
#else
  unsigned long long* prof = nullptr;
  (void)prof;
#endif
  PROF_DECL;
  if (threadIdx.x < kDeferCap) s_defer[threadIdx.x] = 0;
  uint32_t* prev_tab = p.prev_scratch + (size_t)blockIdx.x * p.prev_stride;
  const uint32_t hmask = p.H - 1;

  for (uint64_t ei = blockIdx.x; ei < p.n_exec; ei += gridDim.x) {
   const uint64_t e = p.exec_list ? p.exec_list[ei] : ei;
   uint32_t* ghist = reinterpret_cast<uint32_t*>(p.raw + e * p.rec_bytes + p.H);
   for (int attempt = 0; attempt < 2; ++attempt) {
    const bool packed = attempt == 0;  // first attempt: counters in shared memory (mode MODE)
    Counters counters;
    counters.base = packed ? hist : ghist;
    counters.mode = packed ? MODE : kCntWide;
    counters.overflow = &s_overflow;
    counters.used = &s_used;
    if (packed && MODE == kCntHashed) {
      for (uint32_t i = threadIdx.x; i < kHashCap; i += blockDim.x) {
        hist[i] = kHashEmpty;
        hist[kHashCap + i] = 0;
      }
      // the record's device half: zero-fill now (fire-and-forget stores under the replay), scatter the
      // dirty slots at the end
      uint4* z = reinterpret_cast<uint4*>(ghist);
      for (uint32_t i = threadIdx.x; i < p.H / 4; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    } else {
      for (uint32_t i = threadIdx.x; i < (packed ? p.H / 2 : p.H); i += blockDim.x) counters.base[i] = 0;
    }
    if (threadIdx.x == 0) {
      s_events = 0;
      s_overflow = 0;
      s_used = 0;
    }
    const uint64_t l0 = p.launch_off[e], l1 = p.launch_off[e + 1];
    // prev is carried across launches per flattened gtid (hdvm.cpp:376,426-430): only needed
    // when the exec has more than one launch
    const bool multi = l1 - l0 > 1;
    // Launches of one exec usually share one geometry.  Thread j then has the same flattened
    // gtid in every launch, so its carried prev is the last site of thread j in the nearest
    // earlier launch where it ran any events -- read straight from the trace.  No prev table,
    // no ordering between launches: all simulated warps of the exec go into ONE work queue and
    // the few long (divergent) warps of a launch no longer hold the others at a barrier.
    bool uniform = multi;
    if (multi) {
      const uint32_t* d0 = p.dims + l0 * 6;
      uniform = launch_valid(d0);
      if (uniform) {  // the shared work counter is 32 bits wide
        const uint64_t tpb0 = (uint64_t)d0[3] * d0[4] * d0[5];
        const uint64_t nsw0 = (uint64_t)d0[0] * d0[1] * d0[2] * ((tpb0 + 31) / 32);
        uniform = nsw0 * (l1 - l0) < (1ull << 31);
      }
      for (uint64_t l = l0 + 1; l < l1 && uniform; ++l) {
        const uint32_t* d = p.dims + l * 6;
        uniform = d[0] == d0[0] && d[1] == d0[1] && d[2] == d0[2] && d[3] == d0[3] && d[4] == d0[4] &&
                  d[5] == d0[5];
      }
    }
    if (multi && !uniform) {
      uint64_t mx = 0;
      for (uint64_t l = l0; l < l1; ++l) {
        const uint32_t* d = p.dims + l * 6;
        if (launch_valid(d)) {
          const uint64_t tt = (uint64_t)d[0] * d[1] * d[2] * d[3] * d[4] * d[5];
          mx = tt > mx ? tt : mx;
        }
      }
      for (uint64_t i = threadIdx.x; i < mx; i += blockDim.x) prev_tab[i] = 0;
    }
    __syncthreads();
    PROF(prof, 12);

    uint64_t my_events = 0;
    // uniform: one pass over all launches (sw runs over launch-major simulated warps)
    const uint64_t l_step = uniform ? (l1 - l0) : 1;
    for (uint64_t l = l0; l < l1; l += l_step) {
      const uint32_t* d = p.dims + l * 6;
      if (threadIdx.x == 0) {
        s_next = 0;
        s_dhead = 0;
        s_dtail = 0;
        s_left = 0;
      }
      __syncthreads();
      PROF(prof, 12);
      if (launch_valid(d)) {
        // all of these fit 32 bits: blocks * tpb <= 2^22, tpb <= 1024 (launch_valid)
        const uint32_t gx = d[0], gy = d[1], bdx = d[3], bdy = d[4], bdz = d[5];
        const uint32_t tpb = bdx * bdy * bdz, blocks = gx * gy * d[2];
        const uint32_t wpb = (tpb + 31) / 32;
        const uint32_t n_sw = blocks * wpb;  // <= 2^22 (launch_valid)
        const float r_wpb = 1.0f / (float)wpb, r_gx = 1.0f / (float)gx, r_gy = 1.0f / (float)gy,
                    r_bdx = 1.0f / (float)bdx, r_bdy = 1.0f / (float)bdy;
        const uint64_t n_q = (uint64_t)n_sw * l_step;
        // simulated warps are handed out dynamically: divergent ones take far longer
        for (;;) {
          uint32_t q = 0;
          bool deferred = false;
          if (owner) {  // table-owning warps serve the queue of handed-over simulated warps first
            uint32_t got = 0;
            if (lane == 0) {
              uint32_t h = atomicAdd(&s_dhead, 0u);
              while (h < atomicAdd(&s_dtail, 0u)) {
                const uint32_t seen = atomicCAS(&s_dhead, h, h + 1);
                if (seen == h) {  // ticket h is ours: its slot is filled by a producer that already holds a ticket
                  uint32_t* slot = &s_defer[h % kDeferCap];
                  while ((got = atomicExch(slot, 0u)) == 0u) {
                  }
                  break;
                }
                h = seen;
              }
            }
            got = __shfl_sync(0xffffffffu, got, 0);
            if (got) {
              q = got - 1;
              deferred = true;
#ifdef HFZ_EDGE_DEBUG
              if (q >= n_q && lane == 0) printf("bad deferred q %u n_q %llu blk %d warp %d\n", q, (unsigned long long)n_q, blockIdx.x, threadIdx.x >> 5);
#endif
            }
          }
          if (!deferred) {
            uint32_t done = 0;
            if (lane == 0) {
              q = atomicAdd(&s_next, 0u) < n_q ? atomicAdd(&s_next, 1u) : (uint32_t)n_q;  // n_q < 2^31
              if (q >= n_q && owner)  // an owner leaves once no warp can hand over any more work
                done = atomicAdd(&s_left, 0u) == n_nonowners && atomicAdd(&s_dhead, 0u) == atomicAdd(&s_dtail, 0u);
            }
            q = __shfl_sync(0xffffffffu, q, 0);
            if (q >= n_q) {
              if (!owner) break;
              if (__shfl_sync(0xffffffffu, done, 0)) break;
              __nanosleep(200);
              PROF(prof, 10);
              continue;
            }
          }
          PROF(prof, 0);
#ifdef HFZ_EDGE_DEBUG
          if (q >= n_q && lane == 0) printf("bad q %u n_q %llu blk %d warp %d deferred %d\n", q, (unsigned long long)n_q, blockIdx.x, threadIdx.x >> 5, (int)deferred);
#endif
          const uint32_t lq = uniform ? q / n_sw : 0u;  // launch within the exec (uniform pass only)
          const uint32_t sw = q - lq * n_sw;
          const uint64_t t0 = p.thread_off[l + lq];
          const uint32_t bl = div_small(sw, wpb, r_wpb), tl = (sw - bl * wpb) * 32 + lane;
          const bool active = tl < tpb;
          uint64_t e0 = 0, e1 = 0, gtid = 0;
          uint32_t prev_u = 0;
          if (active) {
            const uint64_t j = (uint64_t)bl * tpb + tl;  // thread index within its launch
            const uint64_t t = t0 + j;
            e0 = p.ev_off[t];
            e1 = p.ev_off[t + 1];
            if (uniform) {
              for (uint32_t lb = lq; lb > 0;) {  // nearest earlier launch where thread j ran events
                --lb;
                const uint64_t tb = p.thread_off[l + lb] + j;
                const uint64_t b1 = p.ev_off[tb + 1];
                if (b1 > p.ev_off[tb]) {
                  prev_u = p.sites[b1 - 1] >> 1;
                  break;
                }
              }
            } else if (multi) {
              const uint32_t bxy = div_small(bl, gx, r_gx), bx = bl - bxy * gx;
              const uint32_t bz = div_small(bxy, gy, r_gy), by = bxy - bz * gy;
              const uint32_t txy = div_small(tl, bdx, r_bdx), tx = tl - txy * bdx;
              const uint32_t tz = div_small(txy, bdy, r_bdy), ty = txy - tz * bdy;
              const uint64_t rowx = (uint64_t)bdx * gx;  // threads per grid row
              gtid = tx + (uint64_t)bx * bdx + (ty + (uint64_t)by * bdy) * rowx +
                     (tz + (uint64_t)bz * bdz) * rowx * bdy * gy;
            }
          }
          const uint32_t n_ev = (uint32_t)(e1 - e0);
          {
            // Traces are contiguous in thread order and the CTA's warps pop simulated warps in
            // order, so what the pop kEdgeWarps ahead will read lies about kEdgeWarps times this
            // warp's own span further on: pull it (and its offsets) into L2 now.
            const uint64_t first = __shfl_sync(0xffffffffu, e0, 0);
            const uint64_t last = __shfl_sync(0xffffffffu, e1, 31);
            const uint64_t span = (last - first) * 4;
            if (span) {
              const uint64_t lines = min((span + 127) / 128, (uint64_t)32);
              if ((uint64_t)lane < lines)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint8_t*>(p.sites + last) +
                                                              span * (kEdgeWarps - 1) + (uint64_t)lane * 128));
            }
            if (lane < 2)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint8_t*>(
                  p.ev_off + t0 + (uint64_t)bl * tpb + (uint64_t)(sw - bl * wpb) * 32 + (uint64_t)kEdgeWarps * 32) + lane * 128));
          }
          PROF(prof, 1);
          const bool use_tab = multi && !uniform;
          uint32_t prev0 = uniform ? prev_u : ((use_tab && active) ? prev_tab[gtid] : 0);
          const uint32_t amask = __ballot_sync(0xffffffffu, active);
          const int lead = __ffs(amask) - 1;  // lowest active lane (always lane 0 of the sim warp)

          // ---- fast path: every active lane walks the same sequence as the lead lane.
          // No votes inside the loop: each lane compares against the lead's sites read
          // straight from global memory (a broadcast load), one vote at the end.
          const uint32_t n_lead = __shfl_sync(0xffffffffu, n_ev, lead);
          const uint64_t e0_lead = __shfl_sync(0xffffffffu, e0, lead);
          const uint32_t* sl = p.sites + e0_lead;
          const uint32_t* sm = p.sites + e0;
          bool same_l = !active || n_ev == n_lead;
          if (same_l && active) {
            uint32_t diff = 0;
#pragma unroll 8
            for (uint32_t i = 0; i < n_lead; ++i) diff |= sl[i] ^ sm[i];
            same_l = diff == 0;
          }
          const bool coherent = __all_sync(0xffffffffu, same_l);
          PROF(prof, 2);
          if (coherent) {
            // only the lead lane can bump, on every event; event i is independent of the
            // others (prev_i = site_{i-1} >> 1), so the lanes share the bumps
            const uint32_t prev_lead = __shfl_sync(0xffffffffu, prev0, lead);
            for (uint32_t i = lane; i < n_lead; i += 32) {
              const uint32_t s = sl[i];
              const uint32_t pv = i ? (sl[i - 1] >> 1) : prev_lead;
              counters.bump_slot((pv ^ s) & hmask);
            }
            if (lane == 0) my_events += n_lead;
            if (use_tab && active && n_ev) prev_tab[gtid] = sm[n_ev - 1] >> 1;
            PROF(prof, 3);
            continue;
          }

          // ---- general path: needs a site table.  A warp without one hands the simulated warp over.
          if (!owner) {
            if (lane == 0) {
              const uint32_t ticket = atomicAdd(&s_dtail, 1u);
              uint32_t* slot = &s_defer[ticket % kDeferCap];
              while (atomicCAS(slot, 0u, q + 1) != 0u) {  // queue full: the owners drain it with priority
                __nanosleep(100);
              }
            }
            PROF(prof, 4);
            continue;
          }
          uint8_t* tmem = pool + (size_t)(threadIdx.x >> 5) * kTabBytes;
          PROF(prof, 1);
          CounterSink sink{counters, 0u};
          if (!transposed_path(tmem, p.sites, e0, n_ev, active, prev0, sink, hmask, lane, prof)) {
            WarpTable tab;
            tab.keys = reinterpret_cast<unsigned long long*>(tmem);
            tab.m = reinterpret_cast<uint32_t*>(tab.keys + kRows);
            tab.c = tab.m + kRows;
            tab.stamp = tab.c + kRows;
            tab.used = tab.stamp + kRows;
            general_path(tab, p.sites, e0, n_ev, prev0, sink, hmask, lane);
          }
          my_events += sink.n;
          __syncwarp();
          if (use_tab && active && n_ev) prev_tab[gtid] = p.sites[e1 - 1] >> 1;
#ifdef HFZ_EDGE_PROF
          _pt = clock64();  // (the table path accounts for itself)
#endif
        }
        if (!owner && lane == 0) atomicAdd(&s_left, 1u);
      }
      PROF(prof, 0);
      __syncthreads();  // prev table and counters are launch-ordered
      PROF(prof, 11);
    }
    // block-reduce the event tally, flush the counters (copy, merge_device_into_map)
    // one 64-bit shared-memory atomic per WARP: 64-bit adds on shared memory are CAS loops, and 768
    // threads retrying on one word at the end of every exec were 13 % of the kernel's instructions
    {
      uint32_t lo = (uint32_t)my_events, hi = (uint32_t)(my_events >> 32);
      const uint32_t lo_sum = __reduce_add_sync(0xffffffffu, lo);           // low words: carries recovered below
      uint32_t carry = 0;
      if (__any_sync(0xffffffffu, hi != 0u) || __reduce_max_sync(0xffffffffu, lo) > 0x07ffffffu) {
        // rare: exact 64-bit warp sum by shuffles
        uint64_t v = my_events;
        for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        if (lane == 0 && v) atomicAdd(&s_events, (unsigned long long)v);
      } else if (lane == 0 && lo_sum) {
        (void)carry;
        atomicAdd(&s_events, (unsigned long long)lo_sum);  // 32 lanes x < 2^27 cannot wrap 32 bits
      }
    }
    __syncthreads();
    const bool redo = packed && s_overflow != 0;
    if (packed && !redo) {
      if (MODE == kCntHashed) {  // scatter the dirty slots over the zero-filled device half
        for (uint32_t i = threadIdx.x; i < kHashCap; i += blockDim.x) {
          const uint32_t k = hist[i];
          if (k != kHashEmpty) ghist[k] = hist[kHashCap + i];
        }
      } else {  // unpack: two counters per word -> the record's u32 device half
        uint2* dst = reinterpret_cast<uint2*>(ghist);
        for (uint32_t i = threadIdx.x; i < p.H / 2; i += blockDim.x) {
          const uint32_t w = hist[i];
          dst[i] = make_uint2(w & 0xffffu, w >> 16);
        }
      }
    }
    if (!redo && threadIdx.x == 0 && p.warp_events) p.warp_events[e] = s_events;
    __syncthreads();
    PROF(prof, 12);
    if (!redo) break;
   }
  }
#ifdef HFZ_EDGE_PROF
  __syncthreads();
  if (threadIdx.x < 32) atomicAdd(&g_edge_prof[threadIdx.x >> 4][threadIdx.x & 15], s_prof[threadIdx.x >> 4][threadIdx.x & 15]);
  if (threadIdx.x == 0) atomicAdd(&g_edge_prof[0][15], (unsigned long long)(clock64() - t_kernel));
#endif
}


// ---------------------------------------------------------------------------
// Flat path (the default): decide, then count.
//
// Which events bump is a question about ONE simulated warp (its site table, the lanes' carried prev);
// only the counting is per exec.  The per-exec kernel above does both under one CTA: the counters
// take 64 KB of the CTA's shared memory, so only half of its warps can own a site table, and every
// exec ends at a CTA-wide barrier behind its slowest divergent warp (a quarter of the warp-time).
// Here the two halves are separate launches:
//   hfz_k_edge_classify   ALL simulated warps of a chunk of execs are one flat queue (a global counter,
//                      kPop warps per pop); no shared memory, no barrier.  A coherent warp (every lane
//                      walked the lead lane's sequence -- the SIMT common case) is recognised straight
//                      from the trace: its events are contiguous, so they are dealt out 32 per coalesced
//                      load and event g is compared with event g - n (the same position one lane down).
//                      Only its lead lane bumps, on every event.  The slots to bump go to the simulated
//                      warp's own region of a scratch list (indexed like the trace: a warp never bumps
//                      more often than it has events) -- one ballot per round, no atomics.  The other
//                      (divergent) warps are appended to a list;
//   hfz_k_edge_divergent  the listed warps, a flat queue again; shared memory holds nothing but one site
//                      table per real warp (22 per SM), so every warp can take one and none waits;
//   hfz_k_edge_count      one CTA per exec streams the exec's bump lists into u32 counters in SHARED
//                      memory (shared-memory atomics; 64 KB per CTA, so three execs are in flight per SM
//                      and one's zero / flush phases hide behind the others' list reads) and flushes
//                      them to the record: still no global atomic per hit.  An exec with fewer than 65,536
//                      bumps in all (summed first) packs two 16-bit counters per word -- 32,768 slots per
//                      pass; any other exec counts in full u32 words, 16,384 slots per pass, saturating.
//                      Either way a counter cannot overflow, so nothing is ever replayed.
// Launches of an exec that differ in geometry carry prev per flattened gtid IN LAUNCH ORDER
// (hdvm.cpp:376,426-430), which a flat queue cannot honour: those execs (and execs whose thread
// offsets are not a CSR of their launch sizes) are left to the per-exec kernel.
constexpr int kFlatWarps = 22;       // divergent kernel: 22 site tables = 226,688 bytes of shared memory
constexpr int kClassifyWarps = 16;   // classify kernel: no shared memory, two CTAs per SM
constexpr uint32_t kPop = 16;        // simulated warps per pop
constexpr uint32_t kCountSlots = 16384;  // u32 counters per pass of the count kernel: 64 KB, three CTAs (execs) in flight per SM
constexpr int kCountWarps = 16;

struct FlatParams {
  const uint64_t* launch_off;
  const uint32_t* dims;
  const uint64_t* thread_off;
  const uint64_t* ev_off;
  const uint32_t* sites;
  uint64_t n_exec, n_launch;
  uint32_t H;
  uint64_t rec_bytes;
  uint8_t* raw;
  uint64_t* warp_events;
  // written by hfz_k_edge_prep / hfz_k_edge_scan
  uint32_t* nsw;        // [n_launch] simulated warps of a launch; 0 = invalid launch or exec left to the per-exec kernel
  uint64_t* sw_off;     // [n_launch + 1] exclusive prefix of nsw: the flat queue
  uint32_t* l_exec;     // [n_launch] exec of a launch
  uint8_t* elig;        // [n_exec] 1 = flat path
  uint64_t* exec_ev0;   // [n_exec + 1] first event of an exec (index into sites)
  uint64_t* exec_sw0;   // [n_exec + 1] first flat simulated warp of an exec
  uint32_t* inelig;     // [n_exec] execs left to the per-exec kernel
  unsigned long long* small;  // [0] their number, [1] max threads of their launches, [2] pop counter, [3]/[4] min/max nsw
  // one chunk of execs
  uint64_t e_lo, e_hi;  // execs
  uint64_t q_lo, q_hi;  // flat simulated warps
  uint64_t l_lo, l_hi;  // launches
  uint64_t ev_lo;       // first event
  uint32_t uni_nsw;     // every launch of the batch has this many simulated warps (0 = they differ)
  uint32_t* scratch;    // bump slots; a simulated warp's list starts at (its first event - ev_lo)
  uint64_t* rec_first;  // [q_hi - q_lo] first event of the simulated warp (list items only)
  uint32_t* rec_cnt;    // [q_hi - q_lo] its bumps; | kSegFlag: listed in scratch, else in its line
  uint32_t* div_list;   // [q_hi - q_lo] simulated warps (chunk-relative) that need a site table; small[5] of them
  uint32_t* lines;      // [q_hi - q_lo][32] a coherent warp's bump slots: one 128-byte line per simulated warp
  // list output (hfz_edge_record_batch_lists): per exec list_cap (logical slot, count) pairs, zero-filled by
  // the host call before the kernels run; list_n[e] = the exec's distinct slots or ~0u (not listed)
  uint2* list_out;
  uint32_t list_cap;
  uint32_t* list_n;
};
constexpr uint32_t kSegFlag = 0x80000000u;  // rec_cnt: the bumps are a list in scratch (rec_first), not a line

// one thread per exec: eligibility, simulated warps per launch, the exec's first event
__global__ void __launch_bounds__(256) hfz_k_edge_prep(const FlatParams p) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= p.n_exec; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t l0 = p.launch_off[e];
    if (l0 > p.n_launch || (e < p.n_exec && (p.launch_off[e + 1] < l0 || p.launch_off[e + 1] > p.n_launch))) {
      p.small[7] = 1;  // launch_off is not a CSR over n_launch launches: the host refuses the batch
      p.exec_ev0[e] = 0;
      if (e < p.n_exec) p.elig[e] = 1;
      continue;
    }
    p.exec_ev0[e] = p.n_launch ? p.ev_off[p.thread_off[l0]] : 0;
    if (e == p.n_exec) break;
    const uint64_t l1 = p.launch_off[e + 1];
    bool ok = true;
    unsigned long long mx = 0;
    for (uint64_t l = l0; l < l1; ++l) {
      const uint32_t* d = p.dims + l * 6;
      if (l > l0) {
        const uint32_t* d0 = p.dims + l0 * 6;
        ok = ok && d[0] == d0[0] && d[1] == d0[1] && d[2] == d0[2] && d[3] == d0[3] && d[4] == d0[4] && d[5] == d0[5];
      }
      const uint64_t ta = p.thread_off[l], tb = p.thread_off[l + 1];
      if (launch_valid(d)) {
        const unsigned long long tt = (unsigned long long)d[0] * d[1] * d[2] * d[3] * d[4] * d[5];
        mx = tt > mx ? tt : mx;
        ok = ok && tb >= ta && tb - ta >= tt;
      } else {
        ok = ok && tb >= ta;
      }
    }
    for (uint64_t l = l0; l < l1; ++l) {
      const uint32_t* d = p.dims + l * 6;
      uint32_t n = 0;
      if (ok && launch_valid(d)) n = d[0] * d[1] * d[2] * ((d[3] * d[4] * d[5] + 31) / 32);  // <= 2^22
      p.nsw[l] = n;
      p.l_exec[l] = (uint32_t)e;
      if (ok) {
        atomicMax(p.small + 3, ~(unsigned long long)n);  // (zero-initialised: the complement's max is the min)
        atomicMax(p.small + 4, (unsigned long long)n);
      }
    }
    p.elig[e] = ok ? 1 : 0;
    if (!ok) {
      p.inelig[atomicAdd(p.small + 0, 1ull)] = (uint32_t)e;
      atomicMax(p.small + 1, mx);
    }
  }
}

// one CTA: sw_off = exclusive prefix sum of nsw; then the flat start of every exec
__global__ void __launch_bounds__(1024, 1) hfz_k_edge_scan(const FlatParams p) {
  __shared__ unsigned long long wsum[32];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long carry = 0;
  if (threadIdx.x == 0) p.sw_off[0] = 0;
  for (uint64_t base = 0; base < p.n_launch; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    unsigned long long x = i < p.n_launch ? p.nsw[i] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= (uint32_t)d) x += o;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      unsigned long long y = wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, y, d);
        if (lane >= (uint32_t)d) y += o;
      }
      wsum[lane] = y;
    }
    __syncthreads();
    const unsigned long long incl = x + (w ? wsum[w - 1] : 0) + carry;
    if (i < p.n_launch) p.sw_off[i + 1] = incl;
    carry += wsum[31];
    __syncthreads();
  }
  __syncthreads();  // (the CTA's own global writes are visible to it after the barrier)
  for (uint64_t e = threadIdx.x; e <= p.n_exec; e += 1024) {
    const uint64_t l = p.launch_off[e];
    p.exec_sw0[e] = p.sw_off[l <= p.n_launch ? l : p.n_launch];
  }
}

// The launch a flat simulated-warp index belongs to, cached between consecutive items.
struct LaunchCtx {
  uint64_t sw0 = 1, sw1 = 0;  // flat range of the launch (empty: forces a lookup)
  uint64_t t0 = 0, tprev = 0; // first thread of the launch / of the launch before it in the same exec
  uint64_t l = 0, l0 = 0;     // the launch, the first launch of its exec
  uint32_t tpb = 1, wpb = 1;
};
__device__ __forceinline__ void flat_locate(const FlatParams& p, uint64_t q, LaunchCtx& c) {
  uint64_t l;
  if (p.uni_nsw) {
    l = q < (1ull << 32) ? (uint64_t)((uint32_t)q / p.uni_nsw) : q / p.uni_nsw;
    c.sw0 = l * p.uni_nsw;
    c.sw1 = c.sw0 + p.uni_nsw;
  } else {  // last launch with sw_off[l] <= q
    uint64_t lo = p.l_lo, hi = p.l_hi;
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (p.sw_off[mid] <= q) lo = mid; else hi = mid;
    }
    l = lo;
    c.sw0 = p.sw_off[l];
    c.sw1 = p.sw_off[l + 1];
  }
  const uint32_t* d = p.dims + l * 6;
  c.tpb = d[3] * d[4] * d[5];
  c.wpb = (c.tpb + 31) / 32;
  c.l = l;
  c.l0 = p.launch_off[p.l_exec[l]];
  c.t0 = p.thread_off[l];
  c.tprev = l > c.l0 ? p.thread_off[l - 1] : 0;
}
// nearest launch below lb_from (within the exec) where thread j ran events: prev is carried per gtid
// (hdvm.cpp:376,426-430), and with one geometry per exec thread j has the same gtid in every launch
__device__ __forceinline__ uint32_t flat_prev_walk(const FlatParams& p, const LaunchCtx& c, uint64_t j, uint32_t lb_from) {
  for (uint32_t lb = lb_from; lb > 0;) {
    --lb;
    const uint64_t tb = p.thread_off[c.l0 + lb] + j;
    const uint64_t b1 = p.ev_off[tb + 1];
    if (b1 > p.ev_off[tb]) return p.sites[b1 - 1] >> 1;
  }
  return 0u;
}

__global__ void __launch_bounds__(kClassifyWarps * 32, 2) hfz_k_edge_classify(const FlatParams p) {
  const int lane = threadIdx.x & 31;
  const uint32_t hmask = p.H - 1;
  const uint64_t n_items = p.q_hi - p.q_lo;
  // the launch the last simulated warp belonged to (a pop is kPop consecutive warps: usually one launch)
  LaunchCtx c;
  for (;;) {
    unsigned long long qb = 0;
    if (lane == 0) qb = atomicAdd(p.small + 2, (unsigned long long)kPop);
    qb = __shfl_sync(0xffffffffu, qb, 0);
    if (qb >= n_items) break;
    const uint64_t qe = qb + kPop < n_items ? qb + kPop : n_items;
    // software pipeline over the pop's items: while item i is worked on, the event offsets of item
    // i + 1 are in flight, and once they have landed its events are pulled into L2
    bool have_next = false;
    uint64_t nx_e0 = 0, nx_e1 = 0, nx_pa = 0, nx_pb = 0;  // (nx_pa / nx_pb / nx_ps: lane 0 only)
    uint32_t nx_ps = 0, nx_bl = 0, nx_wi = 0;
    for (uint64_t qi = qb; qi < qe; ++qi) {
      const uint64_t q = p.q_lo + qi;
      if (q < c.sw0 || q >= c.sw1) {
        have_next = false;
        flat_locate(p, q, c);
      }
      const uint32_t tpb = c.tpb, wpb = c.wpb;
      const uint32_t sw = (uint32_t)(q - c.sw0);
      const uint32_t lq = (uint32_t)(c.l - c.l0);  // launch within its exec: every earlier one has this geometry
      const bool piped = have_next;
      // block and warp within the block: carried over from the look-ahead of the item before (no division)
      const uint32_t bl = piped ? nx_bl : sw / wpb;
      const uint32_t wi = piped ? nx_wi : sw - bl * wpb;
      const uint32_t tl = wi * 32 + lane;
      const bool active = tl < tpb;
      const uint64_t j = (uint64_t)bl * tpb + tl;  // thread within its launch
      uint64_t e0 = 0, e1 = 0, pa = 0, pb = 0;
      uint32_t ps = 0;  // the site that ends the lead lane's events one launch back
      if (piped) {
        e0 = nx_e0;
        e1 = nx_e1;
        pa = nx_pa;
        pb = nx_pb;
        ps = nx_ps;
      } else if (active) {
        e0 = p.ev_off[c.t0 + j];
        e1 = p.ev_off[c.t0 + j + 1];
      }
      have_next = qi + 1 < qe && q + 1 < c.sw1;
      bool nx_active = false;
      if (have_next) {
        const bool wrap = wi + 1 == wpb;  // the next warp of the block, or the first one of the next block
        const uint32_t bl2 = wrap ? bl + 1 : bl, wi2 = wrap ? 0u : wi + 1, tl2 = wi2 * 32 + lane;
        nx_bl = bl2;
        nx_wi = wi2;
        nx_active = tl2 < tpb;
        nx_e0 = nx_e1 = 0;
        const uint64_t j2 = (uint64_t)bl2 * tpb + tl2;
        if (nx_active) {
          nx_e0 = p.ev_off[c.t0 + j2];
          nx_e1 = p.ev_off[c.t0 + j2 + 1];
        }
        if (lq && lane == 0) {
          nx_pa = p.ev_off[c.tprev + j2];
          nx_pb = p.ev_off[c.tprev + j2 + 1];
        }
      }
      if (lq && lane == 0 && !piped) {  // the lead lane's carried prev: usually the end of its events one launch back
        pa = p.ev_off[c.tprev + j];
        pb = p.ev_off[c.tprev + j + 1];
      }
      const uint32_t n_ev = (uint32_t)(e1 - e0);
      const uint64_t first = __shfl_sync(0xffffffffu, e0, 0);
      const uint32_t n_lead = __shfl_sync(0xffffffffu, n_ev, 0);
      const uint32_t n_act = (uint32_t)__popc(__ballot_sync(0xffffffffu, active));
      const bool same_n = __all_sync(0xffffffffu, !active || n_ev == n_lead);
      const uint32_t* ev = p.sites + first;
      uint32_t prev_lead = 0;
      if (lq && lane == 0) {
        if (pb > pa) prev_lead = (piped ? ps : p.sites[pb - 1]) >> 1;
        else prev_lead = flat_prev_walk(p, c, j, lq - 1);
      }
      // ---- coherent?  every active lane walked the lead lane's sequence
      bool coherent = false;
      uint32_t r0 = 0;
      if (same_n && n_lead <= 32u) {
        // the warp's events are contiguous: dealt 32 per load; the lead's events are lanes 0 .. n_lead - 1
        // of the first round
        const uint32_t N = n_act * n_lead;  // <= 1,024
        uint32_t diff = 0;
        if (n_lead) {
          // lane t's i-th event equals lane t - 1's: event g against event g - n_lead, both streams coalesced
          // (blocks of 8 rounds = 16 loads in flight, all predicated: a remainder loop would take its
          // rounds one memory latency at a time)
          const uint32_t* evb = ev - n_lead;
          r0 = (uint32_t)lane < N ? ev[lane] : 0u;
          {
            uint32_t a[7], b[8];
            b[0] = ((uint32_t)lane >= n_lead && (uint32_t)lane < N) ? evb[lane] : r0;
#pragma unroll
            for (int u = 1; u < 8; ++u) {
              const uint32_t g = 32u * u + lane;
              a[u - 1] = g < N ? ev[g] : 0u;
              b[u] = g < N ? evb[g] : 0u;
            }
            diff = r0 ^ b[0];
#pragma unroll
            for (int u = 1; u < 8; ++u) diff |= a[u - 1] ^ b[u];
          }
          for (uint32_t g0 = 256; g0 < N; g0 += 256) {  // warp-uniform
            uint32_t a[8], b[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const uint32_t g = g0 + 32u * u + lane;
              a[u] = g < N ? ev[g] : 0u;
              b[u] = g < N ? evb[g] : 0u;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) diff |= a[u] ^ b[u];
          }
        }
        coherent = __all_sync(0xffffffffu, diff == 0u);
      } else if (same_n) {  // long paths: each lane against the lead's, read as a broadcast load
        uint32_t diff = 0;
        if (active) {
          const uint32_t* mine = p.sites + e0;
#pragma unroll 8
          for (uint32_t i = 0; i < n_lead; ++i) diff |= ev[i] ^ mine[i];
        }
        coherent = __all_sync(0xffffffffu, diff == 0u);
      }
      if (have_next) {  // the next item's events into L2, one 128-byte line per lane (4 KB covers the usual warp)
        const uint32_t am2 = __ballot_sync(0xffffffffu, nx_active);
        const uint64_t f2 = __shfl_sync(0xffffffffu, nx_e0, 0);
        const uint64_t l2 = __shfl_sync(0xffffffffu, nx_e1, 31 - __clz((int)am2));
        const uint8_t* a2 = reinterpret_cast<const uint8_t*>(p.sites + f2) + (uint64_t)lane * 128;
        if (a2 < reinterpret_cast<const uint8_t*>(p.sites + l2)) asm volatile("prefetch.global.L2 [%0];" ::"l"(a2));
        if (lq && lane == 0 && nx_pb > nx_pa) nx_ps = p.sites[nx_pb - 1];
      }
      if (coherent) {
        // only the lead lane can bump, on every event; event i needs site i - 1 only
        if (n_lead <= 32u) {  // the usual case: the bumps fill (part of) the warp's own 128-byte line
          const uint32_t up = __shfl_up_sync(0xffffffffu, r0, 1);
          if ((uint32_t)lane < n_lead) p.lines[qi * 32 + lane] = ((lane ? up >> 1 : prev_lead) ^ r0) & hmask;
          if (lane == 0) p.rec_cnt[qi] = n_lead;
        } else {
          ListSink sink{p.scratch + (first - p.ev_lo), 0u};
          for (uint32_t i0 = 0; i0 < n_lead; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool f = i < n_lead;
            const uint32_t s = f ? ev[i] : 0u;
            const uint32_t pv = (f && i) ? ev[i - 1] >> 1 : prev_lead;
            sink.emit(f, (pv ^ s) & hmask, lane);
          }
          if (lane == 0) {
            p.rec_first[qi] = first;
            p.rec_cnt[qi] = sink.n | kSegFlag;
          }
        }
      } else if (lane == 0) {  // needs a site table: left to hfz_k_edge_divergent
        p.div_list[atomicAdd(p.small + 5, 1ull)] = (uint32_t)qi;
      }
    }
  }
}


// The simulated warps hfz_k_edge_classify set aside: replayed lane by lane with a site table per real warp.
__global__ void __launch_bounds__(kFlatWarps * 32, 1) hfz_k_edge_divergent(const FlatParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  uint8_t* tmem = smem + (size_t)(threadIdx.x >> 5) * kTabBytes;
  const uint32_t hmask = p.H - 1;
  const unsigned long long n_div = p.small[5];
  LaunchCtx c;
  for (;;) {
    unsigned long long di = 0;
    if (lane == 0) di = atomicAdd(p.small + 6, 1ull);
    di = __shfl_sync(0xffffffffu, di, 0);
    if (di >= n_div) break;
    const uint64_t qi = p.div_list[di];
    const uint64_t q = p.q_lo + qi;
    if (q < c.sw0 || q >= c.sw1) flat_locate(p, q, c);
    const uint32_t sw = (uint32_t)(q - c.sw0), lq = (uint32_t)(c.l - c.l0);
    const uint32_t bl = sw / c.wpb, tl = (sw - bl * c.wpb) * 32 + lane;
    const bool active = tl < c.tpb;
    const uint64_t j = (uint64_t)bl * c.tpb + tl;
    uint64_t e0 = 0, e1 = 0;
    uint32_t prev0 = 0;
    if (active) {
      e0 = p.ev_off[c.t0 + j];
      e1 = p.ev_off[c.t0 + j + 1];
      if (lq) prev0 = flat_prev_walk(p, c, j, lq);
    }
    const uint32_t n_ev = (uint32_t)(e1 - e0);
    const uint64_t first = __shfl_sync(0xffffffffu, e0, 0);
    ListSink sink{p.scratch + (first - p.ev_lo), 0u};
    __syncwarp();
    if (!short_divergent_path(tmem, p.sites, e0, n_ev, prev0, sink, hmask, lane) &&
        !transposed_path(tmem, p.sites, e0, n_ev, active, prev0, sink, hmask, lane)) {
      WarpTable tab;
      tab.keys = reinterpret_cast<unsigned long long*>(tmem);
      tab.m = reinterpret_cast<uint32_t*>(tab.keys + kRows);
      tab.c = tab.m + kRows;
      tab.stamp = tab.c + kRows;
      tab.used = tab.stamp + kRows;
      general_path(tab, p.sites, e0, n_ev, prev0, sink, hmask, lane);
    }
    __syncwarp();
    if (lane == 0) {
      p.rec_first[qi] = first;
      p.rec_cnt[qi] = sink.n | kSegFlag;
    }
  }
}

__global__ void __launch_bounds__(kCountWarps * 32, 3) hfz_k_edge_count(const FlatParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  constexpr uint32_t kBigCap = 512;
  __shared__ unsigned long long s_total;
  __shared__ unsigned long long s_big_f[kBigCap];
  __shared__ uint32_t s_big_c[kBigCap];
  __shared__ uint32_t s_nbig;
  __shared__ uint32_t s_wsum[kCountWarps];
  __shared__ uint32_t s_used, s_full;  // dirty-slot table: rows taken / more distinct slots than it holds
  __shared__ uint32_t s_cursor;        // list output: pairs written
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  static_assert(kHashCap * 8 == kCountSlots * 4, "the dirty-slot table and a pass's counters share the 64 KB");
  for (uint64_t e = p.e_lo + blockIdx.x; e < p.e_hi; e += gridDim.x) {
    if (!p.elig[e]) continue;  // the per-exec kernel writes this record
    const uint64_t q0 = p.exec_sw0[e] - p.q_lo, q1 = p.exec_sw0[e + 1] - p.q_lo;
    uint32_t* ghist = p.raw ? reinterpret_cast<uint32_t*>(p.raw + e * p.rec_bytes + p.H) : nullptr;
    // the exec's bumps in all: fewer than 65,536 (the rule) cannot overflow a 16-bit counter, so two
    // counters share a word and a pass covers twice the slots (the whole device half of a 65,536-slot map)
    unsigned long long total = 0;
    for (uint64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) total += p.rec_cnt[q] & ~kSegFlag;
    for (int d = 16; d; d >>= 1) total += __shfl_xor_sync(0xffffffffu, total, d);
    if (lane == 0) s_wsum[w] = (uint32_t)(total < 0xffffffffull ? total : 0xffffffffull);
    if (threadIdx.x == 0) s_total = 0;
    __syncthreads();
    if (lane == 0 && total) atomicAdd(&s_total, total);
    uint64_t bound = 0;  // (saturating per-warp sums: only "below 65,536 or not" matters here)
    for (int i = 0; i < kCountWarps; ++i) bound += s_wsum[i];
    const bool packed = bound < 65536u;
    const uint32_t R = packed ? (p.H < 2 * kCountSlots ? p.H : 2 * kCountSlots) : (p.H < kCountSlots ? p.H : kCountSlots);

    // One walk over the exec's bump lists; add(slot relative to r0) for the slots of [r0, r0 + n).
    // A warp takes 32 consecutive simulated warps: the coherent ones' lines are 4 KB contiguous -- eight
    // 128-bit loads per lane, all in flight at once (lane L, load k: line 4k + L / 8, elements
    // 4 (L % 8) .. + 3); the listed ones (divergent warps) are set aside and then dealt out over ALL
    // warps of the CTA (they sit unevenly in the queue, and the CTA waits for its slowest warp).
    auto walk = [&](uint32_t r0, uint32_t n, auto&& add) {
      for (uint64_t qb = q0 + (uint64_t)w * 32; qb < q1; qb += kCountWarps * 32) {
        const uint64_t q = qb + lane;
        const uint32_t cnt = q < q1 ? p.rec_cnt[q] : 0u;
        const uint4* lines4 = reinterpret_cast<const uint4*>(p.lines + qb * 32) + lane;
        bool seg = (cnt & kSegFlag) != 0u;
        uint64_t f = 0;
        if (seg) {
          f = p.rec_first[q] - p.ev_lo;
          const uint32_t at = atomicAdd(&s_nbig, 1u);
          if (at < kBigCap) {
            s_big_f[at] = f;
            s_big_c[at] = cnt & ~kSegFlag;
            seg = false;
          }
        }
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = lines4[k * 32];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          uint32_t ck = __shfl_sync(0xffffffffu, cnt, 4 * k + (lane >> 3));
          ck = (ck & kSegFlag) ? 0u : ck;  // a listed or absent warp: nothing of its line counts
          const uint32_t i0 = (lane & 7u) * 4u;
          const uint32_t x[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t rel = x[c] - r0;
            if (i0 + c < ck && rel < n) add(rel);
          }
        }
        uint32_t left = __ballot_sync(0xffffffffu, seg);  // more lists than the side list holds: here and now
        while (left) {
          const int k = __ffs(left) - 1;
          left &= left - 1;
          const uint32_t cc = __shfl_sync(0xffffffffu, cnt, k) & ~kSegFlag;
          const uint32_t* list = p.scratch + __shfl_sync(0xffffffffu, f, k);
          for (uint32_t i = lane; i < cc; i += 32) {
            const uint32_t rel = list[i] - r0;
            if (rel < n) add(rel);
          }
        }
      }
      __syncthreads();
      const uint32_t nb = s_nbig < kBigCap ? s_nbig : kBigCap;
      for (uint32_t b = w; b < nb; b += kCountWarps) {
        const uint32_t cc = s_big_c[b];
        const uint32_t* list = p.scratch + s_big_f[b];
#pragma unroll 12
        for (uint32_t i = lane; i < cc; i += 32) {
          const uint32_t rel = list[i] - r0;
          if (rel < n) add(rel);
        }
      }
      __syncthreads();
    };

    bool done = false;
    if (p.H > R || p.list_out) {
      // The device half needs more than one pass of counters (the 262,144-slot map: four), and every pass
      // walks the lists again.  An exec touches a few thousand distinct slots, so first try ONE walk into
      // a dirty-slot table (slot -> saturating u32 count, open addressing, the reference's own dirty list
      // of src/hdvm.cpp:356-366): the record is zero-filled with fire-and-forget stores under the walk and
      // the dirty slots are scattered over it afterwards.  More distinct slots than the table holds:
      // the passes below redo the exec.
      uint32_t* keys = hist;
      uint32_t* counts = hist + kHashCap;
      for (uint32_t i = threadIdx.x; i < kHashCap; i += blockDim.x) {
        keys[i] = kHashEmpty;
        counts[i] = 0;
      }
      if (threadIdx.x == 0) {
        s_nbig = 0;
        s_used = 0;
        s_full = 0;
        s_cursor = 0;
      }
      uint4* zg = reinterpret_cast<uint4*>(ghist);
      if (ghist)
        for (uint32_t i = threadIdx.x; i < p.H / 4; i += blockDim.x) zg[i] = make_uint4(0, 0, 0, 0);
      __syncthreads();
      walk(0u, p.H, [&](uint32_t slot) {
        if (*reinterpret_cast<volatile uint32_t*>(&s_full)) return;
        uint32_t r = (slot * 0x9e3779b1u) >> (32 - kHashBits);
        for (;;) {
          const uint32_t cur = reinterpret_cast<volatile uint32_t*>(keys)[r];
          if (cur == slot) break;
          if (cur == kHashEmpty) {
            const uint32_t old = atomicCAS(keys + r, kHashEmpty, slot);
            if (old == kHashEmpty) {
              if (atomicAdd(&s_used, 1u) >= kHashLimit) s_full = 1u;
              break;
            }
            if (old == slot) break;
          }
          r = (r + 1) & (kHashCap - 1);
        }
        bump(counts + r);
      });
      const bool listed = p.list_out && !s_full && s_used <= p.list_cap;
      if (!s_full) {  // (walk() ended on a barrier: the zero fill is ordered before the scatter)
        uint2* lst = listed ? p.list_out + e * p.list_cap : nullptr;
        for (uint32_t i = threadIdx.x; i < kHashCap; i += blockDim.x) {
          const uint32_t k = keys[i];
          if (k != kHashEmpty) {
            const uint32_t cnt = counts[i];
            if (ghist) ghist[k] = cnt;
            // the exec's touched-slot list, LOGICAL slot indices (device half = upper half of the map), any
            // order: what hfz_feedback_batch_sparse folds without a dense record
            if (lst) lst[atomicAdd(&s_cursor, 1u)] = make_uint2(p.H + k, cnt);
          }
        }
        done = true;
      }
      if (p.list_n && threadIdx.x == 0) p.list_n[e] = listed ? s_used : 0xffffffffu;
      if (!ghist) done = true;  // lists only: an exec that does not fit its list is reported, not counted densely
      __syncthreads();
    }
    for (uint32_t r0 = 0; r0 < p.H && !done; r0 += R) {
      const uint32_t n = p.H - r0 < R ? p.H - r0 : R;
      uint4* z = reinterpret_cast<uint4*>(hist);
      for (uint32_t i = threadIdx.x; i < (packed ? n / 8 : n / 4); i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
      if (threadIdx.x == 0) s_nbig = 0;
      __syncthreads();
      if (packed) walk(r0, n, [&](uint32_t rel) { atomicAdd(hist + (rel >> 1), 1u << ((rel & 1u) * 16u)); });
      else walk(r0, n, [&](uint32_t rel) { bump(hist + rel); });
      uint4* dst = reinterpret_cast<uint4*>(ghist + r0);
      if (packed) {
        const uint2* z2 = reinterpret_cast<const uint2*>(hist);
        for (uint32_t i = threadIdx.x; i < n / 4; i += blockDim.x) {
          const uint2 t = z2[i];
          dst[i] = make_uint4(t.x & 0xffffu, t.x >> 16, t.y & 0xffffu, t.y >> 16);
        }
      } else {
        for (uint32_t i = threadIdx.x; i < n / 4; i += blockDim.x) dst[i] = z[i];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0 && p.warp_events) p.warp_events[e] = s_total;
    __syncthreads();
  }
}

// max simulated threads of any valid launch (sizes the per-CTA prev table)
__global__ void hfz_k_edge_max_threads(const uint32_t* __restrict__ dims, uint64_t n_launch,
                                       unsigned long long* __restrict__ out) {
  unsigned long long mx = 0;
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n_launch;
       l += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* d = dims + l * 6;
    if (launch_valid(d)) {
      const unsigned long long tt = (unsigned long long)d[0] * d[1] * d[2] * d[3] * d[4] * d[5];
      mx = tt > mx ? tt : mx;
    }
  }
  if (mx) atomicMax(out, mx);
}

// ---------------------------------------------------------------------------
// host edges: idx_i = (site_{i-1} >> 1) ^ site_i is independent per event, the never-zero u8
// counter after n hits is (n-1) % 255 + 1 (tests/test_coverage.cpp:34-37) -> histogram + fold.
__global__ void __launch_bounds__(256, 1) hfz_k_host_edge_record(const uint64_t* __restrict__ site_off,
                                                                const uint16_t* __restrict__ sites,
                                                                uint64_t n_exec, uint32_t H,
                                                                uint64_t rec_bytes,
                                                                uint8_t* __restrict__ raw,
                                                                uint32_t* __restrict__ gscratch) {
  extern __shared__ __align__(16) uint8_t smem[];
  // u16 sites: at most 65,536 distinct slots before folding; counters for min(H, 65536) slots
  const uint32_t nslots = H < 65536u ? H : 65536u;
  uint32_t* hist = gscratch ? gscratch + (size_t)blockIdx.x * nslots : reinterpret_cast<uint32_t*>(smem);
  for (uint64_t e = blockIdx.x; e < n_exec; e += gridDim.x) {
    for (uint32_t i = threadIdx.x; i < nslots; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t s0 = site_off[e], s1 = site_off[e + 1];
    for (uint64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
      const uint32_t cur = sites[i];
      const uint32_t prev = i > s0 ? (uint32_t)(sites[i - 1] >> 1) : 0u;  // prev resets per exec
      uint32_t idx = (prev ^ cur) & 0xffffu;
      idx &= (H - 1);  // out-of-half indices are folded (coverage.hpp:25-28)
      atomicAdd(&hist[idx], 1u);
    }
    __syncthreads();
    uint8_t* host_half = raw + e * rec_bytes;
    for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) {
      const uint32_t c = i < nslots ? hist[i] : 0;
      host_half[i] = c ? (uint8_t)((c - 1) % 255 + 1) : 0;
    }
    __syncthreads();
  }
}

}  // namespace

#ifdef HFZ_EDGE_PROF
extern "C" __attribute__((visibility("default"))) int hfz_dbg_edge_prof(unsigned long long* out32, int reset) {
  if (cudaMemcpyFromSymbol(out32, g_edge_prof, sizeof(unsigned long long) * 32) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[32] = {0};
    if (cudaMemcpyToSymbol(g_edge_prof, z, sizeof(z)) != cudaSuccess) return -1;
  }
  return 0;
}
#endif

// The per-exec kernel over all execs (exec_list = NULL) or the listed ones; mx = most threads of any of
// their valid launches (sizes the per-CTA prev table).
static int edge_record_per_exec(hfz_ctx* ctx, const uint64_t* launch_off, const uint32_t* dims,
                                const uint64_t* thread_off, const uint64_t* ev_off, const uint32_t* sites,
                                uint64_t n_exec, const uint32_t* exec_list, unsigned long long mx,
                                uint8_t* raw_maps, uint64_t* warp_events_out) {
  uint32_t grid = (uint32_t)(n_exec < (uint64_t)ctx->num_sms ? n_exec : (uint64_t)ctx->num_sms);
  const uint64_t stride = mx ? mx : 1;
  if (ctx->edge_prev_words < (uint64_t)grid * stride) {
    cudaFree(ctx->edge_prev);
    ctx->edge_prev = nullptr;
    ctx->edge_prev_words = 0;
    if (cudaMalloc(&ctx->edge_prev, (size_t)grid * stride * sizeof(uint32_t)) != cudaSuccess) {
      hfz_set_error("hfz_edge_record_batch: prev table allocation failed (%llu bytes)",
                    (unsigned long long)grid * stride * 4);
      return HFZ_ENOMEM;
    }
    ctx->edge_prev_words = (uint64_t)grid * stride;
  }
  uint32_t* d_prev = ctx->edge_prev;
  cudaError_t e = cudaSuccess;
  EdgeParams p;
  p.launch_off = launch_off;
  p.dims = dims;
  p.thread_off = thread_off;
  p.ev_off = ev_off;
  p.sites = sites;
  p.n_exec = n_exec;
  p.H = ctx->H;
  p.rec_bytes = ctx->rec_bytes;
  p.raw = raw_maps;
  p.warp_events = warp_events_out;
  p.prev_scratch = d_prev;
  p.prev_stride = stride;
  p.exec_list = exec_list;
  const size_t wsmem = (size_t)kPool * kTabBytes;
  // counters in shared memory either way: packed 16-bit pairs when the device half fits, else the
  // hashed dirty-slot table (both 64 KB at most)
  const int mode = ctx->H <= kSmemSlots ? kCntPacked : kCntHashed;
  const size_t smem = wsmem + counters_smem(mode, ctx->H);
  if (mode == kCntPacked) {
    e = cudaFuncSetAttribute(hfz_k_edge_record<kCntPacked>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) hfz_k_edge_record<kCntPacked><<<grid, kEdgeWarps * 32, smem, ctx->stream>>>(p);
  } else {
    e = cudaFuncSetAttribute(hfz_k_edge_record<kCntHashed>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) hfz_k_edge_record<kCntHashed><<<grid, kEdgeWarps * 32, smem, ctx->stream>>>(p);
  }
  ++ctx->launches;
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return hfz_cuda_fail(e, "hfz_edge_record_batch");
  return HFZ_OK;
}

// grow-only device buffer of the context
template <class T>
static bool edge_grow(T** buf, uint64_t* cap, uint64_t want) {
  if (*cap >= want) return true;
  cudaFree(*buf);
  *buf = nullptr;
  *cap = 0;
  const uint64_t n = want + want / 4 + 64;
  if (cudaMalloc(buf, (size_t)n * sizeof(T)) != cudaSuccess) {
    hfz_set_error("hfz_edge_record_batch: scratch allocation failed (%llu bytes)", (unsigned long long)(n * sizeof(T)));
    return false;
  }
  *cap = n;
  return true;
}

// lists: entries_out != NULL -> also (or, with raw_maps == NULL, only) the touched-slot list of every exec
static int edge_record_impl(hfz_ctx* ctx, const uint64_t* launch_off, const uint32_t* dims,
                            const uint64_t* thread_off, const uint64_t* ev_off, const uint32_t* sites, uint64_t n_exec,
                            uint64_t n_launch, uint8_t* raw_maps, uint64_t* warp_events_out, uint32_t* entries_out,
                            uint32_t entry_cap, uint32_t* n_slots_out) {
  const bool lists = entries_out != nullptr;
  if (!ctx || (n_exec && (!launch_off || (!raw_maps && !lists))) ||
      (n_launch && (!dims || !thread_off || !ev_off)) || (lists && (!n_slots_out || entry_cap == 0))) {
    hfz_set_error("hfz_edge_record_batch: null argument");
    return HFZ_EINVAL;
  }
  if (n_exec == 0) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  if (lists) {
    if (!ctx->edge_flat) {
      hfz_set_error("hfz_edge_record_batch_lists: needs the flat path (option edge_flat = 1)");
      return HFZ_EINVAL;
    }
    // every list starts all-zero ({0, 0} pairs are padding: count 0 = unvisited) and not listed
    HFZ_CUDA(cudaMemsetAsync(entries_out, 0, (size_t)n_exec * entry_cap * 8, ctx->stream));
    HFZ_CUDA(cudaMemsetAsync(n_slots_out, 0xff, (size_t)n_exec * 4, ctx->stream));
  }
  if (n_exec >= (1ull << 32) || n_launch >= (1ull << 32)) {
    hfz_set_error("hfz_edge_record_batch: more than 2^32 - 1 execs or launches in one call");
    return HFZ_EINVAL;
  }
  if (!ctx->edge_flat) {  // everything through the per-exec kernel (one 8-byte D2H read sizes its prev table)
    unsigned long long mx = 0;
    HFZ_CUDA(cudaMemsetAsync(ctx->d_small, 0, sizeof(unsigned long long), ctx->stream));
    if (n_launch) {
      hfz_k_edge_max_threads<<<64, 256, 0, ctx->stream>>>(dims, n_launch, ctx->d_small);
      ++ctx->launches;
      HFZ_CUDA(cudaGetLastError());
    }
    HFZ_CUDA(cudaMemcpyAsync(&mx, ctx->d_small, sizeof(mx), cudaMemcpyDeviceToHost, ctx->stream));
    HFZ_CUDA(cudaStreamSynchronize(ctx->stream));
    return edge_record_per_exec(ctx, launch_off, dims, thread_off, ev_off, sites, n_exec, nullptr, mx, raw_maps,
                                warp_events_out);
  }

  // ---- flat path: prep (eligibility, flat queue) -> per chunk of execs: decide, count
  if (!edge_grow(&ctx->fl_nsw, &ctx->fl_nsw_cap, n_launch + 1) || !edge_grow(&ctx->fl_sw_off, &ctx->fl_sw_off_cap, n_launch + 1) ||
      !edge_grow(&ctx->fl_l_exec, &ctx->fl_l_exec_cap, n_launch + 1) || !edge_grow(&ctx->fl_elig, &ctx->fl_elig_cap, n_exec) ||
      !edge_grow(&ctx->fl_exec_ev0, &ctx->fl_exec_ev0_cap, n_exec + 1) ||
      !edge_grow(&ctx->fl_exec_sw0, &ctx->fl_exec_sw0_cap, n_exec + 1) || !edge_grow(&ctx->fl_inelig, &ctx->fl_inelig_cap, n_exec))
    return HFZ_ENOMEM;
  FlatParams p;
  memset(&p, 0, sizeof(p));
  p.launch_off = launch_off;
  p.dims = dims;
  p.thread_off = thread_off;
  p.ev_off = ev_off;
  p.sites = sites;
  p.n_exec = n_exec;
  p.n_launch = n_launch;
  p.H = ctx->H;
  p.rec_bytes = ctx->rec_bytes;
  p.raw = raw_maps;
  p.warp_events = warp_events_out;
  p.nsw = ctx->fl_nsw;
  p.sw_off = ctx->fl_sw_off;
  p.l_exec = ctx->fl_l_exec;
  p.elig = ctx->fl_elig;
  p.exec_ev0 = ctx->fl_exec_ev0;
  p.exec_sw0 = ctx->fl_exec_sw0;
  p.inelig = ctx->fl_inelig;
  p.small = ctx->d_small;
  HFZ_CUDA(cudaMemsetAsync(ctx->d_small, 0, 8 * sizeof(unsigned long long), ctx->stream));
  {
    const uint64_t blocks = (n_exec + 1 + 255) / 256;
    hfz_k_edge_prep<<<(uint32_t)(blocks < 1024 ? blocks : 1024), 256, 0, ctx->stream>>>(p);
    hfz_k_edge_scan<<<1, 1024, 0, ctx->stream>>>(p);
    ctx->launches += 2;
    HFZ_CUDA(cudaGetLastError());
  }
  unsigned long long h_small[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  std::vector<uint64_t> h_ev0, h_sw0;
  try {
    h_ev0.resize(n_exec + 1);
    h_sw0.resize(n_exec + 1);
  } catch (...) {
    hfz_set_error("hfz_edge_record_batch: host allocation failed");
    return HFZ_ENOMEM;
  }
  HFZ_CUDA(cudaMemcpyAsync(h_small, ctx->d_small, sizeof(h_small), cudaMemcpyDeviceToHost, ctx->stream));
  HFZ_CUDA(cudaMemcpyAsync(h_ev0.data(), ctx->fl_exec_ev0, (n_exec + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  HFZ_CUDA(cudaMemcpyAsync(h_sw0.data(), ctx->fl_exec_sw0, (n_exec + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  HFZ_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_small[7]) {
    hfz_set_error("hfz_edge_record_batch: launch_off is not a non-decreasing sequence within [0, n_launch]");
    return HFZ_EINVAL;
  }
  const uint64_t n_inelig = h_small[0];
  if (n_inelig && raw_maps) {  // execs whose launches differ in geometry (prev is launch-ordered there)
    const int rc = edge_record_per_exec(ctx, launch_off, dims, thread_off, ev_off, sites, n_inelig, ctx->fl_inelig,
                                        h_small[1], raw_maps, warp_events_out);
    if (rc != HFZ_OK) return rc;
  }
  // small[3] holds the max of ~nsw, i.e. ~min
  p.uni_nsw = (n_inelig == 0 && h_small[4] > 0 && ~h_small[3] == h_small[4]) ? (uint32_t)h_small[4] : 0u;
  p.l_lo = 0;
  p.l_hi = n_launch;
  const uint64_t cap_events = (uint64_t)ctx->edge_scratch_mb << 18;  // u32 entries
  const uint64_t cap_items = 1ull << 24;
  const size_t tab_smem = (size_t)kFlatWarps * kTabBytes;
  const uint32_t cslots = ctx->H < kCountSlots ? ctx->H : kCountSlots;
  HFZ_CUDA(cudaFuncSetAttribute(hfz_k_edge_divergent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tab_smem));
  HFZ_CUDA(cudaFuncSetAttribute(hfz_k_edge_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(cslots * 4)));
  for (uint64_t e_lo = 0; e_lo < n_exec;) {
    uint64_t e_hi = e_lo + 1;
    while (e_hi < n_exec && h_ev0[e_hi + 1] - h_ev0[e_lo] <= cap_events && h_sw0[e_hi + 1] - h_sw0[e_lo] <= cap_items) ++e_hi;
    const uint64_t n_ev = h_ev0[e_hi] - h_ev0[e_lo], n_items = h_sw0[e_hi] - h_sw0[e_lo];
    if (!edge_grow(&ctx->fl_scratch, &ctx->fl_scratch_cap, n_ev + 1) ||
        !edge_grow(&ctx->fl_rec_first, &ctx->fl_rec_first_cap, n_items + 1) ||
        !edge_grow(&ctx->fl_rec_cnt, &ctx->fl_rec_cnt_cap, n_items + 1) ||
        !edge_grow(&ctx->fl_div, &ctx->fl_div_cap, n_items + 1) ||
        !edge_grow(&ctx->fl_lines, &ctx->fl_lines_cap, (n_items + 32) * 32))
      return HFZ_ENOMEM;
    p.e_lo = e_lo;
    p.e_hi = e_hi;
    p.q_lo = h_sw0[e_lo];
    p.q_hi = h_sw0[e_hi];
    p.ev_lo = h_ev0[e_lo];
    p.scratch = ctx->fl_scratch;
    p.rec_first = ctx->fl_rec_first;
    p.rec_cnt = ctx->fl_rec_cnt;
    p.div_list = ctx->fl_div;
    p.lines = ctx->fl_lines;
    p.list_out = reinterpret_cast<uint2*>(entries_out);
    p.list_cap = entry_cap;
    p.list_n = n_slots_out;
    if (n_items) {
      HFZ_CUDA(cudaMemsetAsync(ctx->d_small + 2, 0, 5 * sizeof(unsigned long long), ctx->stream));  // pop counters, divergent count
      const uint64_t want = (n_items + kPop * kClassifyWarps - 1) / (kPop * kClassifyWarps);
      const uint64_t full = (uint64_t)ctx->num_sms * 2;
      hfz_k_edge_classify<<<(uint32_t)(want < full ? want : full), kClassifyWarps * 32, 0, ctx->stream>>>(p);
      const uint64_t wantd = (n_items + kFlatWarps - 1) / kFlatWarps;  // (the divergent count is known on the device only)
      hfz_k_edge_divergent<<<(uint32_t)(wantd < (uint64_t)ctx->num_sms ? wantd : (uint64_t)ctx->num_sms), kFlatWarps * 32, tab_smem,
                             ctx->stream>>>(p);
      ctx->launches += 2;
    }
    const uint64_t ne = e_hi - e_lo;
    const uint64_t cgrid = (uint64_t)ctx->num_sms * 3;
    hfz_k_edge_count<<<(uint32_t)(ne < cgrid ? ne : cgrid), kCountWarps * 32, cslots * 4, ctx->stream>>>(p);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
    e_lo = e_hi;
  }
  return HFZ_OK;
}

extern "C" int hfz_edge_record_batch(hfz_ctx* ctx, const uint64_t* launch_off, const uint32_t* dims,
                                     const uint64_t* thread_off, const uint64_t* ev_off,
                                     const uint32_t* sites, uint64_t n_exec, uint64_t n_launch,
                                     uint8_t* raw_maps, uint64_t* warp_events_out) {
  if (n_exec && !raw_maps) {
    hfz_set_error("hfz_edge_record_batch: null argument");
    return HFZ_EINVAL;
  }
  return edge_record_impl(ctx, launch_off, dims, thread_off, ev_off, sites, n_exec, n_launch, raw_maps, warp_events_out,
                          nullptr, 0, nullptr);
}

extern "C" int hfz_edge_record_batch_lists(hfz_ctx* ctx, const uint64_t* launch_off, const uint32_t* dims,
                                           const uint64_t* thread_off, const uint64_t* ev_off,
                                           const uint32_t* sites, uint64_t n_exec, uint64_t n_launch,
                                           uint8_t* raw_maps, uint64_t* warp_events_out, uint32_t* entries_out,
                                           uint32_t entry_cap, uint32_t* n_slots_out) {
  if (n_exec && (!entries_out || !n_slots_out || entry_cap == 0)) {
    hfz_set_error("hfz_edge_record_batch_lists: null argument");
    return HFZ_EINVAL;
  }
  return edge_record_impl(ctx, launch_off, dims, thread_off, ev_off, sites, n_exec, n_launch, raw_maps, warp_events_out,
                          entries_out, entry_cap, n_slots_out);
}

extern "C" int hfz_host_edge_record_batch(hfz_ctx* ctx, const uint64_t* site_off,
                                          const uint16_t* sites, uint64_t n_exec, uint8_t* raw_maps) {
  if (!ctx || (n_exec && (!site_off || !raw_maps))) {
    hfz_set_error("hfz_host_edge_record_batch: null argument");
    return HFZ_EINVAL;
  }
  if (n_exec == 0) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  const uint32_t nslots = ctx->H < 65536u ? ctx->H : 65536u;
  const bool in_smem = (size_t)nslots * 4 <= (size_t)ctx->max_smem_optin;
  uint32_t grid = (uint32_t)(n_exec < (uint64_t)ctx->num_sms * 2 ? n_exec : (uint64_t)ctx->num_sms * 2);
  uint32_t* d_scratch = nullptr;
  cudaError_t e = cudaSuccess;
  size_t smem = 0;
  if (in_smem) {
    smem = (size_t)nslots * 4;
    e = cudaFuncSetAttribute(hfz_k_host_edge_record, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  } else {
    e = cudaMalloc(&d_scratch, (size_t)grid * nslots * 4);
  }
  if (e == cudaSuccess) {
    hfz_k_host_edge_record<<<grid, 256, smem, ctx->stream>>>(site_off, sites, n_exec, ctx->H,
                                                            ctx->rec_bytes, raw_maps, d_scratch);
    ++ctx->launches;
    e = cudaGetLastError();
  }
  if (d_scratch) {
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d_scratch);
  }
  if (e != cudaSuccess) return hfz_cuda_fail(e, "hfz_host_edge_record_batch");
  return HFZ_OK;
}
