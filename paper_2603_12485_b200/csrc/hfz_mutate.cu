// hfz_mutate.cu -- K3 batched mutators: havoc, splice, deterministic stage.
//
// Reference semantics (paths under /root/reference/proj):
//   havoc_mutant            src/engine.cpp:119-193   (tables :27-38, write_le :46-49)
//   splice_mutant           src/engine.cpp:195-204
//   for_each_deterministic  src/engine.cpp:53-105
//   Rng                     include/hetfuzz/rng.hpp:11-46
//
// Havoc runs as PLAN then APPLY.  Every Rng bound of the edit loop depends on the current LENGTH
// alone, never on the bytes, so the whole draw sequence of a slot can be walked without touching
// its data:
//   hfz_k_havoc_plan_ops   one THREAD per slot: scalar splitmix64, branch-light walk of the 1..64
//                          stacked edits; writes the slot's edit list (one 64-bit word per edit),
//                          its final length, end Rng state and draw count;
//   hfz_k_havoc_apply      one WARP per slot (dynamic hand-out): reads the edit list with one
//                          coalesced load, applies it -- single-byte edits by lane 0, block moves
//                          (erase / insert) by the whole warp, 16 bytes per lane and step -- on a
//                          working buffer in shared memory when the slot's maximum output fits
//                          (inputs up to ~5 KB: BASELINE.json configs[3]) and directly in the
//                          slot's output region in global memory otherwise (up to 1 MiB).
// (One warp per slot doing both, with a warp-uniform Rng, spent 3/4 of its instructions on the
// scalar control flow that 32 lanes executed redundantly: 8.8 k warp-instructions per mutant.)
#include <string.h>

#include <vector>

#include "hfz_common.cuh"

namespace {

constexpr uint32_t kMaxInput = HFZ_MAX_INPUT_BYTES;
constexpr int kHavocWarps = 8;
constexpr uint64_t kHavocChunk = 1ull << 17;  // slots planned and applied per launch pair
constexpr uint32_t kSmemCap = 6128;  // working buffer bytes per warp (>= 4096 + 1024); + 16 bytes of padding = 6 KB per warp, 48 KB static per CTA

__constant__ int16_t c_interesting16[10] = {-32768, -129, 128, 255, 256, 512, 1000, 1024, 4096, 32767};
__constant__ int32_t c_interesting32[8] = {(-2147483647 - 1), -100663046, -32769, 32768,
                                           65535,             65536,      100663045, 2147483647};

// The slot's splitmix64 stream, warp-uniform.  The state after k draws is seed + k * gamma
// (rng.hpp:15-21), so the warp computes the next 32 outputs at once -- lane i mixes
// s + (i + 1) * gamma -- and hands them out one per draw by shuffle: a draw costs two shuffles
// instead of two 64-bit multiplies on every lane.  next() must be called by the whole warp.
struct WarpRng {
  uint64_t s;      // reference state: seed + draws * gamma
  uint32_t draws;
  uint64_t buf;    // this lane's output of the current batch
  uint32_t pos;    // next unread output of the batch; 32 = none left
  uint32_t lane;
  __device__ __forceinline__ void init(uint64_t state, int lane_) {
    s = state;
    draws = 0;
    pos = 32;
    lane = (uint32_t)lane_;
    buf = 0;
  }
  __device__ __forceinline__ uint64_t next() {
    if (pos == 32) {
      buf = hfz_sm64_mix(s + (uint64_t)(lane + 1) * HFZ_GAMMA);
      pos = 0;
    }
    const uint64_t r = __shfl_sync(0xffffffffu, buf, (int)pos);
    ++pos;
    s += HFZ_GAMMA;
    ++draws;
    return r;
  }
  // below(n): n <= 1 returns 0 WITHOUT drawing (rng.hpp:24-28); (u128(next()) * n) >> 64 otherwise.
  // Every bound on this path fits 32 bits (the largest is 8 x kMaxInputBytes = 2^23 bit positions), so
  // the 64 x 64 -> high-64 product is two 32 x 32 -> 64 multiplies: hi32(r) * n + (lo32(r) * n >> 32).
  __device__ __forceinline__ uint32_t below(uint32_t n) {
    if (n <= 1) return 0;
    const uint64_t r = next();
    const uint64_t t = (uint64_t)(uint32_t)(r >> 32) * n + (((uint64_t)(uint32_t)r * n) >> 32);
    return (uint32_t)(t >> 32);
  }
  // the per-edit interface of the planner (LaneRng below draws ahead here; this stream is warp-uniform already)
  __device__ __forceinline__ void edit_begin() {}
  __device__ __forceinline__ uint32_t take(uint32_t n) { return below(n); }
  __device__ __forceinline__ void edit_end() {}
};

// non-overlapping copy by one warp; loads are issued in batches of 8 per lane so that a
// misaligned (byte-granular) copy from global memory still has 8 requests in flight per lane
__device__ __forceinline__ void warp_copy(uint8_t* dst, const uint8_t* src, uint64_t n, int lane) {
  if ((((uintptr_t)dst ^ (uintptr_t)src) & 15) == 0 && n >= 64) {
    uint64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
    if (head > n) head = n;
    for (uint64_t i = lane; i < head; i += 32) dst[i] = src[i];
    const uint64_t body = (n - head) / 16;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    for (uint64_t b0 = 0; b0 < body; b0 += 32 * 4) {
      uint4 t[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t i = b0 + k * 32 + lane;
        if (i < body) t[k] = s4[i];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t i = b0 + k * 32 + lane;
        if (i < body) d4[i] = t[k];
      }
    }
    for (uint64_t i = head + body * 16 + lane; i < n; i += 32) dst[i] = src[i];
  } else if ((((uintptr_t)dst ^ (uintptr_t)src) & 3) == 0 && n >= 16) {
    uint64_t head = (4 - ((uintptr_t)dst & 3)) & 3;
    if (head > n) head = n;
    if ((uint64_t)lane < head) dst[lane] = src[lane];
    const uint64_t body = (n - head) / 4;
    const uint32_t* s1 = reinterpret_cast<const uint32_t*>(src + head);
    uint32_t* d1 = reinterpret_cast<uint32_t*>(dst + head);
    for (uint64_t b0 = 0; b0 < body; b0 += 32 * 8) {
      uint32_t t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t i = b0 + k * 32 + lane;
        if (i < body) t[k] = s1[i];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t i = b0 + k * 32 + lane;
        if (i < body) d1[i] = t[k];
      }
    }
    for (uint64_t i = head + body * 4 + lane; i < n; i += 32) dst[i] = src[i];
  } else {
    for (uint64_t b0 = 0; b0 < n; b0 += 32 * 8) {
      uint8_t t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t i = b0 + k * 32 + lane;
        if (i < n) t[k] = src[i];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t i = b0 + k * 32 + lane;
        if (i < n) dst[i] = t[k];
      }
    }
  }
}

// overlapping move towards lower addresses: buf[dst + i] = buf[src + i], i ascending (dst < src)
__device__ __forceinline__ void warp_move_down(uint8_t* buf, uint64_t dst, uint64_t src, uint64_t n,
                                               int lane) {
  for (uint64_t base = 0; base < n; base += 128) {
    uint8_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = base + k * 32 + lane;
      v[k] = i < n ? buf[src + i] : 0;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = base + k * 32 + lane;
      if (i < n) buf[dst + i] = v[k];
    }
    __syncwarp();
  }
}

// overlapping move towards higher addresses: buf[dst + i] = buf[src + i], i descending (dst > src)
__device__ __forceinline__ void warp_move_up(uint8_t* buf, uint64_t dst, uint64_t src, uint64_t n,
                                             int lane) {
  uint64_t done = 0;
  while (done < n) {
    const uint64_t chunk = n - done < 128 ? n - done : 128;
    const uint64_t base = n - done - chunk;  // process the highest remaining chunk first
    uint8_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = k * 32 + lane;
      v[k] = i < chunk ? buf[src + base + i] : 0;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = k * 32 + lane;
      if (i < chunk) buf[dst + base + i] = v[k];
    }
    __syncwarp();
    done += chunk;
  }
}

// The same two overlapping moves for a working buffer in SHARED memory, 16 bytes per lane and step
// instead of 4 single bytes: destination block k (16-byte aligned) is assembled from five aligned
// source words with funnel shifts -- the byte distance between source and destination is the same
// for the whole move, so one shift serves every word -- and stored with one 128-bit store.  The
// partial block at the START of the range keeps the bytes below it.  The block at the END is
// written whole: both moves of the edit loop end exactly at the buffer's new length (erase: len -
// count, insert: the new length), so the bytes behind the range are dead.  buf must be 16-byte
// aligned and padded to a whole block beyond the largest length.
// one step: blocks [k0, k0 + 32) of the destination (block k = bytes [16k, 16k + 16)); delta = src - dst (signed);
// the destination range starts at dlo
__device__ __forceinline__ void move_blocks(uint8_t* buf, uint32_t k0, uint32_t k_end, int32_t delta, uint32_t dlo,
                                            int lane) {
  const uint32_t k = k0 + lane;
  const bool on = k < k_end;
  uint4 out = make_uint4(0, 0, 0, 0);
  if (on) {
    const int32_t sb = (int32_t)(k * 16) + delta;  // source byte of the block's first byte (< 0 only for bytes outside the range)
    const int32_t sw = sb >> 2;                    // aligned source word (floor)
    const uint32_t sh = (uint32_t)(sb & 3) * 8;
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(buf);
    uint32_t w[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) w[j] = sw + j >= 0 ? w32[sw + j] : 0u;
    out.x = __funnelshift_r(w[0], w[1], sh);
    out.y = __funnelshift_r(w[1], w[2], sh);
    out.z = __funnelshift_r(w[2], w[3], sh);
    out.w = __funnelshift_r(w[3], w[4], sh);
    const uint32_t b0 = k * 16;
    if (b0 < dlo) {  // the range's first block: keep the bytes below dlo (at most one lane of one step gets here)
      const uint32_t lo8 = (dlo - b0) * 8;  // 8 .. 120 bits to keep
      const uint4 old = reinterpret_cast<const uint4*>(buf)[k];
      // word j keeps its low clamp(lo8 - 32 j, 0, 32) bits: a clamping funnel shift of (ones : zeros)
      const uint32_t m0 = __funnelshift_lc(0u, ~0u, lo8 < 32u ? lo8 : 32u);
      const uint32_t m1 = lo8 <= 32u ? ~0u : __funnelshift_lc(0u, ~0u, lo8 - 32u < 32u ? lo8 - 32u : 32u);
      const uint32_t m2 = lo8 <= 64u ? ~0u : __funnelshift_lc(0u, ~0u, lo8 - 64u < 32u ? lo8 - 64u : 32u);
      const uint32_t m3 = lo8 <= 96u ? ~0u : __funnelshift_lc(0u, ~0u, lo8 - 96u);
      out.x = (out.x & m0) | (old.x & ~m0);
      out.y = (out.y & m1) | (old.y & ~m1);
      out.z = (out.z & m2) | (old.z & ~m2);
      out.w = (out.w & m3) | (old.w & ~m3);
    }
  }
  __syncwarp();  // every block of this step is read before any is written
  if (on) reinterpret_cast<uint4*>(buf)[k] = out;
  __syncwarp();
}
// buf[dst + i] = buf[src + i], i ascending (dst < src)
__device__ __forceinline__ void smem_move_down(uint8_t* buf, uint32_t dst, uint32_t src, uint32_t n, int lane) {
  if (n == 0) return;
  const uint32_t k_first = dst / 16, k_end = (dst + n + 15) / 16;
  for (uint32_t k0 = k_first; k0 < k_end; k0 += 32) move_blocks(buf, k0, k_end, (int32_t)(src - dst), dst, lane);
}
// buf[dst + i] = buf[src + i], i descending (dst > src)
__device__ __forceinline__ void smem_move_up(uint8_t* buf, uint32_t dst, uint32_t src, uint32_t n, int lane) {
  if (n == 0) return;
  const uint32_t k_first = dst / 16, k_end = (dst + n + 15) / 16;
  uint32_t k0 = k_first + ((k_end - k_first - 1) / 32) * 32;  // the highest step first
  for (;;) {
    move_blocks(buf, k0, k_end, -(int32_t)(dst - src), dst, lane);
    if (k0 == k_first) break;
    k0 -= 32;
  }
}

// global (any alignment) -> shared (16-byte aligned dst), 16 bytes per lane: two aligned 128-bit loads
// (the second one is the next lane's first: an L1 hit) + one funnel shift per word + one 128-bit store.
// Reads only 16-byte blocks that hold at least one byte of [src, src + n): no slack needed around the input.
__device__ __forceinline__ void copy_in_smem(uint8_t* dst, const uint8_t* src, uint32_t n, int lane) {
  const uint32_t a = (uint32_t)((uintptr_t)src & 15);
  const uint4* s4 = reinterpret_cast<const uint4*>(src - a);
  const uint32_t sh = (a & 3) * 8, wsel = a >> 2;
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  const uint32_t blocks = (n + 15) / 16;
  const uint32_t src_blocks = (a + n + 15) / 16;  // aligned source blocks that hold input bytes
  for (uint32_t b0 = 0; b0 < blocks; b0 += 32 * 2) {
    uint4 lo[2], hi[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t b = b0 + k * 32 + lane;
      lo[k] = b < blocks ? __ldg(s4 + b) : make_uint4(0, 0, 0, 0);
      hi[k] = (b < blocks && b + 1 < src_blocks) ? __ldg(s4 + b + 1) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t b = b0 + k * 32 + lane;
      if (b >= blocks) continue;
      const uint32_t w[8] = {lo[k].x, lo[k].y, lo[k].z, lo[k].w, hi[k].x, hi[k].y, hi[k].z, hi[k].w};
      uint32_t v[5];
#pragma unroll
      for (int j = 0; j < 5; ++j)  // words wsel .. wsel + 4 of the 8: a 4-way select, wsel is warp-uniform
        v[j] = wsel == 0 ? w[j] : (wsel == 1 ? w[j + 1] : (wsel == 2 ? w[j + 2] : w[j + 3]));
      d4[b] = make_uint4(__funnelshift_r(v[0], v[1], sh), __funnelshift_r(v[1], v[2], sh),
                         __funnelshift_r(v[2], v[3], sh), __funnelshift_r(v[3], v[4], sh));
    }
  }
}
// shared (16-byte aligned src) -> global (any alignment): byte stores up to the first 16-byte boundary of dst,
// 128-bit stores for the body (five aligned shared words + funnel shifts per block), byte stores for the tail
__device__ __forceinline__ void copy_out_smem(uint8_t* dst, const uint8_t* src, uint32_t n, int lane) {
  uint32_t head = (16u - (uint32_t)((uintptr_t)dst & 15)) & 15u;
  if (head > n) head = n;
  if ((uint32_t)lane < head) dst[lane] = src[lane];
  const uint32_t blocks = (n - head) / 16;
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src) + (head >> 2);
  const uint32_t sh = (head & 3) * 8;
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  for (uint32_t b = lane; b < blocks; b += 32) {
    const uint32_t* w = s32 + b * 4;
    const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4];  // w[4]: inside the padded buffer
    d4[b] = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                       __funnelshift_r(w3, w4, sh));
  }
  const uint32_t done = head + blocks * 16;
  if (done + lane < n) dst[done + lane] = src[done + lane];
}

__device__ __forceinline__ uint64_t havoc_cap(uint64_t len) {
  const uint64_t m = len + 64 * 16;
  return m > kMaxInput ? kMaxInput : m;
}

// ---- edit lists.  One 64-bit word per edit: kind (4 bits) | A (23) | B (21) | C (16).
//   0 flip bit        A = bit position (MSB-first inside the byte)
//   1 set byte        A = index, C = value
//   2 byte +/- delta  A = index, B = delta, C = 1 add / 0 subtract
//   3 interesting 16  A = offset, C = table index
//   4 interesting 32  A = offset, C = table index
//   5 delete block    A = offset, B = count
//   6 duplicate block A = source, B = destination, C = count
//   7 constant fill   A = offset, B = count, C = value
//   8 swap bytes      A = i, B = k
//   9 append to an EMPTY input: bits 4-7 = count (1..8), bits 8-63 = bytes 0..6;  10: bits 8-15 = byte 7
// Word 0 of a slot's list is the number of edit words that follow (<= 65).
constexpr uint32_t kOpWords = 66;
__device__ __forceinline__ uint64_t op_word(uint32_t kind, uint32_t a, uint32_t b, uint32_t c) {
  return (uint64_t)kind | ((uint64_t)a << 4) | ((uint64_t)b << 27) | ((uint64_t)c << 48);
}

// scalar splitmix64 of one slot (rng.hpp:15-28).  The state after k draws is seed + k * gamma, so the
// raw outputs of the next draws do not depend on the bounds they will be reduced by: edit_begin()
// mixes the next four at once (independent multiply chains the scheduler overlaps) and take() hands
// them out in order; only "was a draw consumed" (bound > 1) stays on the dependent path.
struct LaneRng {
  uint64_t s;
  uint32_t draws;
  uint64_t r0, r1, r2, r3;
  uint32_t used;
  __device__ __forceinline__ void init(uint64_t state, int) {
    s = state;
    draws = 0;
  }
  static __device__ __forceinline__ uint32_t reduce(uint64_t r, uint32_t n) {  // (u128(r) * n) >> 64 for n < 2^32
    const uint64_t t = (uint64_t)(uint32_t)(r >> 32) * n + (((uint64_t)(uint32_t)r * n) >> 32);
    return (uint32_t)(t >> 32);
  }
  __device__ __forceinline__ uint32_t below(uint32_t n) {
    if (n <= 1) return 0;
    s += HFZ_GAMMA;
    ++draws;
    return reduce(hfz_sm64_mix(s), n);
  }
  __device__ __forceinline__ void edit_begin() {
    r0 = hfz_sm64_mix(s + HFZ_GAMMA);
    r1 = hfz_sm64_mix(s + 2 * HFZ_GAMMA);
    r2 = hfz_sm64_mix(s + 3 * HFZ_GAMMA);
    r3 = hfz_sm64_mix(s + 4 * HFZ_GAMMA);
    used = 0;
  }
  __device__ __forceinline__ uint32_t take(uint32_t n) {  // at most four per edit
    const uint64_t r = used == 0 ? r0 : (used == 1 ? r1 : (used == 2 ? r2 : r3));
    const bool drawn = n > 1;
    used += drawn;
    return drawn ? reduce(r, n) : 0u;
  }
  __device__ __forceinline__ void edit_end() {
    s += (uint64_t)used * HFZ_GAMMA;
    draws += used;
  }
};

// The draw sequence of the stacked-havoc edit loop of one slot (src/engine.cpp:120-191) and, with
// EMIT, its edit list.  Every edit kind is "up to three draws whose bounds depend on the kind, the
// current length and the earlier draws" -- a bound of 0 or 1 draws nothing (rng.hpp:24-28) -- so
// the walk is one straight-line body per edit with selects instead of a nine-way branch: 32
// slots of a warp stay converged whatever kinds they drew.  Returns the final length.
template <class R, bool EMIT>
__device__ __forceinline__ uint32_t havoc_plan(R& rng, uint32_t len, uint64_t* __restrict__ ops) {
  const uint32_t n_edits = 1 + rng.below(64);
  uint32_t n_words = 0;
  for (uint32_t e = 0; e < n_edits; ++e) {
    if (len == 0) {  // engine.cpp:124-129: only an empty INPUT gets here (a delete leaves >= 1 byte)
      const uint32_t cnt = 1 + rng.below(8);
      uint64_t w9 = 9u | ((uint64_t)cnt << 4), w10 = 10u;
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint64_t b = rng.below(256);
        if (i < 7) w9 |= b << (8 + 8 * i);
        else w10 |= b << 8;
      }
      if (EMIT) {
        ops[1 + n_words++] = w9;
        if (cnt == 8) ops[1 + n_words++] = w10;
      }
      len = cnt;
      continue;
    }
    rng.edit_begin();
    const uint32_t kind = rng.take(9);
    // kinds 3 / 4 / 5 are no-ops without draws below 2 / 4 / 2 bytes
    const bool skip = (kind == 3 && len < 2) || (kind == 4 && len < 4) || (kind == 5 && len < 2);
    uint32_t b1 = len;                       // 5, 6, 7, 8: a position
    b1 = kind == 0 ? len * 8 : b1;           // bit position (len <= 2^20)
    b1 = kind == 1 ? 256u : b1;              // the VALUE is drawn before the index (C++17 sequencing of '=')
    b1 = kind == 2 ? 35u : b1;
    b1 = kind == 3 ? len - 1 : b1;
    b1 = kind == 4 ? len - 3 : b1;
    b1 = skip ? 0u : b1;
    const uint32_t r1 = rng.take(b1);
    const uint32_t rest = len - r1;          // kinds 5, 6, 7: bytes from the drawn position to the end
    const uint32_t quarter = len / 4 ? len / 4 : 1u;
    uint32_t b2 = len;                       // 1, 2, 8: an index
    b2 = kind == 0 ? 0u : b2;
    b2 = kind == 3 ? 10u : b2;
    b2 = kind == 4 ? 8u : b2;
    b2 = kind == 5 ? (rest < quarter ? rest : quarter) : b2;
    b2 = (kind == 6 || kind == 7) ? (rest < 16u ? rest : 16u) : b2;
    b2 = skip ? 0u : b2;
    const uint32_t r2 = rng.take(b2);
    uint32_t b3 = 0;
    b3 = kind == 2 ? 2u : b3;
    b3 = kind == 6 ? len + 1 : b3;
    b3 = kind == 7 ? 256u : b3;
    const uint32_t r3 = rng.take(b3);
    rng.edit_end();
    if (EMIT && !skip) {
      uint32_t a = r1, b = r2, c = r3;
      if (kind == 1) a = r2, b = 0, c = r1;
      if (kind == 2) a = r2, b = 1 + r1, c = r3 < 1;
      if (kind == 3 || kind == 4) b = 0, c = r2;
      if (kind == 5) b = 1 + r2, c = 0;
      if (kind == 6) b = r3, c = 1 + r2;
      if (kind == 7) b = 1 + r2;
      ops[1 + n_words++] = op_word(kind, a, b, c);
    }
    if (kind == 5 && !skip) len -= 1 + r2;
    if (kind == 6) {
      len += 1 + r2;
      if (len > kMaxInput) len = kMaxInput;  // the insert is clamped to 1 MiB (engine.cpp:190)
    }
  }
  if (EMIT) ops[0] = n_words;
  return len;
}

// PLAN: one thread per slot of the chunk.
__global__ void __launch_bounds__(64) hfz_k_havoc_plan_ops(const uint64_t* __restrict__ in_off, uint64_t n,
                                                          uint64_t* __restrict__ state, uint64_t* __restrict__ ops,
                                                          uint64_t* __restrict__ out_len, uint32_t* __restrict__ draws_out,
                                                          unsigned long long* __restrict__ next_slot) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0) *next_slot = 0;  // the apply kernel's hand-out counter
  if (j >= n) return;
  uint64_t len64 = in_off[j + 1] - in_off[j];
  // Inputs longer than kMaxInputBytes are rejected by the host-buffer entry points (hfz.h); a
  // device-buffer caller that passes one anyway gets a memory-safe result: the slot's capacity is
  // hfz_havoc_max_out(len) = 1 MiB, so only the first 1 MiB is mutated.
  if (len64 > kMaxInput) len64 = kMaxInput;
  LaneRng rng;
  rng.init(state[j], 0);
  const uint32_t len = havoc_plan<LaneRng, true>(rng, (uint32_t)len64, ops + j * kOpWords);
  out_len[j] = len;
  state[j] = rng.s;
  if (draws_out) draws_out[j] = rng.draws;
}

// APPLY: one warp per slot.  v = the working buffer (SMEM: shared, 16-byte aligned, padded).
template <bool SMEM>
__device__ __forceinline__ uint32_t havoc_apply(uint8_t* v, uint32_t len, const uint64_t* __restrict__ ops, int lane) {
  // the whole list with one coalesced load: lane l holds words l, 32 + l and (lanes 0, 1) 64 + l
  const uint64_t w_a = ops[lane];
  const uint32_t n_words = (uint32_t)__shfl_sync(0xffffffffu, w_a, 0);
  const uint64_t w_b = 32u + lane <= n_words ? ops[32 + lane] : 0ull;
  const uint64_t w_c = 64u + lane <= n_words ? ops[64 + lane] : 0ull;
  for (uint32_t i = 1; i <= n_words; ++i) {
    // (the word's holder changes every 32 edits: selecting it per edit is cheaper than three copies of the switch)
    const uint64_t held = i < 32 ? w_a : (i < 64 ? w_b : w_c);
    const uint64_t w = __shfl_sync(0xffffffffu, held, (int)(i & 31));
    const uint32_t kind = (uint32_t)w & 15u, a = (uint32_t)(w >> 4) & 0x7fffffu, b = (uint32_t)(w >> 27) & 0x1fffffu,
                   c = (uint32_t)(w >> 48);
    switch (kind) {
      case 0:
        if (lane == 0) v[a / 8] ^= (uint8_t)(0x80u >> (a % 8));
        break;
      case 1:
        if (lane == 0) v[a] = (uint8_t)c;
        break;
      case 2:
        if (lane == 0) v[a] = (uint8_t)(c ? v[a] + b : v[a] - b);
        break;
      case 3: {  // little endian (write_le, engine.cpp:46-49)
        const uint32_t val = (uint16_t)c_interesting16[c];
        if (lane < 2) v[a + lane] = (uint8_t)(val >> (8 * lane));
        break;
      }
      case 4: {
        const uint32_t val = (uint32_t)c_interesting32[c];
        if (lane < 4) v[a + lane] = (uint8_t)(val >> (8 * lane));
        break;
      }
      case 5:
        if (SMEM) smem_move_down(v, a, a + b, len - a - b, lane);
        else warp_move_down(v, a, a + b, len - a - b, lane);
        len -= b;
        break;
      case 6: {  // copy the block first, then insert it (the 1 MiB clamp folded in: bytes past the cap are dropped)
        const uint8_t blk = (uint32_t)lane < c ? v[a + lane] : 0;
        const uint32_t new_len = len + c > kMaxInput ? kMaxInput : len + c;
        __syncwarp();
        if (new_len > b + c) {
          if (SMEM) smem_move_up(v, b + c, b, new_len - b - c, lane);
          else warp_move_up(v, b + c, b, new_len - b - c, lane);
        }
        if ((uint32_t)lane < c && b + lane < new_len) v[b + lane] = blk;
        len = new_len;
        break;
      }
      case 7:
        if ((uint32_t)lane < b) v[a + lane] = (uint8_t)c;
        break;
      case 8:
        if (lane == 0) {
          const uint8_t t = v[a];
          v[a] = v[b];
          v[b] = t;
        }
        break;
      case 9: {
        const uint32_t cnt = (uint32_t)(w >> 4) & 15u;
        if ((uint32_t)lane < cnt && lane < 7) v[lane] = (uint8_t)(w >> (8 + 8 * lane));
        len = cnt;
        break;
      }
      default:  // 10: the eighth appended byte
        if (lane == 0) v[7] = (uint8_t)(w >> 8);
        break;
    }
    __syncwarp();  // edits are ordered; successive ones may be done by different lanes
  }
  return len;
}

__global__ void __launch_bounds__(kHavocWarps * 32, 4) hfz_k_havoc_apply(
    const uint8_t* __restrict__ in_bytes, const uint64_t* __restrict__ in_off, uint64_t n,
    const uint64_t* __restrict__ ops, uint8_t* __restrict__ out_bytes, const uint64_t* __restrict__ out_off,
    unsigned long long* __restrict__ next_slot) {
  __shared__ __align__(16) uint8_t s_buf[kHavocWarps][kSmemCap + 16];  // + 16: the block moves read one block past the data
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // slots are handed out dynamically: a mutant stacks 1..64 edits, so their costs differ widely
  for (;;) {
    unsigned long long jj = 0;
    if (lane == 0) jj = atomicAdd(next_slot, 1ull);
    const uint64_t j = __shfl_sync(0xffffffffu, jj, 0);
    if (j >= n) break;
    const uint64_t i0 = in_off[j];
    uint64_t len64 = in_off[j + 1] - i0;
    if (len64 > kMaxInput) len64 = kMaxInput;
    const uint32_t len = (uint32_t)len64;
    uint8_t* out = out_bytes + out_off[j];
    const uint64_t* my_ops = ops + j * kOpWords;
    if (havoc_cap(len) <= kSmemCap) {
      uint8_t* v = s_buf[warp];
      copy_in_smem(v, in_bytes + i0, len, lane);
      __syncwarp();
      const uint32_t out_n = havoc_apply<true>(v, len, my_ops, lane);
      copy_out_smem(out, v, out_n, lane);
      __syncwarp();  // the buffer is reused for the warp's next slot
    } else {
      warp_copy(out, in_bytes + i0, len, lane);
      __syncwarp();
      havoc_apply<false>(out, len, my_ops, lane);
    }
  }
}

// Serial-stream plan: ONE Rng threaded through n mutants in slot order, as Campaign::fuzz_entry
// does (src/engine.cpp:561-562).  A dry run per slot yields the state each slot starts from.
__global__ void hfz_k_havoc_plan(const uint64_t* __restrict__ in_off, uint64_t n,
                                 uint64_t* __restrict__ stream_state, uint64_t* __restrict__ slot_states) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;  // one warp: the draws are handed out by shuffle
  const int lane = threadIdx.x;
  WarpRng rng;
  rng.init(*stream_state, lane);
  __syncwarp();
  for (uint64_t j = 0; j < n; ++j) {
    if (lane == 0) slot_states[j] = rng.s;
    uint64_t len = in_off[j + 1] - in_off[j];
    if (len > kMaxInput) len = kMaxInput;
    havoc_plan<WarpRng, false>(rng, (uint32_t)len, nullptr);
  }
  __syncwarp();
  if (lane == 0) *stream_state = rng.s;
}

__global__ void __launch_bounds__(256) hfz_k_splice(
    const uint8_t* __restrict__ in_bytes, const uint64_t* __restrict__ in_off,
    const uint32_t* __restrict__ a_idx, const uint32_t* __restrict__ b_idx, uint64_t n,
    uint64_t* __restrict__ state, uint8_t* __restrict__ out_bytes,
    const uint64_t* __restrict__ out_off, uint64_t* __restrict__ out_len) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t j = warp; j < n; j += nw) {
    const uint64_t a0 = in_off[a_idx[j]], alen = in_off[a_idx[j] + 1] - a0;
    const uint64_t b0 = in_off[b_idx[j]], blen = in_off[b_idx[j] + 1] - b0;
    WarpRng rng;
    rng.init(state[j], lane);
    const uint64_t ca = rng.below(alen + 1);
    const uint64_t cb = rng.below(blen + 1);  // (draws use the true lengths; the copies below are clamped to 1 MiB)
    const uint64_t total = ca + (blen - cb);
    const uint64_t keep = total > kMaxInput ? kMaxInput : total;
    const uint64_t head = ca < keep ? ca : keep;
    uint8_t* out = out_bytes + out_off[j];
    warp_copy(out, in_bytes + a0, head, lane);
    warp_copy(out + head, in_bytes + b0 + cb, keep - head, lane);
    if (lane == 0) {
      out_len[j] = keep;
      state[j] = rng.s;
    }
  }
}

struct DetPatch {
  uint32_t off, width, value;
};

__global__ void __launch_bounds__(128) hfz_k_deterministic(const uint8_t* __restrict__ in,
                                                           uint64_t len,
                                                           const DetPatch* __restrict__ patches,
                                                           uint8_t* __restrict__ out, uint64_t count) {
  for (uint64_t m = blockIdx.x; m < count; m += gridDim.x) {
    const DetPatch p = patches[m];
    uint8_t* o = out + m * len;
    for (uint64_t i = threadIdx.x; i < len; i += blockDim.x) {
      uint8_t b = in[i];
      if (i >= p.off && i < (uint64_t)p.off + p.width) b = (uint8_t)(p.value >> (8 * (i - p.off)));
      o[i] = b;
    }
  }
}

// host enumeration of the deterministic stage in the reference's order (engine.cpp:53-105)
const int8_t kI8[9] = {-128, -1, 0, 1, 16, 32, 64, 100, 127};
const int16_t kI16[10] = {-32768, -129, 128, 255, 256, 512, 1000, 1024, 4096, 32767};
const int32_t kI32[8] = {(-2147483647 - 1), -100663046, -32769, 32768, 65535, 65536, 100663045, 2147483647};

uint64_t read_le(const uint8_t* p, unsigned w) {
  uint64_t v = 0;
  for (unsigned i = 0; i < w; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

uint64_t enumerate_det(const uint8_t* in, uint64_t len, std::vector<DetPatch>* out) {
  uint64_t count = 0;
  auto emit = [&](uint64_t off, unsigned w, uint64_t v) {
    if (out) out->push_back(DetPatch{(uint32_t)off, w, (uint32_t)v});
    ++count;
  };
  const uint64_t cap = len < 32 ? len : 32;  // kDetOffsetCap
  for (uint64_t i = 0; i < cap; ++i)
    for (int b = 7; b >= 0; --b) emit(i, 1, in[i] ^ (1u << b));
  const unsigned widths[3] = {1, 2, 4};
  for (unsigned w : widths) {
    if (len < w) continue;
    const uint64_t end = len - w + 1 < cap ? len - w + 1 : cap;
    const uint64_t mask = (1ull << (8 * w)) - 1;
    for (uint64_t i = 0; i < end; ++i) {
      const uint64_t orig = read_le(in + i, w);
      for (uint64_t d = 1; d <= 35; ++d) {
        emit(i, w, (orig + d) & mask);
        emit(i, w, (orig - d) & mask);
      }
    }
  }
  for (int wi = 0; wi < 3; ++wi) {
    const unsigned w = widths[wi];
    if (len < w) continue;
    const uint64_t end = len - w + 1 < cap ? len - w + 1 : cap;
    const uint64_t mask = (1ull << (8 * w)) - 1;
    const int nv = wi == 0 ? 9 : (wi == 1 ? 10 : 8);
    for (uint64_t i = 0; i < end; ++i) {
      const uint64_t orig = read_le(in + i, w);
      for (int k = 0; k < nv; ++k) {
        const int64_t vv = wi == 0 ? kI8[k] : (wi == 1 ? kI16[k] : kI32[k]);
        const uint64_t v = (uint64_t)vv & mask;
        if (v == orig) continue;  // no-op overwrites are skipped
        emit(i, w, v);
      }
    }
  }
  return count;
}

}  // namespace

extern "C" uint64_t hfz_havoc_max_out(uint64_t in_len) {
  const uint64_t m = in_len + 64 * 16;
  return m > kMaxInput ? kMaxInput : m;
}

extern "C" int hfz_havoc_batch(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                               uint64_t n, uint64_t* rng_state_inout, uint8_t* out_bytes,
                               const uint64_t* out_off, uint64_t* out_len, uint32_t* draws_out) {
  if (!ctx || (n && (!in_bytes || !in_off || !rng_state_inout || !out_bytes || !out_off || !out_len))) {
    hfz_set_error("hfz_havoc_batch: null argument");
    return HFZ_EINVAL;
  }
  if (n == 0) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  // plan + apply per chunk of slots: the edit lists of a chunk live in context scratch (528 bytes per
  // slot, at most kHavocChunk slots = 69 MB, grown geometrically and kept for the context's lifetime)
  const uint64_t chunk = n < kHavocChunk ? n : kHavocChunk;
  if (ctx->hv_ops_cap < chunk) {
    uint64_t want = ctx->hv_ops_cap * 2 > chunk ? ctx->hv_ops_cap * 2 : chunk;
    if (want > kHavocChunk) want = kHavocChunk;
    HFZ_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(ctx->hv_ops);
    ctx->hv_ops = nullptr;
    ctx->hv_ops_cap = 0;
    HFZ_CUDA(cudaMalloc(&ctx->hv_ops, want * kOpWords * sizeof(uint64_t)));
    ctx->hv_ops_cap = want;
  }
  unsigned long long* next_slot = ctx->d_small + 5;
  // four CTAs' working buffers (4 x 48 KB) need the large shared-memory carve-out
  HFZ_CUDA(cudaFuncSetAttribute(hfz_k_havoc_apply, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  for (uint64_t j0 = 0; j0 < n; j0 += chunk) {
    const uint64_t m = n - j0 < chunk ? n - j0 : chunk;
    hfz_k_havoc_plan_ops<<<(uint32_t)((m + 63) / 64), 64, 0, ctx->stream>>>(
        in_off + j0, m, rng_state_inout + j0, ctx->hv_ops, out_len + j0, draws_out ? draws_out + j0 : nullptr, next_slot);
    uint64_t blocks = (m + kHavocWarps - 1) / kHavocWarps;
    const uint64_t maxb = (uint64_t)ctx->num_sms * 4;  // 4 CTAs of 48 KB and 256 threads x 64 registers fit an SM
    if (blocks > maxb) blocks = maxb;
    hfz_k_havoc_apply<<<(uint32_t)blocks, kHavocWarps * 32, 0, ctx->stream>>>(in_bytes, in_off + j0, m, ctx->hv_ops, out_bytes,
                                                                               out_off + j0, next_slot);
    ctx->launches += 2;
  }
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

extern "C" int hfz_havoc_serial_plan(hfz_ctx* ctx, const uint64_t* in_off, uint64_t n,
                                     uint64_t* stream_state_inout, uint64_t* slot_states_out) {
  if (!ctx || !stream_state_inout || (n && (!in_off || !slot_states_out))) {
    hfz_set_error("hfz_havoc_serial_plan: null argument");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  hfz_k_havoc_plan<<<1, 32, 0, ctx->stream>>>(in_off, n, stream_state_inout, slot_states_out);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

extern "C" int hfz_splice_batch(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                                const uint32_t* a_idx, const uint32_t* b_idx, uint64_t n,
                                uint64_t* rng_state_inout, uint8_t* out_bytes,
                                const uint64_t* out_off, uint64_t* out_len) {
  if (!ctx || (n && (!in_bytes || !in_off || !a_idx || !b_idx || !rng_state_inout || !out_bytes ||
                     !out_off || !out_len))) {
    hfz_set_error("hfz_splice_batch: null argument");
    return HFZ_EINVAL;
  }
  if (n == 0) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  uint64_t blocks = (n + 7) / 8;
  const uint64_t maxb = (uint64_t)ctx->num_sms * 8;
  if (blocks > maxb) blocks = maxb;
  hfz_k_splice<<<(uint32_t)blocks, 256, 0, ctx->stream>>>(in_bytes, in_off, a_idx, b_idx, n,
                                                           rng_state_inout, out_bytes, out_off, out_len);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

extern "C" uint64_t hfz_deterministic_count(const uint8_t* in_host, uint64_t in_len) {
  if (!in_host && in_len) return 0;
  return enumerate_det(in_host, in_len, nullptr);
}

extern "C" int hfz_deterministic_batch(hfz_ctx* ctx, const uint8_t* in_dev, uint64_t in_len,
                                       const uint8_t* in_host, uint8_t* out_dev, uint64_t count) {
  if (!ctx || (in_len && (!in_dev || !in_host)) || (count && in_len && !out_dev)) {
    hfz_set_error("hfz_deterministic_batch: null argument");
    return HFZ_EINVAL;
  }
  std::vector<DetPatch> patches;
  const uint64_t want = enumerate_det(in_host, in_len, &patches);
  if (want != count) {
    hfz_set_error("hfz_deterministic_batch: count %llu does not match the input (%llu)",
                  (unsigned long long)count, (unsigned long long)want);
    return HFZ_EINVAL;
  }
  if (count == 0 || in_len == 0) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  DetPatch* d_p = nullptr;
  HFZ_CUDA(cudaMalloc(&d_p, count * sizeof(DetPatch)));
  cudaError_t e = cudaMemcpyAsync(d_p, patches.data(), count * sizeof(DetPatch),
                                  cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) {
    const uint32_t blocks = (uint32_t)(count < 65535 ? count : 65535);
    hfz_k_deterministic<<<blocks, 128, 0, ctx->stream>>>(in_dev, in_len, d_p, out_dev, count);
    ++ctx->launches;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // patches / d_p must outlive the kernel
  cudaFree(d_p);
  if (e != cudaSuccess) return hfz_cuda_fail(e, "hfz_deterministic_batch");
  return HFZ_OK;
}

// ---------------------------------------------------------------------------
// host-buffer forms: stage through temporary device buffers, synchronous

namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, n ? n : 16); }
  template <typename T> T* as() { return static_cast<T*>(p); }
};
#define HFZ_TRY(call)                                          \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return hfz_cuda_fail(_e, #call);    \
  } while (0)
}  // namespace


namespace {
// host-side validation of packed inputs: lengths up to kMaxInputBytes, offsets non-decreasing
int check_lengths(const char* who, const uint64_t* in_off, uint64_t n) {
  for (uint64_t j = 0; j < n; ++j) {
    if (in_off[j + 1] < in_off[j] || in_off[j + 1] - in_off[j] > kMaxInput) {
      hfz_set_error("%s: input %llu is longer than HFZ_MAX_INPUT_BYTES (or its offsets decrease); the reference accepts "
                    "such inputs and truncates after the first edit (src/engine.cpp:190), this library rejects them",
                    who, (unsigned long long)j);
      return HFZ_EINVAL;
    }
  }
  return HFZ_OK;
}
}  // namespace

extern "C" int hfz_havoc_batch_host(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                                    uint64_t n, uint64_t* rng_state_inout, uint8_t* out_bytes,
                                    const uint64_t* out_off, uint64_t* out_len, uint32_t* draws_out) {
  if (!ctx || (n && (!in_off || !rng_state_inout || !out_bytes || !out_off || !out_len))) {
    hfz_set_error("hfz_havoc_batch_host: null argument");
    return HFZ_EINVAL;
  }
  if (n == 0) return HFZ_OK;
  if (int rc = check_lengths("hfz_havoc_batch_host", in_off, n)) return rc;
  HFZ_TRY(cudaSetDevice(ctx->device));
  const uint64_t in_total = in_off[n], out_total = out_off[n];
  DevBuf d_in, d_ioff, d_state, d_out, d_ooff, d_olen, d_draws;
  HFZ_TRY(d_in.alloc(in_total + 16));
  HFZ_TRY(d_ioff.alloc((n + 1) * 8));
  HFZ_TRY(d_state.alloc(n * 8));
  HFZ_TRY(d_out.alloc(out_total + 16));
  HFZ_TRY(d_ooff.alloc((n + 1) * 8));
  HFZ_TRY(d_olen.alloc(n * 8));
  HFZ_TRY(d_draws.alloc(n * 4));
  cudaStream_t st = ctx->stream;
  if (in_total) HFZ_TRY(cudaMemcpyAsync(d_in.p, in_bytes, in_total, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_ioff.p, in_off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_state.p, rng_state_inout, n * 8, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_ooff.p, out_off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
  int rc = hfz_havoc_batch(ctx, d_in.as<uint8_t>(), d_ioff.as<uint64_t>(), n, d_state.as<uint64_t>(),
                           d_out.as<uint8_t>(), d_ooff.as<uint64_t>(), d_olen.as<uint64_t>(),
                           d_draws.as<uint32_t>());
  if (rc) return rc;
  if (out_total) HFZ_TRY(cudaMemcpyAsync(out_bytes, d_out.p, out_total, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaMemcpyAsync(out_len, d_olen.p, n * 8, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaMemcpyAsync(rng_state_inout, d_state.p, n * 8, cudaMemcpyDeviceToHost, st));
  if (draws_out) HFZ_TRY(cudaMemcpyAsync(draws_out, d_draws.p, n * 4, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaStreamSynchronize(st));
  return HFZ_OK;
}

extern "C" int hfz_havoc_serial_host(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                                     uint64_t n, uint64_t* stream_state_inout, uint8_t* out_bytes,
                                     const uint64_t* out_off, uint64_t* out_len) {
  if (!ctx || !stream_state_inout || (n && (!in_off || !out_bytes || !out_off || !out_len))) {
    hfz_set_error("hfz_havoc_serial_host: null argument");
    return HFZ_EINVAL;
  }
  if (n == 0) return HFZ_OK;
  if (int rc = check_lengths("hfz_havoc_serial_host", in_off, n)) return rc;
  HFZ_TRY(cudaSetDevice(ctx->device));
  const uint64_t in_total = in_off[n], out_total = out_off[n];
  DevBuf d_in, d_ioff, d_stream, d_state, d_out, d_ooff, d_olen;
  HFZ_TRY(d_in.alloc(in_total + 16));
  HFZ_TRY(d_ioff.alloc((n + 1) * 8));
  HFZ_TRY(d_stream.alloc(8));
  HFZ_TRY(d_state.alloc(n * 8));
  HFZ_TRY(d_out.alloc(out_total + 16));
  HFZ_TRY(d_ooff.alloc((n + 1) * 8));
  HFZ_TRY(d_olen.alloc(n * 8));
  cudaStream_t st = ctx->stream;
  if (in_total) HFZ_TRY(cudaMemcpyAsync(d_in.p, in_bytes, in_total, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_ioff.p, in_off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_stream.p, stream_state_inout, 8, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_ooff.p, out_off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
  int rc = hfz_havoc_serial_plan(ctx, d_ioff.as<uint64_t>(), n, d_stream.as<uint64_t>(), d_state.as<uint64_t>());
  if (rc) return rc;
  rc = hfz_havoc_batch(ctx, d_in.as<uint8_t>(), d_ioff.as<uint64_t>(), n, d_state.as<uint64_t>(),
                       d_out.as<uint8_t>(), d_ooff.as<uint64_t>(), d_olen.as<uint64_t>(), nullptr);
  if (rc) return rc;
  if (out_total) HFZ_TRY(cudaMemcpyAsync(out_bytes, d_out.p, out_total, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaMemcpyAsync(out_len, d_olen.p, n * 8, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaMemcpyAsync(stream_state_inout, d_stream.p, 8, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaStreamSynchronize(st));
  return HFZ_OK;
}

extern "C" int hfz_splice_batch_host(hfz_ctx* ctx, const uint8_t* in_bytes, const uint64_t* in_off,
                                     uint64_t n_inputs, const uint32_t* a_idx, const uint32_t* b_idx,
                                     uint64_t n, uint64_t* rng_state_inout, uint8_t* out_bytes,
                                     const uint64_t* out_off, uint64_t* out_len) {
  if (!ctx || (n && (!in_off || !a_idx || !b_idx || !rng_state_inout || !out_bytes || !out_off || !out_len))) {
    hfz_set_error("hfz_splice_batch_host: null argument");
    return HFZ_EINVAL;
  }
  if (n == 0) return HFZ_OK;
  for (uint64_t j = 0; j < n; ++j)
    if (a_idx[j] >= n_inputs || b_idx[j] >= n_inputs) {
      hfz_set_error("hfz_splice_batch_host: input index out of range");
      return HFZ_EINVAL;
    }
  if (int rc = check_lengths("hfz_splice_batch_host", in_off, n_inputs)) return rc;
  HFZ_TRY(cudaSetDevice(ctx->device));
  const uint64_t in_total = in_off[n_inputs], out_total = out_off[n];
  DevBuf d_in, d_ioff, d_a, d_b, d_state, d_out, d_ooff, d_olen;
  HFZ_TRY(d_in.alloc(in_total + 16));
  HFZ_TRY(d_ioff.alloc((n_inputs + 1) * 8));
  HFZ_TRY(d_a.alloc(n * 4));
  HFZ_TRY(d_b.alloc(n * 4));
  HFZ_TRY(d_state.alloc(n * 8));
  HFZ_TRY(d_out.alloc(out_total + 16));
  HFZ_TRY(d_ooff.alloc((n + 1) * 8));
  HFZ_TRY(d_olen.alloc(n * 8));
  cudaStream_t st = ctx->stream;
  if (in_total) HFZ_TRY(cudaMemcpyAsync(d_in.p, in_bytes, in_total, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_ioff.p, in_off, (n_inputs + 1) * 8, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_a.p, a_idx, n * 4, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_b.p, b_idx, n * 4, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_state.p, rng_state_inout, n * 8, cudaMemcpyHostToDevice, st));
  HFZ_TRY(cudaMemcpyAsync(d_ooff.p, out_off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
  int rc = hfz_splice_batch(ctx, d_in.as<uint8_t>(), d_ioff.as<uint64_t>(), d_a.as<uint32_t>(),
                            d_b.as<uint32_t>(), n, d_state.as<uint64_t>(), d_out.as<uint8_t>(),
                            d_ooff.as<uint64_t>(), d_olen.as<uint64_t>());
  if (rc) return rc;
  if (out_total) HFZ_TRY(cudaMemcpyAsync(out_bytes, d_out.p, out_total, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaMemcpyAsync(out_len, d_olen.p, n * 8, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaMemcpyAsync(rng_state_inout, d_state.p, n * 8, cudaMemcpyDeviceToHost, st));
  HFZ_TRY(cudaStreamSynchronize(st));
  return HFZ_OK;
}

extern "C" int hfz_deterministic_host(hfz_ctx* ctx, const uint8_t* in, uint64_t in_len, uint8_t* out,
                                      uint64_t count) {
  if (!ctx || (in_len && !in) || (count && in_len && !out)) {
    hfz_set_error("hfz_deterministic_host: null argument");
    return HFZ_EINVAL;
  }
  if (count == 0 || in_len == 0) {
    if (hfz_deterministic_count(in, in_len) != count) {
      hfz_set_error("hfz_deterministic_host: count mismatch");
      return HFZ_EINVAL;
    }
    return HFZ_OK;
  }
  HFZ_TRY(cudaSetDevice(ctx->device));
  DevBuf d_in, d_out;
  HFZ_TRY(d_in.alloc(in_len));
  HFZ_TRY(d_out.alloc(count * in_len));
  HFZ_TRY(cudaMemcpyAsync(d_in.p, in, in_len, cudaMemcpyHostToDevice, ctx->stream));
  int rc = hfz_deterministic_batch(ctx, d_in.as<uint8_t>(), in_len, in, d_out.as<uint8_t>(), count);
  if (rc) return rc;
  HFZ_TRY(cudaMemcpyAsync(out, d_out.p, count * in_len, cudaMemcpyDeviceToHost, ctx->stream));
  HFZ_TRY(cudaStreamSynchronize(ctx->stream));
  return HFZ_OK;
}
