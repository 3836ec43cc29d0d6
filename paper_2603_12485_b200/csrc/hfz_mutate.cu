// hfz_mutate.cu -- K3 batched mutators: havoc, splice, deterministic stage.
//
// Reference semantics (paths under /root/reference/proj):
//   havoc_mutant            src/engine.cpp:119-193   (tables :27-38, write_le :46-49)
//   splice_mutant           src/engine.cpp:195-204
//   for_each_deterministic  src/engine.cpp:53-105
//   Rng                     include/hetfuzz/rng.hpp:11-46
//
// One warp owns one slot.  The splitmix64 stream is warp-uniform (every lane advances the
// same state), single-byte edits are done by lane 0 and block moves (erase / insert / copy)
// by the whole warp on a working buffer that lives in shared memory when the slot's maximum
// output fits (inputs up to ~5 KB: BASELINE.json configs[3]) and directly in the slot's
// output region in global memory otherwise (inputs up to kMaxInputBytes = 1 MiB).
#include <string.h>

#include <vector>

#include "hfz_common.cuh"

namespace {

constexpr uint32_t kMaxInput = HFZ_MAX_INPUT_BYTES;
constexpr int kHavocWarps = 8;
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
// for the whole move, so one shift serves every word -- and stored with one 128-bit store; the two
// partial blocks at the ends of the range keep the bytes outside it.  buf must be 16-byte aligned
// and readable for 16 bytes beyond the data (the working buffers are padded).  A quarter of the
// kernel's instructions used to be the byte-granular version of these loops.
__device__ __forceinline__ uint32_t block_mask(uint64_t blk_lo, uint64_t lo, uint64_t hi) {
  // 16-bit mask of the bytes of block [blk_lo, blk_lo + 16) that lie inside [lo, hi)
  const uint64_t a = lo > blk_lo ? lo - blk_lo : 0, b = hi < blk_lo + 16 ? (hi > blk_lo ? hi - blk_lo : 0) : 16;
  return a >= b ? 0u : ((0xffffu >> (16 - (uint32_t)(b - a))) << (uint32_t)a);
}
__device__ __forceinline__ uint32_t bytes_of(uint32_t m4) {  // 4-bit byte mask -> 32-bit lane mask
  return ((m4 & 1u) * 0xffu) | (((m4 >> 1) & 1u) * 0xff00u) | (((m4 >> 2) & 1u) * 0xff0000u) | (((m4 >> 3) & 1u) * 0xff000000u);
}
// one step: blocks [k0, k0 + 32) of the destination (block k = bytes [16k, 16k + 16)); delta = src - dst (signed)
__device__ __forceinline__ void move_blocks(uint8_t* buf, uint64_t k0, uint64_t k_end, int64_t delta, uint64_t dlo, uint64_t dhi,
                                            int lane) {
  const uint64_t k = k0 + lane;
  const bool on = k < k_end;
  uint4 out = make_uint4(0, 0, 0, 0);
  uint32_t m = 0;
  if (on) {
    const int64_t sb = (int64_t)(k * 16) + delta;          // source byte of the block's first byte (may be < 0 only for masked bytes)
    const int64_t sw = sb >> 2;                              // aligned source word (floor)
    const uint32_t sh = (uint32_t)(sb & 3) * 8;
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(buf);
    uint32_t w[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) w[j] = sw + j >= 0 ? w32[sw + j] : 0u;
    out.x = __funnelshift_r(w[0], w[1], sh);
    out.y = __funnelshift_r(w[1], w[2], sh);
    out.z = __funnelshift_r(w[2], w[3], sh);
    out.w = __funnelshift_r(w[3], w[4], sh);
    m = block_mask(k * 16, dlo, dhi);
    if (m != 0xffffu) {  // a partial block at either end of the range: keep the bytes outside it
      const uint4 old = reinterpret_cast<const uint4*>(buf)[k];
      const uint32_t m0 = bytes_of(m), m1 = bytes_of(m >> 4), m2 = bytes_of(m >> 8), m3 = bytes_of(m >> 12);
      out.x = (out.x & m0) | (old.x & ~m0);
      out.y = (out.y & m1) | (old.y & ~m1);
      out.z = (out.z & m2) | (old.z & ~m2);
      out.w = (out.w & m3) | (old.w & ~m3);
    }
  }
  __syncwarp();  // every block of this step is read before any is written
  if (on && m) reinterpret_cast<uint4*>(buf)[k] = out;
  __syncwarp();
}
// buf[dst + i] = buf[src + i], i ascending (dst < src)
__device__ __forceinline__ void smem_move_down(uint8_t* buf, uint64_t dst, uint64_t src, uint64_t n, int lane) {
  if (n == 0) return;
  const uint64_t k_first = dst / 16, k_end = (dst + n + 15) / 16;
  for (uint64_t k0 = k_first; k0 < k_end; k0 += 32) move_blocks(buf, k0, k_end, (int64_t)(src - dst), dst, dst + n, lane);
}
// buf[dst + i] = buf[src + i], i descending (dst > src)
__device__ __forceinline__ void smem_move_up(uint8_t* buf, uint64_t dst, uint64_t src, uint64_t n, int lane) {
  if (n == 0) return;
  const uint64_t k_first = dst / 16, k_end = (dst + n + 15) / 16;
  uint64_t k0 = k_first + ((k_end - k_first - 1) / 32) * 32;  // the highest step first
  for (;;) {
    move_blocks(buf, k0, k_end, -(int64_t)(dst - src), dst, dst + n, lane);
    if (k0 == k_first) break;
    k0 -= 32;
  }
}

// global (any alignment) -> shared (16-byte aligned dst): aligned 32-bit loads + one funnel shift per word
__device__ __forceinline__ void copy_in_smem(uint8_t* dst, const uint8_t* src, uint64_t n, int lane) {
  const uint32_t a = (uint32_t)((uintptr_t)src & 3);
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src - a);  // aligned down: the first word may start before src
  const uint32_t sh = a * 8;
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
  const uint64_t words = (n + 3) / 4;
  // the last source word read is s32[words] when a != 0: it holds bytes of the input itself or, for the batch's
  // last input, of the 16 bytes of slack callers keep behind the packed inputs (hfz.h); guard it anyway
  const uint64_t last_word = ((uint64_t)a + n + 3) / 4;  // exclusive bound of words that hold input bytes
  for (uint64_t w0 = 0; w0 < words; w0 += 32 * 4) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t w = w0 + k * 32 + lane;
      lo[k] = w < words ? __ldg(s32 + w) : 0u;
      hi[k] = (w < words && w + 1 < last_word) ? __ldg(s32 + w + 1) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t w = w0 + k * 32 + lane;
      if (w < words) d32[w] = __funnelshift_r(lo[k], hi[k], sh);
    }
  }
}

__device__ __forceinline__ uint64_t havoc_cap(uint64_t len) {
  const uint64_t m = len + 64 * 16;
  return m > kMaxInput ? kMaxInput : m;
}

// The stacked-havoc edit loop of one slot (src/engine.cpp:120-191).  DRY = true runs only the
// Rng draws and the length bookkeeping -- every below() bound depends on the current length
// alone, never on the bytes -- which is what a serial-stream plan needs (hfz_havoc_serial_plan).
template <bool DRY, bool SMEM = false>
__device__ __forceinline__ uint64_t havoc_edit(uint8_t* v, uint64_t len, WarpRng& rng, int lane) {
  const uint64_t ops = 1 + rng.below(64);
  for (uint64_t op = 0; op < ops; ++op) {
    if (len == 0) {  // engine.cpp:124-129 (no 1 MiB clamp on this branch)
      const uint64_t cnt = 1 + rng.below(8);
      for (uint64_t i = 0; i < cnt; ++i) {
        const uint8_t b = (uint8_t)rng.below(256);
        if (!DRY && lane == 0) v[len] = b;
        ++len;
      }
      if (!DRY) __syncwarp();
      continue;
    }
    switch ((uint32_t)rng.below(9)) {
      case 0: {  // flip one bit, MSB-first numbering
        const uint64_t pos = rng.below((uint32_t)(len * 8));
        if (!DRY && lane == 0) v[pos / 8] ^= (uint8_t)(0x80u >> (pos % 8));
        break;
      }
      case 1: {  // random byte: the VALUE is drawn before the index (C++17 sequencing of '=')
        const uint8_t val = (uint8_t)rng.below(256);
        const uint64_t i = rng.below(len);
        if (!DRY && lane == 0) v[i] = val;
        break;
      }
      case 2: {  // byte +/- delta
        const uint8_t d = (uint8_t)(1 + rng.below(35));
        const uint64_t i = rng.below(len);
        const bool add = rng.below(2) < 1;
        if (!DRY && lane == 0) v[i] = (uint8_t)(add ? v[i] + d : v[i] - d);
        break;
      }
      case 3: {  // interesting 16-bit, little endian
        if (len < 2) break;
        const uint64_t off = rng.below(len - 1);
        const uint16_t val = (uint16_t)c_interesting16[rng.below(10)];
        if (!DRY && lane < 2) v[off + lane] = (uint8_t)(val >> (8 * lane));
        break;
      }
      case 4: {  // interesting 32-bit, little endian
        if (len < 4) break;
        const uint64_t off = rng.below(len - 3);
        const uint32_t val = (uint32_t)c_interesting32[rng.below(8)];
        if (!DRY && lane < 4) v[off + lane] = (uint8_t)(val >> (8 * lane));
        break;
      }
      case 5: {  // delete a block
        if (len < 2) break;
        const uint64_t off = rng.below(len);
        const uint64_t q = len / 4 ? len / 4 : 1;
        const uint64_t max_n = len - off < q ? len - off : q;
        const uint64_t cnt = 1 + rng.below(max_n);
        if (!DRY) __syncwarp();
        if (!DRY) {
          if (SMEM) smem_move_down(v, off, off + cnt, len - off - cnt, lane);
          else warp_move_down(v, off, off + cnt, len - off - cnt, lane);
        }
        len -= cnt;
        break;
      }
      case 6: {  // duplicate a block elsewhere (copy first, then insert)
        const uint64_t src = rng.below(len);
        const uint64_t lim = len - src < 16 ? len - src : 16;
        const uint64_t cnt = 1 + rng.below(lim);
        const uint64_t dst = rng.below(len + 1);
        if (!DRY) __syncwarp();
        const uint8_t blk = (!DRY && (uint64_t)lane < cnt) ? v[src + lane] : 0;
        // insert with the 1 MiB clamp folded in: bytes that would land past the cap are dropped
        const uint64_t new_len = len + cnt > kMaxInput ? kMaxInput : len + cnt;
        if (!DRY) __syncwarp();
        if (!DRY && new_len > dst + cnt) {
          if (SMEM) smem_move_up(v, dst + cnt, dst, new_len - dst - cnt, lane);
          else warp_move_up(v, dst + cnt, dst, new_len - dst - cnt, lane);
        }
        if (!DRY && (uint64_t)lane < cnt && dst + lane < new_len) v[dst + lane] = blk;
        len = new_len;
        break;
      }
      case 7: {  // constant fill
        const uint64_t off = rng.below(len);
        const uint64_t lim = len - off < 16 ? len - off : 16;
        const uint64_t cnt = 1 + rng.below(lim);
        const uint8_t b = (uint8_t)rng.below(256);
        if (!DRY && (uint64_t)lane < cnt) v[off + lane] = b;
        break;
      }
      default: {  // 8: swap two bytes
        const uint64_t i = rng.below(len);
        const uint64_t k = rng.below(len);
        if (!DRY && lane == 0) {
          const uint8_t t = v[i];
          v[i] = v[k];
          v[k] = t;
        }
        break;
      }
    }
    if (!DRY) __syncwarp();
    if (len > kMaxInput) len = kMaxInput;
  }
  return len;
}

__global__ void __launch_bounds__(kHavocWarps * 32) hfz_k_havoc(
    const uint8_t* __restrict__ in_bytes, const uint64_t* __restrict__ in_off, uint64_t n,
    uint64_t* __restrict__ state, uint8_t* __restrict__ out_bytes,
    const uint64_t* __restrict__ out_off, uint64_t* __restrict__ out_len,
    uint32_t* __restrict__ draws_out, unsigned long long* __restrict__ next_slot) {
  __shared__ __align__(16) uint8_t s_buf[kHavocWarps][kSmemCap + 16];  // + 16: the block moves read one block past the data
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // slots are handed out dynamically: a mutant stacks 1..64 edits, so their costs differ widely
  for (;;) {
    unsigned long long jj = 0;
    if (lane == 0) jj = atomicAdd(next_slot, 1ull);
    const uint64_t j = __shfl_sync(0xffffffffu, jj, 0);
    if (j >= n) break;
    const uint64_t i0 = in_off[j];
    uint64_t len = in_off[j + 1] - i0;
    // Inputs longer than kMaxInputBytes are rejected by the host-buffer entry points (hfz.h); a
    // device-buffer caller that passes one anyway gets a memory-safe result: the slot's capacity is
    // hfz_havoc_max_out(len) = 1 MiB, so only the first 1 MiB is mutated.
    if (len > kMaxInput) len = kMaxInput;
    uint8_t* out = out_bytes + out_off[j];
    const bool in_smem = havoc_cap(len) <= kSmemCap;
    uint8_t* v = in_smem ? s_buf[warp] : out;
    if (in_smem) copy_in_smem(v, in_bytes + i0, len, lane);
    else warp_copy(v, in_bytes + i0, len, lane);
    __syncwarp();

    WarpRng rng;
    rng.init(state[j], lane);
    len = in_smem ? havoc_edit<false, true>(v, len, rng, lane) : havoc_edit<false, false>(v, len, rng, lane);
    if (in_smem) {
      warp_copy(out, v, len, lane);
      __syncwarp();
    }
    if (lane == 0) {
      out_len[j] = len;
      state[j] = rng.s;
      if (draws_out) draws_out[j] = rng.draws;
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
    havoc_edit<true>(nullptr, in_off[j + 1] - in_off[j], rng, lane);
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
  uint64_t blocks = (n + kHavocWarps - 1) / kHavocWarps;
  const uint64_t maxb = (uint64_t)ctx->num_sms * 4;  // at most 4 CTAs of 48 KB fit an SM
  if (blocks > maxb) blocks = maxb;
  unsigned long long* next_slot = ctx->d_small + 5;
  HFZ_CUDA(cudaMemsetAsync(next_slot, 0, sizeof(unsigned long long), ctx->stream));
  hfz_k_havoc<<<(uint32_t)blocks, kHavocWarps * 32, 0, ctx->stream>>>(
      in_bytes, in_off, n, rng_state_inout, out_bytes, out_off, out_len, draws_out, next_slot);
  ++ctx->launches;
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
