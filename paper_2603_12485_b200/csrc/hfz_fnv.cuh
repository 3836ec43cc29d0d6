// hfz_fnv.cuh -- 64-bit FNV-1a over a byte stream, computed by a whole warp in parallel.
//
// trace_signature (src/coverage.cpp:89-97, include/hetfuzz/coverage.hpp:208-220) is h = (h ^ b) * P per
// byte, P = 2^40 + 0x1b3: a serial chain (the XOR is not affine), ~4,000 dependent steps for a map
// at 2 % density.  One lane running it costs ~20 cycles per step whatever else the warp does; that chain
// was what a small batch's step time consisted of.  It can be taken apart:
//   * h ^ b = h + d with d = (l ^ b) - l = b - 2 (b & l), l = h mod 256, so h' = (h + d) * P: AFFINE in h
//     once the low bytes l_i of the running hash are known:  h_n = h_0 P^n + sum_i d_i P^(n - i);
//   * the low byte is a chain of its own, l' = ((l ^ b) * 0xb3) mod 256, and bit j of a product
//     depends on bits <= j of the factor only: bit j of l' = x_j ^ g_j(x_0 .. x_{j-1}), x = l ^ b.  With the
//     lower bit planes resolved, plane j of the whole sequence is an exclusive prefix XOR.
// So: every lane takes 32 consecutive steps, bit-sliced (8 words = 8 bit planes of its 32 bytes); plane
// by plane the multiplier's lower-bit contribution g_j is a fixed network of ~34 three-input logic
// ops on words, the prefix XOR is five shift-xor steps inside the word plus one ballot across the lanes;
// the low bytes are un-sliced again, and each lane's share of the sum is a dot product of its 32
// deltas with compile-time powers of P; one 64-bit warp sum combines the lanes.  1,024 steps per block,
// ~850 warp-instructions, no serial dependence longer than the 8 planes.
// (Validated against the byte-serial definition by tests/test_feedback_gpu.py::test_warp_fnv through
// hfz_dbg_warp_fnv; the step-by-step model it was ported from is scripts/fnv_bitslice_model.py.)
#pragma once
#include <stdint.h>

namespace pfnv {

constexpr uint64_t kPrime = 0x100000001b3ull;
__host__ __device__ constexpr uint64_t ipow(unsigned k) {
  uint64_t r = 1;
  for (unsigned i = 0; i < k; ++i) r *= kPrime;
  return r;
}
struct PowTab {
  uint64_t pw[32];  // P^(32 (31 - L)): what lane L's share is multiplied by (the lanes after it hold 32 steps each)
  uint64_t pt[33];  // P^k
  constexpr PowTab() : pw{}, pt{} {
    for (int L = 0; L < 32; ++L) pw[L] = ipow(32u * (31u - (unsigned)L));
    for (int k = 0; k <= 32; ++k) pt[k] = ipow((unsigned)k);
  }
};
__constant__ PowTab c_pow = PowTab();

// 8 x 8 bit-matrix transpose of the bytes of x (bit i of byte j <-> bit j of byte i)
__device__ __forceinline__ uint64_t t8x8(uint64_t x) {
  uint64_t t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
  x = x ^ t ^ (t << 7);
  t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
  x = x ^ t ^ (t << 14);
  t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
  x = x ^ t ^ (t << 28);
  return x;
}

// One block of up to 1,024 steps.  w: this lane's 32 bytes (steps 32 lane .. 32 lane + 31 of the block,
// byte k in word k / 4), invalid steps hold 0; vm: its valid steps.  Invalid steps sit at the FRONT of
// the block only, so every lane after a valid step holds 32 valid ones.  h_in: the hash before the
// block's first valid step.  Returns the hash after the block (in every lane); at least one step valid.
__device__ __forceinline__ uint64_t block(uint64_t h_in, const uint32_t (&w)[8], uint32_t vm, int lane) {
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t l0 = (uint32_t)h_in & 0xffu;
  uint32_t B[8], Lp[8];
  {  // bytes -> bit planes
    uint64_t x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = t8x8((uint64_t)w[2 * q] | ((uint64_t)w[2 * q + 1] << 32));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int jj = j & 3;
      const uint32_t a = j < 4 ? (uint32_t)x[0] : (uint32_t)(x[0] >> 32), b = j < 4 ? (uint32_t)x[1] : (uint32_t)(x[1] >> 32);
      const uint32_t c = j < 4 ? (uint32_t)x[2] : (uint32_t)(x[2] >> 32), d = j < 4 ? (uint32_t)x[3] : (uint32_t)(x[3] >> 32);
      const uint32_t sel = (uint32_t)(((4 + jj) << 4) | jj);
      B[j] = __byte_perm(__byte_perm(a, b, sel), __byte_perm(c, d, sel), 0x5410);
    }
  }
  // plane j: T = (b_j ^ g_j) on valid steps; l_j = l0_j ^ exclusive prefix XOR of T over the block
#define PFNV_PLANE(j)                                                                  \
  {                                                                                    \
    uint32_t p = (B[j] ^ G##j) & vm;                                                   \
    p ^= p << 1;                                                                       \
    p ^= p << 2;                                                                       \
    p ^= p << 4;                                                                       \
    p ^= p << 8;                                                                       \
    p ^= p << 16;                                                                      \
    const uint32_t par = __ballot_sync(0xffffffffu, (p >> 31) != 0u);                  \
    const uint32_t carry = ((l0 >> j) ^ (uint32_t)__popc(par & lt)) & 1u;              \
    Lp[j] = (p << 1) ^ (0u - carry);                                                   \
  }                                                                                    \
  const uint32_t X##j = Lp[j] ^ B[j];                                                  \
  const uint32_t K##j = X##j & G##j;
  // column 0 of (x mod 2^0) * 0xb3
  const uint32_t G0 = 0u;
  PFNV_PLANE(0)
  // column 1 of (x mod 2^1) * 0xb3
  const uint32_t t1 = K0 ^ X0;
  const uint32_t t2 = K0 & X0;
  const uint32_t G1 = t1;
  PFNV_PLANE(1)
  // column 2 of (x mod 2^2) * 0xb3
  const uint32_t t3 = t2 ^ K1 ^ X1;
  const uint32_t t4 = (t2 & K1) | (X1 & (t2 ^ K1));
  const uint32_t G2 = t3;
  PFNV_PLANE(2)
  // column 3 of (x mod 2^3) * 0xb3
  const uint32_t t5 = t4 ^ K2 ^ X2;
  const uint32_t t6 = (t4 & K2) | (X2 & (t4 ^ K2));
  const uint32_t G3 = t5;
  PFNV_PLANE(3)
  // column 4 of (x mod 2^4) * 0xb3
  const uint32_t t7 = t6 ^ K3 ^ X3;
  const uint32_t t8 = (t6 & K3) | (X3 & (t6 ^ K3));
  const uint32_t t9 = X0 ^ t7;
  const uint32_t t10 = X0 & t7;
  const uint32_t G4 = t9;
  PFNV_PLANE(4)
  // column 5 of (x mod 2^5) * 0xb3
  const uint32_t t11 = t8 ^ t10 ^ K4;
  const uint32_t t12 = (t8 & t10) | (K4 & (t8 ^ t10));
  const uint32_t t13 = X4 ^ X1 ^ X0;
  const uint32_t t14 = (X4 & X1) | (X0 & (X4 ^ X1));
  const uint32_t t15 = t11 ^ t13;
  const uint32_t t16 = t11 & t13;
  const uint32_t G5 = t15;
  PFNV_PLANE(5)
  // column 6 of (x mod 2^6) * 0xb3
  const uint32_t t17 = t12 ^ t14 ^ t16;
  const uint32_t t18 = (t12 & t14) | (t16 & (t12 ^ t14));
  const uint32_t t19 = K5 ^ X5 ^ X2;
  const uint32_t t20 = (K5 & X5) | (X2 & (K5 ^ X5));
  const uint32_t t21 = X1 ^ t17 ^ t19;
  const uint32_t t22 = (X1 & t17) | (t19 & (X1 ^ t17));
  const uint32_t G6 = t21;
  PFNV_PLANE(6)
  // column 7 of (x mod 2^7) * 0xb3
  const uint32_t t23 = t18 ^ t20 ^ t22;
  const uint32_t t25 = K6 ^ X6 ^ X3;
  const uint32_t t27 = X2 ^ X0 ^ t23;
  const uint32_t t29 = t25 ^ t27;
  const uint32_t G7 = t29;
  PFNV_PLANE(7)
  (void)K7;
#undef PFNV_PLANE

  uint32_t lw[8];
  {  // low-byte planes -> bytes
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t sel = (uint32_t)(((4 + q) << 4) | q);
      const uint32_t lo = __byte_perm(__byte_perm(Lp[0], Lp[1], sel), __byte_perm(Lp[2], Lp[3], sel), 0x5410);
      const uint32_t hi = __byte_perm(__byte_perm(Lp[4], Lp[5], sel), __byte_perm(Lp[6], Lp[7], sel), 0x5410);
      const uint64_t x = t8x8((uint64_t)lo | ((uint64_t)hi << 32));
      lw[2 * q] = (uint32_t)x;
      lw[2 * q + 1] = (uint32_t)(x >> 32);
    }
  }
  // this lane's share: sum_s d_s P^(32 - s), d = b - 2 (b & l) (0 on invalid steps: their b is 0)
  uint64_t acc = 0;
#pragma unroll
  for (int s = 0; s < 32; ++s) {
    const uint32_t bw = w[s >> 2], mw = bw & lw[s >> 2];
    const int32_t d = (int32_t)((bw >> (8 * (s & 3))) & 0xffu) - 2 * (int32_t)((mw >> (8 * (s & 3))) & 0xffu);
    acc += (uint64_t)((int64_t)d * (int64_t)ipow(32u - (unsigned)s));
  }
  const uint32_t live = __ballot_sync(0xffffffffu, vm != 0u);
  if (lane == __ffs(live) - 1) acc += h_in * c_pow.pt[32 - (__ffs(vm) - 1)];  // the hash so far enters at the first valid step
  acc *= c_pow.pw[lane];
#pragma unroll
  for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  return acc;
}

// Both signatures of an ordered entry list in SHARED memory (entry = slot | rung << 24; Full hashes the
// slot's two low bytes and the class byte 1 << rung, Simple the two slot bytes: src/coverage.cpp:91-95),
// continuing hf / hs.  stream: 3,072 + 16 bytes of scratch in shared memory, 16-byte aligned; n <= 1,024.
// Called by all 32 lanes; entries must be visible to the warp (__syncwarp() before).
template <int BPE>
__device__ __forceinline__ uint64_t chain_entries(uint64_t h, const uint32_t* en, uint32_t n, uint8_t* stream, int lane) {
  if (n == 0) return h;
  const uint32_t steps = n * BPE, nb = (steps + 1023u) / 1024u, pad = nb * 1024u - steps;
  // the byte stream, right-aligned in nb blocks (the padding of the first block reads as zeros)
  reinterpret_cast<uint4*>(stream)[lane] = make_uint4(0, 0, 0, 0);
  reinterpret_cast<uint4*>(stream)[lane + 32] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  for (uint32_t i = lane; i < n; i += 32) {
    const uint32_t e = en[i];
    uint8_t* o = stream + pad + i * BPE;
    o[0] = (uint8_t)e;
    o[1] = (uint8_t)(e >> 8);
    if (BPE == 3) o[2] = (uint8_t)(1u << (e >> 24));
  }
  __syncwarp();
  for (uint32_t b = 0; b < nb; ++b) {
    const uint4* src = reinterpret_cast<const uint4*>(stream + b * 1024u + (uint32_t)lane * 32u);
    const uint4 v0 = src[0], v1 = src[1];
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    const uint32_t t0 = b * 1024u + (uint32_t)lane * 32u;  // first padded step of this lane
    const uint32_t vm = t0 >= pad ? 0xffffffffu : (t0 + 32u <= pad ? 0u : 0xffffffffu << (pad - t0));
    h = block(h, w, vm, lane);
  }
  __syncwarp();
  return h;
}

}  // namespace pfnv
