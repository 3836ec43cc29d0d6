// hfz_feedback.cu -- K2 fused feedback scan, K2b first-occurrence resolve, K4 virgin merge.
//
// Reference semantics being reproduced (paths under /root/reference/proj):
//   classify_trace  src/coverage.cpp:58-72      trace_signature  src/coverage.cpp:89-97
//   has_new_bits    src/coverage.cpp:74-87      VirginMap::observe include/hetfuzz/coverage.hpp:166-174
//   per-exec order  src/engine.cpp:471-478
//
// Design (DESIGN.md has the long form):
//  * scan: ONE coalesced pass over the raw maps (see hfz_k_scan below).  Nothing is written
//    back except 21 bytes per map.
//  * exact sequential has_new_bits without a sequential pass: for every (slot, class bit) not
//    in V0 the scan records the FIRST exec that shows it (atomicMin into `first`).  An exec's
//    Admit code then only depends on which table entries name it (resolve: one pass over the
//    table, whatever the number of novel maps).  Final virgin = V0 | OR of the novelty deltas (merge).
#include <stdio.h>
#include <string.h>

#include <cooperative_groups.h>

#include <type_traits>

#include "hfz_common.cuh"
#include "hfz_fnv.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr uint32_t kNone = 0xffffffffu;
constexpr int kPad = 16;  // per-lane slot padding: makes 128-bit shared loads conflict-free

struct ScanParams {
  const uint8_t* raw;
  uint64_t n_exec;
  uint32_t S, H;
  uint64_t rec_bytes;
  const uint8_t* v0;
  uint32_t* first;
  uint64_t* sig_full;
  uint64_t* sig_simple;
  uint32_t* nnz;
  uint8_t* classed;
  uint32_t n_groups;
  int prefetch;
};

// first-occurrence update: entry = min(entry, e).  Entries only ever decrease, so an L2 read
// that already shows an exec <= e proves the atomic redundant -- on a batch folded into an empty virgin map
// every non-zero slot of every map comes here (86 M updates of ~2.6 k entries for 65,536 maps), and a load is
// cheaper in L2 than a reduction on a contended address.
__device__ __forceinline__ void note_first(uint32_t* entry, uint32_t e) {
  if (__ldcg(entry) > e) atomicMin(entry, e);
}

// non-zero-byte bitmask (4 bits) of a 32-bit word
__device__ __forceinline__ uint32_t nz_bytes(uint32_t w) {
  uint32_t t = (((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) & 0x80808080u;  // bit 7 of each non-zero byte
  return (t * 0x00204081u) >> 28;                                      // gather to bits 0..3
}

template <bool VSMEM, bool CLASSED>
struct Lane {
  uint64_t hf, hs;
  uint32_t nnz;
  // one non-zero slot: both FNV chains, novelty versus V0 (`known` = V0[idx]), optional class store
  __device__ __forceinline__ void visit(uint32_t idx, uint32_t klass, uint32_t known, uint32_t* first,
                                        uint32_t e, uint8_t* classed_row) {
    const uint32_t b0 = idx & 0xffu, b1 = (idx >> 8) & 0xffu;
    hf = hfz_fnv(hfz_fnv(hfz_fnv(hf, b0), b1), klass);
    hs = hfz_fnv(hfz_fnv(hs, b0), b1);
    ++nnz;
    // (rare once the virgin map is warm; hinted so: the block stays out of the chain loop's schedule -- measured
    // 1.62 vs 1.68 ms per 65,536 maps.  A read-before-update as in note_first costs the serial loop more than it
    // saves except on a batch folded into an EMPTY map: 1.86 vs 2.5 ms there, 1.06 vs 0.95 on iid maps.)
    if (__builtin_expect((klass & ~known) != 0u, 0)) atomicMin(first + (size_t)idx * 8 + (31 - __clz(klass)), e);
    if (CLASSED) classed_row[idx] = (uint8_t)klass;
  }
};

// ---------------------------------------------------------------------------
// K2 scan.
//   phase A (per row of ROW bytes per map, per map m of the warp's group): the whole warp
//           loads map m's chunk with ONE coalesced 128-bit load per lane (registers,
//           L1::no_allocate, two register buffers of 16 loads); one ballot gives the chunk's
//           non-zero-vector mask (handed to lane m through shared memory) and only the
//           non-zero 16-byte vectors are scattered into lane m's padded shared-memory slot;
//   phase B (per row): lane m walks ITS map's non-zero vectors: classify, virgin lookup in
//           the TMA-staged shared copy of V0, both FNV chains -- 32 serial chains per warp.
// The FNV-1a signature is a strictly serial 64-bit chain per map, so the only way to keep all
// 32 lanes busy on it is to run 32 independent chains ("lane-per-map").
// Work split: maps are dealt evenly to all warps (groups of <= 32 lanes), so the last wave is
// never a mostly-empty one.  REC_CT is the compile-time record size (0 = run-time): it turns
// the 32 per-map addresses of a row into immediates of one base register.
template <int ROW>
struct RowCfg {
  static constexpr int kSlot = ROW + kPad;      // per-lane shared slot
  static constexpr int kMapsPerLoad = ROW >= 512 ? 1 : 512 / ROW;  // maps covered by one warp-wide 128-bit load
  static constexpr int kLoadsPerMap = ROW >= 512 ? ROW / 512 : 1;  // warp-wide loads per map and row
  static constexpr int kLanesPerMap = (ROW >= 512 ? 512 : ROW) / 16;
  static constexpr int kLoads = 32 / kMapsPerLoad;  // loads per row (32 for 512- and 1,024-byte rows)
  static constexpr int kGroup = 32 / kLoadsPerMap;  // maps per warp: 1,024-byte rows = 16 maps, lanes 16..31 idle in phase B
};

template <bool HOST, int ROW, bool VSMEM, bool CLASSED>
__device__ __forceinline__ void phase_b(const uint8_t* slot, uint32_t vm, uint32_t slot_base,
                                        Lane<VSMEM, CLASSED>& st, const uint8_t* virgin,
                                        uint32_t* first, uint32_t e, uint8_t* classed_row) {
  // Warp-uniform loop (exit by vote) so the warp is provably converged around it; lanes that
  // have run out of entries are predicated off inside.  Software-pipelined: the shared-memory
  // loads of the NEXT non-zero slot (vector, element, virgin byte) are issued before the FNV
  // chains of the current one, so their latency hides behind the dependent multiplies.
  uint32_t em = 0, vpos = 0;  // remaining non-zero elements of the current vector
  uint32_t n_idx = 0, n_c = 0, n_known = 0;
  bool n_valid = false;
  auto fetch = [&]() {
    if (em == 0 && vm != 0) {
      vpos = __ffs(vm) - 1;
      vm &= vm - 1;
      const uint4 v = *reinterpret_cast<const uint4*>(slot + vpos * 16);
      if (HOST)
        em = nz_bytes(v.x) | (nz_bytes(v.y) << 4) | (nz_bytes(v.z) << 8) | (nz_bytes(v.w) << 12);
      else
        em = min(v.x, 1u) | (min(v.y, 1u) << 1) | (min(v.z, 1u) << 2) | (min(v.w, 1u) << 3);
    }
    n_valid = em != 0;
    if (n_valid) {
      const uint32_t k = __ffs(em) - 1;
      em &= em - 1;
      if (HOST) {
        n_c = slot[vpos * 16 + k];
        n_idx = slot_base + vpos * 16 + k;
      } else {
        n_c = *reinterpret_cast<const uint32_t*>(slot + vpos * 16 + k * 4);
        n_idx = slot_base + vpos * 4 + k;
      }
      n_known = VSMEM ? (uint32_t)virgin[n_idx] : (uint32_t)__ldg(virgin + n_idx);
    }
  };
  fetch();
  while (__any_sync(0xffffffffu, n_valid)) {
    const bool valid = n_valid;
    const uint32_t idx = n_idx, c = n_c, known = n_known;
    fetch();
    if (valid) st.visit(idx, HOST ? hfz_class_host(c) : hfz_class_device(c), known, first, e, classed_row);
  }
}

template <int REC_CT, int ROW, bool VSMEM, bool CLASSED>
__global__ void __launch_bounds__(ROW >= 512 ? 320 : 640, 1) hfz_k_scan(const ScanParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  using C = RowCfg<ROW>;
  constexpr int LB = C::kLoads / 2;  // loads per register buffer
  constexpr int G = C::kGroup;  // maps per warp and group
  constexpr int WARP_SMEM = G * C::kSlot + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const uint64_t rec = REC_CT ? (uint64_t)REC_CT : p.rec_bytes;
  uint8_t* s_virgin = smem;
  uint8_t* s_buf = smem + (VSMEM ? p.S : 0) + (size_t)warp * WARP_SMEM;
  uint64_t* bar_virgin =
      reinterpret_cast<uint64_t*>(smem + (VSMEM ? p.S : 0) + (size_t)nwarps * WARP_SMEM);
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(s_buf + G * C::kSlot);  // [32] u32 per warp

  if (VSMEM) {
    if (threadIdx.x == 0) {
      hfz_mbar_init(bar_virgin, 1);
      hfz_fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // V0 -> shared memory with TMA bulk copies (SASS: UBLKCP), kept in L2 for the other CTAs
      const uint64_t pol = hfz_policy_evict_last();
      hfz_mbar_expect_tx(bar_virgin, p.S);
      for (uint32_t off = 0; off < p.S; off += 16384u) {
        const uint32_t n = p.S - off < 16384u ? p.S - off : 16384u;
        hfz_bulk_g2s_stream(s_virgin + off, p.v0 + off, n, bar_virgin, pol);
      }
    }
  }
  const uint8_t* virgin = VSMEM ? s_virgin : p.v0;
  bool virgin_ready = !VSMEM;

  // even split of the batch over all warps of the grid
  // Work split: every active warp gets g full groups of 32 maps (g = the fewest groups per warp
  // that cover the batch); a partial group costs as much as a full one (absent maps alias the
  // last one), so warps are left idle rather than given a few maps each.  Only the last active
  // warp sees a partial group.
  const uint64_t Wall = (uint64_t)gridDim.x * nwarps;
  const uint64_t groups = (p.n_exec + G - 1) / G;
  const uint64_t g = (groups + Wall - 1) / Wall;
  const uint64_t wg = (uint64_t)warp * gridDim.x + blockIdx.x;
  const uint64_t start = wg * g * G < p.n_exec ? wg * g * G : p.n_exec;
  const uint64_t stop = (wg + 1) * g * G < p.n_exec ? (wg + 1) * g * G : p.n_exec;
  const uint64_t cnt = stop - start;
  const uint32_t rows_host = p.H / ROW;
  const uint32_t rows = (uint32_t)(rec / ROW);
  const uint8_t* my_slot = s_buf + lane * C::kSlot;
  // lane -> (map within load, 16-byte unit within the map's chunk)
  const uint32_t sub = lane / C::kLanesPerMap, unit = lane % C::kLanesPerMap;
  uint8_t* scat = s_buf + sub * C::kSlot + unit * 16;

  for (uint64_t base = start; base < start + cnt; base += G) {
    const uint32_t nm = (uint32_t)min((uint64_t)G, start + cnt - base);
    const bool valid = (uint32_t)lane < nm;
    const uint64_t e64 = base + lane;
    const uint32_t e = (uint32_t)e64;
    uint8_t* classed_row = CLASSED ? p.classed + e64 * p.S : nullptr;
    // lane's source for load i: map (i*kMapsPerLoad + sub), unit `unit`
    const uint8_t* gsrc = p.raw + (base + sub) * rec + unit * 16;

    Lane<VSMEM, CLASSED> st;
    st.hf = HFZ_FNV_OFFSET;
    st.hs = HFZ_FNV_OFFSET;
    st.nnz = 0;

    // maps >= nm of a partial group alias the group's last map: always in bounds, their
    // votes are masked off below and their lanes never run phase B.
    const uint32_t last = nm - 1;
    auto run = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      uint4 A[LB], B[LB];
      auto load = [&](uint4* X, uint32_t row, int half) {
        const uint8_t* src = gsrc + (size_t)row * ROW;
#pragma unroll
        for (int i = 0; i < LB; ++i) {
          const uint32_t li = half * LB + i;                                    // load index within the row
          const uint32_t m0 = li * C::kMapsPerLoad / C::kLoadsPerMap;           // first map of this load
          constexpr uint32_t kPartMask = C::kLoadsPerMap - 1;
          const uint32_t part = (li & kPartMask) * 512;                         // 512-byte part of the map's row
          if (FULL) {
            X[i] = hfz_ldg_stream(reinterpret_cast<const uint4*>(src + (size_t)m0 * rec + part));
          } else {
            const uint32_t m = min(m0 + sub, last) - sub;  // clamp to the last map of the group
            X[i] = hfz_ldg_stream(reinterpret_cast<const uint4*>(src + (int64_t)(int32_t)m * (int64_t)rec + part));
          }
        }
      };
      auto scatter = [&](const uint4* X, int half) {
#pragma unroll
        for (int i = 0; i < LB; ++i) {
          const uint32_t li = half * LB + i;
          const uint32_t m0 = li * C::kMapsPerLoad / C::kLoadsPerMap;
          constexpr uint32_t kPartMask = C::kLoadsPerMap - 1;
          const uint32_t part = (li & kPartMask) * 512;
          bool nz = (X[i].x | X[i].y | X[i].z | X[i].w) != 0u;
          if (!FULL) nz = nz && (m0 + sub < nm);
          const uint32_t b = __ballot_sync(0xffffffffu, nz);
          if (lane == 0) {
            if (C::kMapsPerLoad == 1) {
              s_mask[li] = b;  // mask of (map m0, part): lane m0 reads s_mask[m0 * kLoadsPerMap + part]
            } else {
              *reinterpret_cast<uint2*>(s_mask + m0) = make_uint2(b & 0xffffu, b >> 16);
            }
          }
          if (nz) *reinterpret_cast<uint4*>(scat + m0 * C::kSlot + part) = X[i];
        }
      };
      // L2 prefetch of the row after next (32 maps x ROW bytes, one 128-byte line per lane-step)
      constexpr int PF_LINES = G * ROW / 128;  // lines per row
      const uint32_t pf_map = (uint32_t)lane / (ROW / 128), pf_off = ((uint32_t)lane % (ROW / 128)) * 128;
      auto prefetch = [&](uint32_t row) {
        if (p.prefetch && row < rows) {
#pragma unroll
          for (int j = 0; j < PF_LINES / 32; ++j) {
            const uint32_t m = pf_map + j * (32 / (ROW / 128));
            if (FULL || m < nm)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(p.raw + (base + m) * rec + pf_off +
                                                            (size_t)row * ROW));
          }
        }
      };

      prefetch(1);
      load(A, 0, 0);
      if (!virgin_ready) {
        hfz_mbar_wait(bar_virgin, 0);
        virgin_ready = true;
      }
      for (uint32_t r = 0; r < rows; ++r) {
        load(B, r, 1);
        prefetch(r + 2);
        scatter(A, 0);
        load(A, r + 1 < rows ? r + 1 : r, 0);  // unconditional (last one reloads row r, unused)
        scatter(B, 1);
        __syncwarp();
        if (C::kLoadsPerMap == 1) {
          uint32_t vm = s_mask[lane];
          if (!FULL && !valid) vm = 0;  // no branch on `valid`: idle lanes just see an empty mask
          if (r < rows_host)
            phase_b<true, ROW, VSMEM, CLASSED>(my_slot, vm, r * ROW, st, virgin, p.first, e, classed_row);
          else
            phase_b<false, ROW, VSMEM, CLASSED>(my_slot, vm, p.H + (r - rows_host) * (ROW / 4), st,
                                                virgin, p.first, e, classed_row);
        } else {
          // 1,024-byte rows: lane m < 16 walks the two 512-byte parts of ITS map's row one after the other
#pragma unroll
          for (int part = 0; part < C::kLoadsPerMap; ++part) {
            uint32_t vm = s_mask[(lane & (G - 1)) * C::kLoadsPerMap + part];
            if (!valid) vm = 0;
            if (r < rows_host)
              phase_b<true, ROW, VSMEM, CLASSED>(my_slot + part * 512, vm, r * ROW + part * 512, st, virgin, p.first, e,
                                                 classed_row);
            else
              phase_b<false, ROW, VSMEM, CLASSED>(my_slot + part * 512, vm, p.H + (r - rows_host) * (ROW / 4) + part * 128,
                                                  st, virgin, p.first, e, classed_row);
          }
        }
        __syncwarp();
      }
    };
    if (nm == G)
      run(std::true_type{});
    else
      run(std::false_type{});

    if (valid) {
      p.sig_full[e64] = st.hf;
      p.sig_simple[e64] = st.hs;
      if (p.nnz) p.nnz[e64] = st.nnz;
    }
  }
  if (!virgin_ready) hfz_mbar_wait(bar_virgin, 0);  // never leave the bulk copy in flight
}

// ---------------------------------------------------------------------------
// K2 scan for MEDIUM batches ("pipelined lane-per-map").  With only a few 32-map groups per SM
// the kernel above is latency-bound: the warp that owns a group issues a row's loads, waits for
// them, scatters, and only then runs the 32 FNV chains over that row.  Here the two halves are
// split between warps of a TEAM that owns one group: P producer warps stream the group's rows
// (row r by producer r % P: 32 maps x ROW bytes, coalesced 128-bit loads, ballot, scatter of the
// non-zero vectors into ring slot r % P in shared memory) and ONE consumer warp runs phase B --
// the serial chains -- row after row without ever waiting for HBM.  Full/empty hand-over per
// ring slot through mbarriers.  A CTA holds G teams; per-group latency drops from
// rows x (load latency + phase B) to rows x phase B.
template <int REC_CT, int ROW, int P, bool VSMEM, bool CLASSED>
__global__ void __launch_bounds__(ROW == 512 ? 320 : 640, 1) hfz_k_scan_pipe(const ScanParams p, const int G) {
  extern __shared__ __align__(128) uint8_t smem[];
  using C = RowCfg<ROW>;
  constexpr int LB = C::kLoads / 2;
  constexpr int SLOT = 32 * C::kSlot + 128;  // one row of a group: 32 padded lane slots + 32 masks
  constexpr int TEAM = 1 + P;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp / TEAM, role = warp % TEAM;
  const uint64_t rec = REC_CT ? (uint64_t)REC_CT : p.rec_bytes;
  uint8_t* s_virgin = smem;
  uint8_t* s_ring = smem + (VSMEM ? p.S : 0) + (size_t)g * P * SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (VSMEM ? p.S : 0) + (size_t)G * P * SLOT);
  uint64_t* bar_virgin = bars;
  uint64_t* full = bars + 1 + (size_t)g * 2 * P;
  uint64_t* empty = full + P;
  if (threadIdx.x == 0) {
    hfz_mbar_init(bar_virgin, 1);
    for (int i = 0; i < G * 2 * P; ++i) hfz_mbar_init(bars + 1 + i, 32);
    hfz_fence_barrier_init();
  }
  __syncthreads();
  if (VSMEM && threadIdx.x == 0) {  // thread 0 = consumer lane of team 0, whose group always exists
    const uint64_t pol = hfz_policy_evict_last();
    hfz_mbar_expect_tx(bar_virgin, p.S);
    for (uint32_t off = 0; off < p.S; off += 16384u) {
      const uint32_t n = p.S - off < 16384u ? p.S - off : 16384u;
      hfz_bulk_g2s_stream(s_virgin + off, p.v0 + off, n, bar_virgin, pol);
    }
  }
  const uint64_t base = ((uint64_t)g * gridDim.x + blockIdx.x) * 32;  // team g of CTA b owns group g * grid + b
  if (base >= p.n_exec) return;
  const uint32_t nm = (uint32_t)min((uint64_t)32, p.n_exec - base);
  const uint32_t rows = (uint32_t)(rec / ROW), rows_host = p.H / ROW;

  if (role != 0) {
    // ---- producer: rows pr, pr + P, ... into ring slot pr
    const int pr = role - 1;
    uint8_t* slot = s_ring + (size_t)pr * SLOT;
    uint32_t* s_mask = reinterpret_cast<uint32_t*>(slot + 32 * C::kSlot);
    const uint32_t sub = lane / C::kLanesPerMap, unit = lane % C::kLanesPerMap;
    uint8_t* scat = slot + sub * C::kSlot + unit * 16;
    const uint8_t* gsrc = p.raw + (base + sub) * rec + unit * 16;
    const uint32_t last = nm - 1;
    auto run = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      uint4 A[LB], B[LB];
      auto load = [&](uint4* X, uint32_t row, int half) {
        const uint8_t* src = gsrc + (size_t)row * ROW;
#pragma unroll
        for (int i = 0; i < LB; ++i) {
          const uint32_t m0 = (half * LB + i) * C::kMapsPerLoad;
          if (FULL) {
            X[i] = hfz_ldg_stream(reinterpret_cast<const uint4*>(src + (size_t)m0 * rec));
          } else {  // maps >= nm alias the group's last map; their votes are masked below
            const uint32_t m = min(m0 + sub, last) - sub;
            X[i] = hfz_ldg_stream(reinterpret_cast<const uint4*>(src + (int64_t)(int32_t)m * (int64_t)rec));
          }
        }
      };
      auto scatter = [&](const uint4* X, int half) {
#pragma unroll
        for (int i = 0; i < LB; ++i) {
          const uint32_t m0 = (half * LB + i) * C::kMapsPerLoad;
          bool nz = (X[i].x | X[i].y | X[i].z | X[i].w) != 0u;
          if (!FULL) nz = nz && (m0 + sub < nm);
          const uint32_t b = __ballot_sync(0xffffffffu, nz);
          if (lane == 0) {
            if (C::kMapsPerLoad == 1)
              s_mask[m0] = b;
            else
              *reinterpret_cast<uint2*>(s_mask + m0) = make_uint2(b & 0xffffu, b >> 16);
          }
          if (nz) *reinterpret_cast<uint4*>(scat + m0 * C::kSlot) = X[i];
        }
      };
      uint32_t it = 0;
      for (uint32_t r = pr; r < rows; r += P, ++it) {
        load(A, r, 0);
        load(B, r, 1);
        if (it) hfz_mbar_wait(&empty[pr], (it - 1) & 1u);  // the consumer is done with the slot's previous row
        scatter(A, 0);
        scatter(B, 1);
        hfz_mbar_arrive(&full[pr]);
      }
    };
    if (nm == 32)
      run(std::true_type{});
    else
      run(std::false_type{});
    return;
  }

  // ---- consumer: lane m runs map m's chains over the rows in order
  const bool valid = (uint32_t)lane < nm;
  const uint64_t e64 = base + lane;
  const uint32_t e = (uint32_t)e64;
  uint8_t* classed_row = CLASSED ? p.classed + e64 * p.S : nullptr;
  Lane<VSMEM, CLASSED> st;
  st.hf = HFZ_FNV_OFFSET;
  st.hs = HFZ_FNV_OFFSET;
  st.nnz = 0;
  if (VSMEM) hfz_mbar_wait(bar_virgin, 0);
  const uint8_t* virgin = VSMEM ? s_virgin : p.v0;
  for (uint32_t r = 0; r < rows; ++r) {
    const uint32_t s = r % P, it = r / P;
    const uint8_t* slot = s_ring + (size_t)s * SLOT;
    hfz_mbar_wait(&full[s], it & 1u);
    uint32_t vm = reinterpret_cast<const uint32_t*>(slot + 32 * C::kSlot)[lane];
    if (!valid) vm = 0;
    const uint8_t* my_slot = slot + lane * C::kSlot;
    if (r < rows_host)
      phase_b<true, ROW, VSMEM, CLASSED>(my_slot, vm, r * ROW, st, virgin, p.first, e, classed_row);
    else
      phase_b<false, ROW, VSMEM, CLASSED>(my_slot, vm, p.H + (r - rows_host) * (ROW / 4), st, virgin,
                                          p.first, e, classed_row);
    hfz_mbar_arrive(&empty[s]);
  }
  if (valid) {
    p.sig_full[e64] = st.hf;
    p.sig_simple[e64] = st.hs;
    if (p.nnz) p.nnz[e64] = st.nnz;
  }
}

// ---------------------------------------------------------------------------
// K2 scan for SMALL batches ("warp-per-map").  With fewer maps than ~6 per warp of the grid the
// lane-per-map kernel above is latency-bound (one warp walks 320+ rows serially).  Here every
// warp owns ONE map: the 32 lanes stream it coalesced and compact the non-zero slots, in index
// order, into a per-warp shared list (classification, virgin test and first-occurrence update
// happen in parallel on the way); then lanes 0 and 1 run the Full and the Simple FNV chain over
// the list.  ~5x more instructions per map than lane-per-map, but the latency of a batch drops
// from rows x row-latency to one map's chain (~20 us).
constexpr uint32_t kListCap = 2048;  // entries per warp: idx (24 bits) | rung << 24

template <bool VSMEM, bool CLASSED>
__global__ void __launch_bounds__(512, 1) hfz_k_scan_wpm(const ScanParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  uint8_t* s_virgin = smem;
  uint32_t* list = reinterpret_cast<uint32_t*>(smem + (VSMEM ? p.S : 0)) + (size_t)warp * kListCap;
  uint64_t* bar_virgin =
      reinterpret_cast<uint64_t*>(smem + (VSMEM ? p.S : 0) + (size_t)nwarps * kListCap * 4);
  if (VSMEM) {
    if (threadIdx.x == 0) {
      hfz_mbar_init(bar_virgin, 1);
      hfz_fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t pol = hfz_policy_evict_last();
      hfz_mbar_expect_tx(bar_virgin, p.S);
      for (uint32_t off = 0; off < p.S; off += 16384u) {
        const uint32_t n = p.S - off < 16384u ? p.S - off : 16384u;
        hfz_bulk_g2s_stream(s_virgin + off, p.v0 + off, n, bar_virgin, pol);
      }
    }
    hfz_mbar_wait(bar_virgin, 0);
  }
  const uint8_t* virgin = VSMEM ? s_virgin : p.v0;
  const uint32_t lane_lt = (1u << lane) - 1u;

  for (uint64_t e64 = (uint64_t)blockIdx.x * nwarps + warp; e64 < p.n_exec;
       e64 += (uint64_t)gridDim.x * nwarps) {
    const uint32_t e = (uint32_t)e64;
    const uint4* src = reinterpret_cast<const uint4*>(p.raw + e64 * p.rec_bytes);
    uint8_t* classed_row = CLASSED ? p.classed + e64 * p.S : nullptr;
    uint64_t h = HFZ_FNV_OFFSET;  // lane 0: Full chain, lane 1: Simple chain
    uint32_t fill = 0, nnz = 0;

    auto drain = [&]() {
      __syncwarp();
      if (lane < 2) {
#pragma unroll 4
        for (uint32_t i = 0; i < fill; ++i) {
          const uint32_t en = list[i];
          const uint32_t idx = en & 0xffffffu;
          h = hfz_fnv(hfz_fnv(h, idx & 0xffu), (idx >> 8) & 0xffu);
          if (lane == 0) h = hfz_fnv(h, 1u << (en >> 24));
        }
      }
      fill = 0;
      __syncwarp();
    };
    // one element (count c at logical slot idx): everything except the hash chains
    auto element = [&](uint32_t idx, uint32_t klass, uint32_t pos) {
      list[pos] = idx | ((31 - __clz(klass)) << 24);
      const uint32_t known = VSMEM ? (uint32_t)virgin[idx] : (uint32_t)__ldg(virgin + idx);
      if (klass & ~known) note_first(p.first + (size_t)idx * 8 + (31 - __clz(klass)), e);
      if (CLASSED) classed_row[idx] = (uint8_t)klass;
    };

    const uint32_t host_vecs = p.H / 16, total_vecs = (uint32_t)(p.rec_bytes / 16);
    auto load8 = [&](uint4* x, uint32_t v0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t v = v0 + j * 32 + lane;
        x[j] = v < total_vecs ? hfz_ldg_stream(src + v) : make_uint4(0, 0, 0, 0);
      }
    };
    auto process8 = [&](const uint4* x, uint32_t v0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t vb = v0 + j * 32;  // first vector of this warp-wide load (uniform)
        if (vb < total_vecs) {
          const bool host = vb < host_vecs;  // H is a multiple of 512: a load never straddles the halves
          const uint32_t w[4] = {x[j].x, x[j].y, x[j].z, x[j].w};
          uint32_t c;
          if (host)
            c = __popc(nz_bytes(w[0])) + __popc(nz_bytes(w[1])) + __popc(nz_bytes(w[2])) + __popc(nz_bytes(w[3]));
          else
            c = (w[0] != 0u) + (w[1] != 0u) + (w[2] != 0u) + (w[3] != 0u);
          if (__any_sync(0xffffffffu, c != 0u)) {
            // warp-wide exclusive prefix sum of the per-lane element counts
            uint32_t inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
              if (lane >= d) inc += o;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            if (fill + tot > kListCap) drain();
            uint32_t pos = fill + inc - c;
            if (c) {
              const uint32_t v = vb + lane;
              if (host) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  uint32_t bm = nz_bytes(w[k]);
                  while (bm) {
                    const uint32_t b = __ffs(bm) - 1;
                    bm &= bm - 1;
                    element(v * 16 + k * 4 + b, hfz_class_host((w[k] >> (8 * b)) & 0xffu), pos++);
                  }
                }
              } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  if (w[k]) element(p.H + (v - host_vecs) * 4 + k, hfz_class_device(w[k]), pos++);
              }
            }
            fill += tot;
            nnz += tot;
          }
        }
      }
    };
    uint4 xa[8], xb[8];
    load8(xa, 0);
    for (uint32_t v0 = 0; v0 < total_vecs; v0 += 2 * 256) {
      load8(xb, v0 + 256);
      process8(xa, v0);
      load8(xa, v0 + 512);
      process8(xb, v0 + 256);
    }
    drain();
    const uint64_t h_simple = __shfl_sync(0xffffffffu, h, 1);
    if (lane == 0) {
      p.sig_full[e64] = h;
      p.sig_simple[e64] = h_simple;
      if (p.nnz) p.nnz[e64] = nnz;
    }
  }
}

// ---------------------------------------------------------------------------
// novelty delta of this rank: D[s] = OR of class bits whose first-occurrence entry is set
__global__ void hfz_k_delta(const uint32_t* __restrict__ first, uint8_t* __restrict__ delta,
                            uint32_t S) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const uint4* f = reinterpret_cast<const uint4*>(first + (size_t)s * 8);
  const uint4 a = f[0], b = f[1];
  const uint32_t d = (a.x != kNone) | ((a.y != kNone) << 1) | ((a.z != kNone) << 2) |
                     ((a.w != kNone) << 3) | ((b.x != kNone) << 4) | ((b.y != kNone) << 5) |
                     ((b.z != kNone) << 6) | ((b.w != kNone) << 7);
  delta[s] = (uint8_t)d;
}

// ---------------------------------------------------------------------------
// K4: virgin |= D_0 | D_1 | ... in fixed rank order; prior_out = virgin before D_rank;
// edge counters += slots that turned non-zero, split by half (VirginMap::observe).
__global__ void hfz_k_merge(uint8_t* __restrict__ virgin, const uint8_t* __restrict__ deltas,
                            uint32_t n_ranks, uint32_t rank, uint8_t* __restrict__ prior_out,
                            unsigned long long* __restrict__ edge_counts, uint32_t S, uint32_t H) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;  // 16-byte vector index
  uint32_t newh = 0, newd = 0;
  if (v < S / 16) {
    uint4 acc = reinterpret_cast<uint4*>(virgin)[v];
    const uint4 old = acc;
    for (uint32_t q = 0; q < n_ranks; ++q) {
      if (prior_out && q == rank) reinterpret_cast<uint4*>(prior_out)[v] = acc;
      const uint4 d = reinterpret_cast<const uint4*>(deltas + (size_t)q * S)[v];
      acc.x |= d.x; acc.y |= d.y; acc.z |= d.z; acc.w |= d.w;
    }
    if (prior_out && rank >= n_ranks) reinterpret_cast<uint4*>(prior_out)[v] = acc;
    reinterpret_cast<uint4*>(virgin)[v] = acc;
    const uint32_t turned = __popc(nz_bytes(acc.x) & ~nz_bytes(old.x)) +
                            __popc(nz_bytes(acc.y) & ~nz_bytes(old.y)) +
                            __popc(nz_bytes(acc.z) & ~nz_bytes(old.z)) +
                            __popc(nz_bytes(acc.w) & ~nz_bytes(old.w));
    if (v * 16 < H) newh = turned; else newd = turned;
  }
  newh = __reduce_add_sync(0xffffffffu, newh);
  newd = __reduce_add_sync(0xffffffffu, newd);
  if ((threadIdx.x & 31) == 0) {
    if (newh) atomicAdd(edge_counts + 0, (unsigned long long)newh);
    if (newd) atomicAdd(edge_counts + 1, (unsigned long long)newd);
  }
}

// K4 over peer memory: the same ordered merge, but every rank's delta is loaded from where it was
// produced -- ptrs.p[q] is rank q's delta, own or peer-mapped (NVLink) device memory -- instead
// of from an allgathered staging copy.  64 KB per rank: one 128-bit load per thread and rank.
constexpr int kMaxPeers = 16;
struct PeerPtrs {
  const uint8_t* p[kMaxPeers];
};

__global__ void hfz_k_merge_peers(uint8_t* __restrict__ virgin, const PeerPtrs ptrs, uint32_t n_ranks, uint32_t rank,
                                  uint8_t* __restrict__ prior_out, unsigned long long* __restrict__ edge_counts,
                                  uint32_t S, uint32_t H) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;  // 16-byte vector index
  uint32_t newh = 0, newd = 0;
  if (v < S / 16) {
    uint4 acc = reinterpret_cast<uint4*>(virgin)[v];
    const uint4 old = acc;
    for (uint32_t q = 0; q < n_ranks; ++q) {
      if (q == rank) reinterpret_cast<uint4*>(prior_out)[v] = acc;
      const uint4 d = reinterpret_cast<const uint4*>(ptrs.p[q])[v];
      acc.x |= d.x; acc.y |= d.y; acc.z |= d.z; acc.w |= d.w;
    }
    reinterpret_cast<uint4*>(virgin)[v] = acc;
    const uint32_t turned = __popc(nz_bytes(acc.x) & ~nz_bytes(old.x)) + __popc(nz_bytes(acc.y) & ~nz_bytes(old.y)) +
                            __popc(nz_bytes(acc.z) & ~nz_bytes(old.z)) + __popc(nz_bytes(acc.w) & ~nz_bytes(old.w));
    if (v * 16 < H) newh = turned; else newd = turned;
  }
  newh = __reduce_add_sync(0xffffffffu, newh);
  newd = __reduce_add_sync(0xffffffffu, newd);
  if ((threadIdx.x & 31) == 0) {
    if (newh) atomicAdd(edge_counts + 0, (unsigned long long)newh);
    if (newd) atomicAdd(edge_counts + 1, (unsigned long long)newd);
  }
}

// ---------------------------------------------------------------------------
// K2b: the Admit codes of ALL execs straight from the first-occurrence table -- no candidate is
// walked, no map or list is read again.  Entry (slot, bit) = e names the first exec of the batch that shows
// class bit `bit` on `slot`, recorded only when the bit is not in V0.  With P = the virgin map before this
// rank's first exec (V0 | the deltas of the ranks before it):
//   bit in P[slot]                       -> an earlier rank had it: nothing;
//   P[slot] == 0 and e == min over bits  -> exec e is the first ever on the slot: NewEdges (2);
//   otherwise                            -> exec e adds a class to a known slot: NewCounts (1);
// and Admit[e] is the maximum over the entries that name e (has_new_bits, src/coverage.cpp:74-87: the result is
// the max over the map's slots).  One thread per slot: 32 bytes of table + 1 byte of P each (2 MB for the
// 64 KB map, L2-resident: the scan has just written it), whatever the number of candidate execs -- a batch
// folded into an empty virgin map costs what a warm one does.
// Flags are ORed into a per-exec u32 (context scratch, zero between calls); hfz_k_admit_codes turns them into
// the Admit bytes and re-zeroes them.
__device__ __forceinline__ void resolve_slot(const uint4 a, const uint4 b, uint32_t pr, uint32_t* __restrict__ flags) {
  if ((a.x & a.y & a.z & a.w & b.x & b.y & b.z & b.w) == kNone) return;  // no exec showed anything new here
  const uint32_t lo = min(min(min(a.x, a.y), min(a.z, a.w)), min(min(b.x, b.y), min(b.z, b.w)));
  const uint32_t ent[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int bit = 0; bit < 8; ++bit) {
    const uint32_t e = ent[bit];
    if (e == kNone || ((pr >> bit) & 1u)) continue;
    const uint32_t code = (pr == 0 && e == lo) ? 2u : 1u;
    const uint32_t cur = __ldcg(flags + e);  // an exec that opens many slots: one atomic, then reads
    if (!(cur & (2u | code))) atomicOr(flags + e, code);
  }
}

__global__ void __launch_bounds__(256) hfz_k_resolve_table(const uint32_t* __restrict__ first,
                                                           const uint8_t* __restrict__ prior, uint32_t S,
                                                           uint32_t* __restrict__ flags) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const uint4* f = reinterpret_cast<const uint4*>(first + (size_t)s * 8);
  resolve_slot(__ldcg(f), __ldcg(f + 1), __ldg(prior + s), flags);
}

// One word (4 slots) of the single-rank fold, everything the table says about them in one read: delta word,
// virgin |= delta, the slots that turned non-zero, and -- the virgin word as it stood being P -- the Admit
// flags of the execs the slots' entries name.  `fold` = false: the delta word only (multi-rank scan half).
__device__ __forceinline__ void fold_word(const uint32_t* __restrict__ first, uint64_t t, bool fold, uint8_t* virgin,
                                          uint8_t* __restrict__ delta_out, uint32_t* __restrict__ flags, uint32_t H,
                                          uint32_t& newh, uint32_t& newd) {
  const uint4* f = reinterpret_cast<const uint4*>(first + t * 32);
  uint32_t* vw = reinterpret_cast<uint32_t*>(virgin) + t;
  const uint32_t old = fold ? *vw : 0u;
  uint32_t d = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 a = __ldcg(f + 2 * q), b = __ldcg(f + 2 * q + 1);
    const uint32_t byte = (a.x != kNone) | ((a.y != kNone) << 1) | ((a.z != kNone) << 2) | ((a.w != kNone) << 3) |
                          ((b.x != kNone) << 4) | ((b.y != kNone) << 5) | ((b.z != kNone) << 6) | ((b.w != kNone) << 7);
    d |= byte << (8 * q);
    if (fold) resolve_slot(a, b, (old >> (8 * q)) & 0xffu, flags);
  }
  if (delta_out) reinterpret_cast<uint32_t*>(delta_out)[t] = d;
  if (fold) {
    const uint32_t nw = old | d;
    if (nw != old) *vw = nw;
    const uint32_t turned = __popc(nz_bytes(nw) & ~nz_bytes(old));
    if (t * 4 < H) newh += turned; else newd += turned;
  }
}

// delta + merge + resolve of a single-rank fold in one pass over the table (hfz_feedback_batch and the list
// folds; the multi-rank path keeps hfz_k_delta / hfz_k_merge / hfz_k_resolve_table around its exchange step)
__global__ void __launch_bounds__(256) hfz_k_fold_single(const uint32_t* __restrict__ first, uint8_t* virgin,
                                                         uint32_t* __restrict__ flags,
                                                         unsigned long long* __restrict__ edge_counts, uint32_t S,
                                                         uint32_t H) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;  // word index
  uint32_t newh = 0, newd = 0;
  if (t < S / 4) fold_word(first, t, true, virgin, nullptr, flags, H, newh, newd);
  newh = __reduce_add_sync(0xffffffffu, newh);
  newd = __reduce_add_sync(0xffffffffu, newd);
  if ((threadIdx.x & 31) == 0) {
    if (newh) atomicAdd(edge_counts + 0, (unsigned long long)newh);
    if (newd) atomicAdd(edge_counts + 1, (unsigned long long)newd);
  }
}

__global__ void __launch_bounds__(256) hfz_k_admit_codes(uint32_t* __restrict__ flags, uint8_t* __restrict__ admit,
                                                         uint64_t n_exec) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_exec) return;
  const uint32_t f = flags[e];
  admit[e] = (f & 2u) ? 2 : (uint8_t)(f & 1u);
  if (f) flags[e] = 0;
}

// ---------------------------------------------------------------------------
// Sparse-native scan: the fold on touched-slot lists without ever building a dense record.
//   rank   one warp per exec: the (slot, count) pairs arrive in any order; a bitmap of the map's
//          slots in shared memory (S bits) + a popcount prefix give every slot its RANK among the
//          exec's non-zero slots, so the pairs are written out as `slot | rung << 24` in ascending
//          slot order without a sort; classification, the virgin test against the TMA-staged
//          V0 and the first-occurrence update ride along;
//   chain  one lane per exec runs both FNV chains over its ordered list -- dense iterations, no
//          row-synchronous max over lanes as in the dense kernels.
// 65,536 execs (76 M pairs) take ~0.3 ms instead of ~10 ms through the dense staging buffer.
constexpr int kRankWarps = 18;  // 18 x (8 KB bitmap + 4 KB prefix + padding) = 225 KB for S = 65,536; V0 is read through L1 / L2

// shared memory of one warp of the rank kernel: padded bitmap, padded 16-bit prefix, lane bases + counter
__host__ __device__ constexpr size_t rank_warp_bytes(uint32_t words) {
  return ((size_t)(words + 32) * 4 + (size_t)(words + 64) * 2 + 256 + 15) / 16 * 16;
}

struct SparseParams {
  const uint2* pairs;       // wide pairs {slot, count}; may be null
  const uint64_t* off;
  const uint32_t* cpairs;   // compact pairs slot | count << 16; may be null
  const uint64_t* coff;
  int packed;               // packed lists: `pairs` / `off` are the host-half list -- 3-byte entries {slot lo, slot hi,
                            // count u8}, four per three words, every exec padded to a multiple of four (off in entries) --
                            // and `cpairs` the device-half list (slot - H) | min(count, 65536) << 15
  uint64_t n_exec;
  uint32_t S, H;
  const uint8_t* v0;
  uint32_t* first;
  uint32_t* sorted;
  uint32_t* cnt;
  uint8_t* classed;
  unsigned long long* bad;
};

__global__ void __launch_bounds__(kRankWarps * 32, 1) hfz_k_sparse_rank(const SparseParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t words = p.S / 32, per = words / 32;  // bitmap words, words per lane in the prefix pass
  const uint32_t per_shift = 31 - __clz(per);         // S is a power of two >= 1024
  // (Round 1 staged V0 in shared memory by TMA: 64 KB that held the CTA at 12 warps, and the kernel's
  // stalls are shared-memory round trips of the bitmap -- more warps hide them; V0's 64 KB stay hot in L2.)
  // In the prefix pass lane l walks ITS words [l * per, (l + 1) * per): a lane stride of `per` words puts all 32
  // lanes on one bank (91 % of the kernel's shared-memory wavefronts were conflicts of that pass).  One pad
  // word per lane segment (two for the 16-bit prefix array) makes the stride odd: word w lives at
  // w + (w >> per_shift), its prefix at w + 2 (w >> per_shift).
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem + (size_t)warp * rank_warp_bytes(words));
  uint16_t* pre = reinterpret_cast<uint16_t*>(bm + words + 32);
  uint32_t* lane_base = reinterpret_cast<uint32_t*>(pre + words + 64);  // [32]
  for (uint32_t i = lane; i < words + 32; i += 32) bm[i] = 0;
  __syncwarp();
  uint32_t nbad = 0;
  const uint32_t n_warps = blockDim.x >> 5;  // as many as the bitmaps leave room for (18 at 65,536 slots, 4 at 262,144)
  for (uint64_t e64 = (uint64_t)blockIdx.x * n_warps + warp; e64 < p.n_exec; e64 += (uint64_t)gridDim.x * n_warps) {
    const uint32_t e = (uint32_t)e64;
    // exec e owns wide pairs [b, t) and compact pairs [cb, ct); its ordered list starts at b + cb
    const uint64_t b = p.off ? p.off[e64] : 0, t = p.off ? p.off[e64 + 1] : 0;
    const uint64_t cb = p.coff ? p.coff[e64] : 0, ct = p.coff ? p.coff[e64 + 1] : 0;
    // calls f(slot, count) for every pair of the exec, four loads in flight per lane
    auto for_pairs = [&](auto&& f) {
      if (p.packed) {
        // host half: one group of four 3-byte entries (three aligned words) per lane and step
        const uint32_t* h3 = reinterpret_cast<const uint32_t*>(p.pairs);
        for (uint64_t g0 = b / 4; g0 < t / 4; g0 += 32) {
          const uint64_t g = g0 + lane;
          uint32_t w0 = 0, w1 = 0, w2 = 0;
          if (g < t / 4) {
            w0 = __ldg(h3 + 3 * g);
            w1 = __ldg(h3 + 3 * g + 1);
            w2 = __ldg(h3 + 3 * g + 2);
          }
          const uint32_t en[4] = {w0 & 0xffffffu, (w0 >> 24) | ((w1 & 0xffffu) << 8), (w1 >> 16) | ((w2 & 0xffu) << 16), w2 >> 8};
#pragma unroll
          for (int j = 0; j < 4; ++j) f(en[j] & 0xffffu, en[j] >> 16);
        }
        for (uint64_t i0 = cb; i0 < ct; i0 += 128) {
          uint32_t x[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t i = i0 + j * 32 + lane;
            x[j] = i < ct ? __ldg(p.cpairs + i) : 0u;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) f(p.H + (x[j] & 0x7fffu), x[j] >> 15);
        }
        return;
      }
      for (uint64_t i0 = b; i0 < t; i0 += 128) {
        uint2 x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t i = i0 + j * 32 + lane;
          x[j] = i < t ? __ldg(p.pairs + i) : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) f(x[j].x, x[j].y);
      }
      for (uint64_t i0 = cb; i0 < ct; i0 += 128) {
        uint32_t x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t i = i0 + j * 32 + lane;
          x[j] = i < ct ? __ldg(p.cpairs + i) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) f(x[j] & 0xffffu, x[j] >> 16);
      }
    };
    // pass 1: mark the slots (padding pairs are {0, 0}: count 0 = unvisited)
    for_pairs([&](uint32_t slot, uint32_t cnt_raw) {
      const uint32_t c = slot < p.H ? (cnt_raw & 0xffu) : cnt_raw;
      if (slot >= p.S) {
        ++nbad;
      } else if (c) {
        const uint32_t w = slot >> 5;
        atomicOr(&bm[w + (w >> per_shift)], 1u << (slot & 31));
      }
    });
    __syncwarp();
    // popcount prefix: lane l owns words [l * per, (l + 1) * per)
    uint32_t sum = 0;
    for (uint32_t k = 0; k < per; ++k) {
      const uint32_t w = lane * per + k;
      pre[w + 2 * lane] = (uint16_t)sum;
      sum += __popc(bm[w + lane]);
    }
    uint32_t inc = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += o;
    }
    lane_base[lane] = inc - sum;
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    __syncwarp();
    // pass 2: rank, classify, novelty, ordered write
    uint8_t* classed_row = p.classed ? p.classed + e64 * p.S : nullptr;
    uint32_t* out = p.sorted + b + cb;
    for_pairs([&](uint32_t slot, uint32_t cnt_raw) {
      if (slot >= p.S) return;
      const uint32_t c = slot < p.H ? (cnt_raw & 0xffu) : cnt_raw;
      if (!c) return;
      const uint32_t w = slot >> 5, seg = w >> per_shift;
      const uint32_t rank = lane_base[seg] + pre[w + 2 * seg] + __popc(bm[w + seg] & ((1u << (slot & 31)) - 1u));
      const uint32_t klass = slot < p.H ? hfz_class_host(c) : hfz_class_device(c);
      const uint32_t rung = 31 - __clz(klass);
      const uint32_t en = slot | (rung << 24);
      out[rank] = en;
      if (klass & ~(uint32_t)__ldg(p.v0 + slot)) note_first(p.first + (size_t)slot * 8 + rung, e);
      if (classed_row) classed_row[slot] = (uint8_t)klass;
    });
    __syncwarp();
    if (lane == 0) p.cnt[e64] = total;
    for (uint32_t i = lane; i < (words + 32) / 4; i += 32) reinterpret_cast<uint4*>(bm)[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();
  }
  nbad = __reduce_add_sync(0xffffffffu, nbad);
  if (lane == 0 && nbad && p.bad) atomicAdd(p.bad, (unsigned long long)nbad);
}

// Both FNV chains over `n` ordered entries (slot | rung << 24).  The next four entries are
// loaded BEFORE the chains of the current four run, so their latency (the lists usually sit in
// L2) hides behind the dependent multiplies.
__device__ __forceinline__ void chain_list(const uint32_t* __restrict__ list, uint32_t n, uint64_t& hf, uint64_t& hs) {
  auto step = [&](uint32_t en) {
    const uint32_t b0 = en & 0xffu, b1 = (en >> 8) & 0xffu;
    hf = hfz_fnv(hfz_fnv(hfz_fnv(hf, b0), b1), 1u << (en >> 24));
    hs = hfz_fnv(hfz_fnv(hs, b0), b1);
  };
  uint32_t cur[4], nxt[4];
  uint32_t i = 0;
  if (n >= 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k) cur[k] = __ldg(list + k);
    for (; i + 8 <= n; i += 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) nxt[k] = __ldg(list + i + 4 + k);
#pragma unroll
      for (int k = 0; k < 4; ++k) step(cur[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) cur[k] = nxt[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) step(cur[k]);
    i += 4;
  }
  for (; i < n; ++i) step(__ldg(list + i));
}

__global__ void __launch_bounds__(128) hfz_k_sparse_chain(const uint32_t* __restrict__ sorted,
                                                          const uint64_t* __restrict__ off,
                                                          const uint64_t* __restrict__ coff,
                                                          const uint32_t* __restrict__ cnt, uint64_t n_exec,
                                                          uint64_t* __restrict__ sig_full,
                                                          uint64_t* __restrict__ sig_simple,
                                                          uint32_t* __restrict__ nnz_out) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_exec) return;
  const uint32_t* list = sorted + (off ? off[e] : 0) + (coff ? coff[e] : 0);
  const uint32_t n = cnt[e];
  uint64_t hf = HFZ_FNV_OFFSET, hs = HFZ_FNV_OFFSET;
  chain_list(list, n, hf, hs);
  sig_full[e] = hf;
  sig_simple[e] = hs;
  if (nnz_out) nnz_out[e] = n;
}

// The same for SMALL batches (at most one exec per resident warp): one WARP per exec, both chains by the
// warp-parallel FNV of hfz_fnv.cuh over rounds of 1,024 entries staged in shared memory.  A lane
// running an exec's chains alone needs ~100 cycles per entry (2,110 entries of a 262,144-slot map:
// 0.24 ms however few execs there are); the warp needs ~850 instructions per 1,024 steps.
constexpr uint32_t kChainRoundSp = 1024;
constexpr int kChainWarps = 4;
__global__ void __launch_bounds__(kChainWarps * 32) hfz_k_sparse_chain_warp(const uint32_t* __restrict__ sorted,
                                                                            const uint64_t* __restrict__ off,
                                                                            const uint64_t* __restrict__ coff,
                                                                            const uint32_t* __restrict__ cnt, uint64_t n_exec,
                                                                            uint64_t* __restrict__ sig_full,
                                                                            uint64_t* __restrict__ sig_simple,
                                                                            uint32_t* __restrict__ nnz_out) {
  __shared__ __align__(16) uint32_t s_buf[kChainWarps][kChainRoundSp];
  __shared__ __align__(16) uint8_t s_stream[kChainWarps][3072 + 16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t e = (uint64_t)blockIdx.x * kChainWarps + warp;
  if (e >= n_exec) return;
  const uint32_t* list = sorted + (off ? off[e] : 0) + (coff ? coff[e] : 0);
  const uint32_t n = cnt[e];
  uint64_t hf = HFZ_FNV_OFFSET, hs = HFZ_FNV_OFFSET;
  for (uint32_t i0 = 0; i0 < n; i0 += kChainRoundSp) {
    const uint32_t m = n - i0 < kChainRoundSp ? n - i0 : kChainRoundSp;
    for (uint32_t i = lane; i < m; i += 32) s_buf[warp][i] = __ldg(list + i0 + i);
    __syncwarp();
    hf = pfnv::chain_entries<3>(hf, s_buf[warp], m, s_stream[warp], lane);
    hs = pfnv::chain_entries<2>(hs, s_buf[warp], m, s_stream[warp], lane);
    __syncwarp();
  }
  if (lane == 0) {
    sig_full[e] = hf;
    sig_simple[e] = hs;
    if (nnz_out) nnz_out[e] = n;
  }
}

// ---------------------------------------------------------------------------
// Two-stage scan of DENSE records for small and medium batches ("compact + chain").
//   compact  work item = (map, 16 KB piece of its record), one warp each: the piece is streamed
//            coalesced (4 x 128-bit loads in flight per lane), the non-zero slots are compacted IN
//            ORDER (warp scan of the per-lane element counts) as `slot | rung << 24` into the
//            piece's own slot range of a scratch list [n_exec][S] -- no offsets to compute, only
//            the used prefix of a range is ever touched; classification, the virgin test and the
//            first-occurrence update ride along;
//   chain    one lane per map walks its pieces' lists and runs both FNV chains.
// Nothing is row-synchronous and every warp of the grid has work from the first microsecond, so
// a batch costs its HBM time plus one map's chain (~50 us) instead of rows x row latency.
constexpr uint32_t kTsPiece = 16384;  // bytes per piece (divides H and 4H for H >= 16,384; halved otherwise)

struct CompactParams {
  const uint8_t* raw;
  uint64_t n_exec, rec_bytes;
  uint32_t S, H, piece, host_pieces, pieces;
  const uint8_t* v0;
  uint32_t* first;
  uint32_t* sorted;   // [n_exec][S]
  uint32_t* cnt;      // [n_exec][pieces]
  uint8_t* classed;
};

// one work item of the compact stage: (map, piece) by one warp.  `staged` = the piece already in
// shared memory (fused step: TMA bulk copy), or null = stream it from global memory.
__device__ __forceinline__ void compact_item(const CompactParams& p, uint64_t it, uint32_t lane,
                                             const uint4* staged = nullptr) {
  {
    const uint64_t e64 = it / p.pieces;
    const uint32_t pc = (uint32_t)(it - e64 * p.pieces), e = (uint32_t)e64;
    const bool host = pc < p.host_pieces;
    const uint32_t slot0 = host ? pc * p.piece : p.H + (pc - p.host_pieces) * (p.piece / 4);
    const uint4* src = reinterpret_cast<const uint4*>(p.raw + e64 * p.rec_bytes + (uint64_t)pc * p.piece);
    uint32_t* out = p.sorted + e64 * p.S + slot0;
    uint8_t* classed_row = p.classed ? p.classed + e64 * p.S : nullptr;
    uint32_t fill = 0;
    const uint32_t vecs = p.piece / 16;
    for (uint32_t v0 = 0; v0 < vecs; v0 += 128) {
      uint4 x[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t v = v0 + j * 32 + lane;
        x[j] = v < vecs ? (staged ? staged[v] : hfz_ldg_stream(src + v)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t w[4] = {x[j].x, x[j].y, x[j].z, x[j].w};
        // element mask of this lane's vector: 16 bits (host bytes) or 4 bits (device words)
        uint32_t m;
        if (host)
          m = nz_bytes(w[0]) | (nz_bytes(w[1]) << 4) | (nz_bytes(w[2]) << 8) | (nz_bytes(w[3]) << 12);
        else
          m = (w[0] != 0u) | ((w[1] != 0u) << 1) | ((w[2] != 0u) << 2) | ((w[3] != 0u) << 3);
        if (!__any_sync(0xffffffffu, m != 0u)) continue;
        const uint32_t c = __popc(m);
        uint32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += o;
        }
        uint32_t pos = fill + inc - c;
        fill += __shfl_sync(0xffffffffu, inc, 31);
        const uint32_t v = v0 + j * 32 + lane;
        while (m) {
          const uint32_t b = __ffs(m) - 1;
          m &= m - 1;
          uint32_t idx, klass;
          // word b >> 2 (host) / b (device) of the vector, by selects (no local-memory indexing)
          const uint32_t wi = host ? (b >> 2) : b;
          const uint32_t word = wi == 0 ? w[0] : (wi == 1 ? w[1] : (wi == 2 ? w[2] : w[3]));
          if (host) {
            idx = slot0 + v * 16 + b;
            klass = hfz_class_host((word >> (8 * (b & 3))) & 0xffu);
          } else {
            idx = slot0 + v * 4 + b;
            klass = hfz_class_device(word);
          }
          const uint32_t rung = 31 - __clz(klass);
          const uint32_t en = idx | (rung << 24);
          out[pos++] = en;
          if (klass & ~(uint32_t)__ldg(p.v0 + idx)) note_first(p.first + (size_t)idx * 8 + rung, e);
          if (classed_row) classed_row[idx] = (uint8_t)klass;
        }
      }
    }
    if (lane == 0) p.cnt[it] = fill;
  }
}

__global__ void __launch_bounds__(256) hfz_k_compact(const CompactParams p) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t items = p.n_exec * p.pieces;
  for (uint64_t it = warp; it < items; it += nwarps) compact_item(p, it, lane);
}

// one lane per map: chains over the map's piece lists, nnz
__global__ void __launch_bounds__(128) hfz_k_chain_pieces(const CompactParams p, uint64_t* __restrict__ sig_full,
                                                          uint64_t* __restrict__ sig_simple,
                                                          uint32_t* __restrict__ nnz_out) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.n_exec) return;
  uint64_t hf = HFZ_FNV_OFFSET, hs = HFZ_FNV_OFFSET;
  uint32_t nnz = 0;
  for (uint32_t pc = 0; pc < p.pieces; ++pc) {
    const uint32_t slot0 = pc < p.host_pieces ? pc * p.piece : p.H + (pc - p.host_pieces) * (p.piece / 4);
    const uint32_t* list = p.sorted + e * p.S + slot0;
    const uint32_t n = p.cnt[e * p.pieces + pc];
    nnz += n;
    chain_list(list, n, hf, hs);
  }
  sig_full[e] = hf;
  sig_simple[e] = hs;
  if (nnz_out) nnz_out[e] = nnz;
}

// ---------------------------------------------------------------------------
// Small batches as ONE cooperative launch ("fused step").  The two-stage path above is latency-
// bound by its launches: 7 kernels + 4 memsets for 26 us of HBM time at 1,024 maps.  Here the
// whole fold -- compact, chains, delta, ordered merge, resolve, Admit codes -- is one persistent
// kernel (one 768-thread CTA per SM, cooperative launch) with two grid-wide barriers, and nothing
// is memset between calls:
//   * the first-occurrence table is double-buffered: a call uses one table (all-ones on entry)
//     and scrubs the OTHER one, which the previous call left dirty, while it streams the maps;
//   * the per-exec Admit flags are zeroed again by the thread that turns them into codes.
//   phase 1   all warps: (map, piece) items -> ordered piece lists + first-occurrence updates
//   --- grid barrier ---
//   phase 2   by role: delta + merge + resolve (4 slots per thread: delta word from the table,
//             virgin |= delta, edge counters, and -- the virgin word as it stood being P -- the
//             Admit flags of the execs the slots' entries name, resolve_slot) | one warp per map:
//             both FNV chains over its piece lists (hfz_fnv.cuh)
//   --- grid barrier ---
//   phase 3   Admit flags -> codes, one thread per exec
// The scan and resolve halves can also be launched separately (multi-rank: the deltas of all ranks
// are exchanged in between); the resolve half then starts with the rank-ordered merge.
struct StepParams {
  CompactParams c;           // phase 1 (c.first = this call's table)
  uint32_t* first_prev;      // the other table, scrubbed to all-ones (scan half)
  uint64_t* sig_full;
  uint64_t* sig_simple;
  uint32_t* nnz;
  uint8_t* delta_out;        // this rank's novelty delta (S bytes)
  uint8_t* virgin;           // resolve half: virgin_inout
  uint8_t* prior;            // P_r
  unsigned long long* edge_counts;
  const uint8_t* deltas;     // n_ranks x S (== delta_out when fused)
  uint32_t n_ranks, rank;
  uint8_t* admit;
  uint32_t* flags;           // per-exec novelty flags of the table resolve (zero on entry, zero again on exit)
  int do_scan, do_resolve;
  unsigned long long* dbg;   // optional: [8] latest %globaltimer at each phase boundary (dev probe)
};

__device__ __forceinline__ void dbg_mark(const StepParams& p, int k) {
  if (p.dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (k == 0) atomicMin(p.dbg + 0, t); else atomicMax(p.dbg + k, t);
  }
}

__device__ __forceinline__ uint32_t piece_slot0(const CompactParams& c, uint32_t pc) {
  return pc < c.host_pieces ? pc * c.piece : c.H + (pc - c.host_pieces) * (c.piece / 4);
}

constexpr int kStepWarps = 24;
constexpr uint32_t kStepBuf = 8192;                 // shared memory per warp: two staging buffers of one piece (phase 1),
constexpr uint32_t kStepPiece = kStepBuf / 2;       //   then one list buffer of kStepCap entries (phase 2)
constexpr uint32_t kStepCap = kStepBuf / 4;
constexpr uint32_t kChainRound = 1024;              // entries per round of the signature chains (phase 2)

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(hfz_smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

constexpr uint32_t kDescCap = 256;  // element descriptors buffered per warp between two lane-parallel passes

constexpr size_t kStepSmem = (size_t)kStepWarps * (kStepBuf + kDescCap * 4 + 16);  // staging + descriptors + 2 mbarriers per warp

// Compaction of one staged piece, in two loops so that the expensive per-element work runs with
// all lanes busy: loop 1 (per 512-byte row: element masks, one warp scan) only drops a 4-byte
// descriptor `local slot | count << 12` per non-zero element into a shared buffer at its rank;
// loop 2 walks the buffer one element per lane: classification, virgin test, first-occurrence
// update, and the ordered list entries go out as coalesced stores.  (A 2 %-dense row has ~10
// non-zero elements spread over 32 lanes: doing the per-element work in loop 1 kept 5 of 32 lanes
// busy.)  Device counts are clipped at 65,536, the last rung boundary, to fit the descriptor.
__device__ __noinline__ void compact_staged_rows(const CompactParams& p, uint64_t it, uint32_t lane, const uint4* src,
                                                uint32_t* desc) {
  const uint64_t e64 = it / p.pieces;
  const uint32_t pc = (uint32_t)(it - e64 * p.pieces), e = (uint32_t)e64;
  const bool host = pc < p.host_pieces;
  const uint32_t slot0 = host ? pc * p.piece : p.H + (pc - p.host_pieces) * (p.piece / 4);
  uint32_t* out = p.sorted + e64 * p.S + slot0;
  uint8_t* classed_row = p.classed ? p.classed + e64 * p.S : nullptr;
  uint32_t fill = 0, nbuf = 0;
  const uint32_t vecs = p.piece / 16;
  auto element = [&](uint32_t idx, uint32_t cnt, uint32_t pos) {
    const uint32_t klass = host ? hfz_class_host(cnt) : hfz_class_device(cnt);
    const uint32_t rung = 31 - __clz(klass);
    const uint32_t en = idx | (rung << 24);
    out[pos] = en;
    if (klass & ~(uint32_t)__ldg(p.v0 + idx)) note_first(p.first + (size_t)idx * 8 + rung, e);
    if (classed_row) classed_row[idx] = (uint8_t)klass;
  };
  auto flush = [&]() {
    __syncwarp();
    for (uint32_t t = lane; t < nbuf; t += 32) {
      const uint32_t d = desc[t];
      element(slot0 + (d & 0xfffu), d >> 12, fill + t);
    }
    fill += nbuf;
    nbuf = 0;
    __syncwarp();
  };
  for (uint32_t v0 = 0; v0 < vecs; v0 += 32) {
    const uint32_t v = v0 + lane;
    const uint4 x = v < vecs ? src[v] : make_uint4(0, 0, 0, 0);
    uint32_t m;
    if (host)
      m = nz_bytes(x.x) | (nz_bytes(x.y) << 4) | (nz_bytes(x.z) << 8) | (nz_bytes(x.w) << 12);
    else
      m = (x.x != 0u) | ((x.y != 0u) << 1) | ((x.z != 0u) << 2) | ((x.w != 0u) << 3);
    if (!__any_sync(0xffffffffu, m != 0u)) continue;
    const uint32_t cn = __popc(m);
    uint32_t inc = cn;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += o;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    if (nbuf + total > kDescCap) flush();
    const bool direct = total > kDescCap;  // a dense row: per-lane element work, no buffering
    uint32_t pos = (direct ? fill : nbuf) + inc - cn;
    while (m) {
      const uint32_t b = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t wi = host ? (b >> 2) : b;
      const uint32_t word = wi == 0 ? x.x : (wi == 1 ? x.y : (wi == 2 ? x.z : x.w));
      const uint32_t local = host ? v * 16 + b : v * 4 + b;
      const uint32_t cnt = host ? ((word >> (8 * (b & 3))) & 0xffu) : min(word, 65536u);
      if (direct)
        element(slot0 + local, cnt, pos++);
      else
        desc[pos++] = local | (cnt << 12);
    }
    if (direct) fill += total; else nbuf += total;
  }
  flush();
  if (lane == 0) p.cnt[it] = fill;
}

// The usual (sparse) piece: every lane owns a CONTIGUOUS span of the piece (8 vectors = 128 bytes of
// a 4 KB piece), so ascending slot order is lane-major and ONE warp scan of the per-lane element
// counts ranks the whole piece (the row-wise version above needs one scan per 512-byte row, and the
// dependent shuffles were what a piece cost).  The lane's vectors are read in a rotated order
// (vector (j + lane) mod 8 at step j: the 8 lanes of a quarter-warp then touch 8 different bank
// groups, no conflicts for the 128-byte lane stride) and their element masks are merged into one
// bitset in true order, which the lane then walks: descriptor = local slot | count << 12, the
// count read back from the staged bytes.  Loop 2 is the lane-parallel element pass as above.
__device__ __forceinline__ void compact_staged(const CompactParams& p, uint32_t it, uint32_t lane, const uint4* src,
                                               uint32_t* desc) {
  const uint32_t e = it / p.pieces;
  const uint32_t pc = it - e * p.pieces;
  const bool host = pc < p.host_pieces;
  const uint32_t vpl = p.piece / 512;  // vectors per lane: 8 for the 4 KB piece (1, 2, 4 for tiny maps)
  if (vpl == 0) {                      // pieces below 512 bytes (maps of fewer than 1,024 slots): row-wise path
    compact_staged_rows(p, it, lane, src, desc);
    return;
  }
  uint64_t w0 = 0, w1 = 0;             // element bitset of the lane's span, true order (host: 1 bit per byte, 128 bits;
  const uint4* mine = src + lane * vpl;  // device: 1 bit per u32, 32 bits)
#pragma unroll
  for (uint32_t j = 0; j < 8; ++j) {
    if (j < vpl) {
      const uint32_t t = (j + lane) & (vpl - 1);
      const uint4 x = mine[t];
      if (host) {
        const uint64_t m = nz_bytes(x.x) | (nz_bytes(x.y) << 4) | (nz_bytes(x.z) << 8) | (nz_bytes(x.w) << 12);
        if (t < 4) w0 |= m << (16 * t); else w1 |= m << (16 * (t - 4));
      } else {
        const uint32_t m = (x.x != 0u) | ((x.y != 0u) << 1) | ((x.z != 0u) << 2) | ((x.w != 0u) << 3);
        w0 |= (uint64_t)m << (4 * t);
      }
    }
  }
  const uint32_t cn = __popcll(w0) + __popcll(w1);
  uint32_t inc = cn;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
  if (total == 0) {
    if (lane == 0) p.cnt[it] = 0;
    return;
  }
  if (total > kDescCap) {  // a dense piece: the row-wise path handles any density
    compact_staged_rows(p, it, lane, src, desc);
    return;
  }
  // loop 1: descriptors at their rank
  uint32_t pos = inc - cn;
  const uint8_t* bytes = reinterpret_cast<const uint8_t*>(mine);
  const uint32_t span0 = host ? lane * vpl * 16 : lane * vpl * 4;  // first local slot of the lane's span
  if (host) {
    while (w0) {
      const uint32_t g = __ffsll((long long)w0) - 1;
      w0 &= w0 - 1;
      desc[pos++] = (span0 + g) | ((uint32_t)bytes[g] << 12);
    }
    while (w1) {
      const uint32_t g = 64 + __ffsll((long long)w1) - 1;
      w1 &= w1 - 1;
      desc[pos++] = (span0 + g) | ((uint32_t)bytes[g] << 12);
    }
  } else {
    uint32_t w = (uint32_t)w0;
    while (w) {
      const uint32_t g = __ffs(w) - 1;
      w &= w - 1;
      desc[pos++] = (span0 + g) | (min(reinterpret_cast<const uint32_t*>(mine)[g], 65536u) << 12);
    }
  }
  __syncwarp();
  // loop 2: one element per lane
  const uint32_t slot0 = host ? pc * p.piece : p.H + (pc - p.host_pieces) * (p.piece / 4);
  uint32_t* out = p.sorted + (uint64_t)e * p.S + slot0;
  uint8_t* classed_row = p.classed ? p.classed + (uint64_t)e * p.S : nullptr;
  for (uint32_t t = lane; t < total; t += 32) {
    const uint32_t d = desc[t];
    const uint32_t idx = slot0 + (d & 0xfffu), cnt = d >> 12;
    const uint32_t klass = host ? hfz_class_host(cnt) : hfz_class_device(cnt);
    const uint32_t rung = 31 - __clz(klass);
    const uint32_t en = idx | (rung << 24);
    out[t] = en;
    if (klass & ~(uint32_t)__ldg(p.v0 + idx)) note_first(p.first + (size_t)idx * 8 + rung, e);
    if (classed_row) classed_row[idx] = (uint8_t)klass;
  }
  if (lane == 0) p.cnt[it] = total;
  __syncwarp();
}

__global__ void __launch_bounds__(kStepWarps * 32, 1) hfz_k_small_step(const StepParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  cg::grid_group grid = cg::this_grid();
  const CompactParams& c = p.c;
  const uint32_t lane = threadIdx.x & 31, wic = threadIdx.x >> 5;
  const uint64_t W = (uint64_t)gridDim.x * kStepWarps;
  const uint64_t gw = (uint64_t)wic * gridDim.x + blockIdx.x;  // consecutive warps sit on different SMs
  const uint64_t gthread = gw * 32 + lane, nthreads = W * 32;
  const bool fused = p.do_scan && p.do_resolve;
  const uint4 ones = make_uint4(kNone, kNone, kNone, kNone);
  uint8_t* wbuf = smem + (size_t)wic * kStepBuf;
  uint32_t* desc = reinterpret_cast<uint32_t*>(smem + (size_t)kStepWarps * kStepBuf) + wic * kDescCap;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kStepWarps * (kStepBuf + kDescCap * 4)) + wic * 2;

  dbg_mark(p, 0);
  if (p.do_scan) {
    // ---- phase 1: compact.  (map, piece) items dealt round-robin over all warps of the grid; the
    // piece is staged in shared memory by ONE TMA bulk copy per item (SASS: UBLKCP), double-buffered:
    // item k + 1 is in flight while item k is compacted.
    if (lane == 0) {
      hfz_mbar_init(bars + 0, 1);
      hfz_mbar_init(bars + 1, 1);
      hfz_fence_barrier_init();
    }
    __syncwarp();
    const uint64_t items = c.n_exec * c.pieces;
    const uint64_t pol = hfz_policy_evict_first();
    auto issue = [&](uint64_t it, uint32_t b) {
      if (lane == 0) {
        const uint64_t e64 = it / c.pieces;
        const uint32_t pc = (uint32_t)(it - e64 * c.pieces);
        hfz_fence_proxy_async();  // the buffer's last readers (generic proxy) are done: ordered before the async write
        hfz_mbar_expect_tx(bars + b, c.piece);
        hfz_bulk_g2s_stream(wbuf + b * kStepPiece, c.raw + e64 * c.rec_bytes + (uint64_t)pc * c.piece, c.piece, bars + b, pol);
      }
    };
    if (gw < items) issue(gw, 0);
    uint32_t k = 0;
    long long t_wait = 0, t_work = 0;
    for (uint64_t it = gw; it < items; it += W, ++k) {
      const uint32_t b = k & 1;
      if (it + W < items) issue(it + W, b ^ 1);
      const long long t0 = clock64();
      hfz_mbar_wait(bars + b, (k >> 1) & 1);
      const long long t1 = clock64();
      compact_staged(c, (uint32_t)it, lane, reinterpret_cast<const uint4*>(wbuf + b * kStepPiece), desc);
      __syncwarp();
      t_wait += t1 - t0;
      t_work += clock64() - t1;
    }
    if (p.dbg && gw == 0 && lane == 0) {
      p.dbg[11] = (unsigned long long)t_wait;
      p.dbg[12] = (unsigned long long)t_work;
      p.dbg[13] = k;
    }
    dbg_mark(p, 1);
    // scrub the previous call's table (nobody reads it in this launch)
    for (uint64_t s = gthread; s < c.S; s += nthreads) {
      uint4* f = reinterpret_cast<uint4*>(p.first_prev + s * 8);
      const uint4 a = f[0], b = f[1];
      if ((a.x & a.y & a.z & a.w & b.x & b.y & b.z & b.w) != kNone) {
        f[0] = ones;
        f[1] = ones;
      }
    }
    dbg_mark(p, 2);
    __threadfence();
    grid.sync();
    dbg_mark(p, 3);

    // ---- phase 2, by role: [0, D) delta (+ merge + resolve), then one warp per map: chains
    const uint64_t D = c.S / 128;  // warps: 4 slots per thread
    uint32_t newh = 0, newd = 0;
    for (uint64_t role = gw; role < D + c.n_exec; role += W) {
      if (role < D) {
        // delta word of 4 slots from the table; fused: the single-rank merge and the Admit flags right here
        const uint64_t t = role * 32 + lane;  // word index, < S / 4
        fold_word(c.first, t, fused, p.virgin, p.delta_out, p.flags, c.H, newh, newd);
      } else {
        // signatures: ONE map per warp, the whole warp on its two chains (hfz_fnv.cuh).  The warp gathers the
        // map's ordered piece lists into shared memory (cp.async; one piece per lane, every copy in flight
        // at once), 1,024 entries per round, then runs the Full and the Simple chain over the buffer
        // bit-sliced, 32 steps per lane.  (Until round 2 of the build, lanes 0..3 ran the four chains of two
        // maps serially: 53-64 cycles per entry, ~78 k cycles for two maps at 2 % density; a scheduler had
        // one such warp to issue for and nothing could shorten the dependency.)
        const uint64_t e = role - D;
        uint32_t* buf = reinterpret_cast<uint32_t*>(wbuf);
        uint8_t* stream = wbuf + kChainRound * 4;  // 3,072 bytes of byte stream + slack (the buffer is 8 KB)
        static_assert(kChainRound * 4 + 3072 + 16 <= kStepBuf, "entry buffer + byte stream must fit the warp's staging buffer");
        uint64_t hf = HFZ_FNV_OFFSET, hs = HFZ_FNV_OFFSET;
        uint32_t cur_pc = 0, cur_i = 0, nnz = 0;
        const uint32_t* base = c.sorted + e * c.S;
        const uint32_t* cnt = c.cnt + e * c.pieces;
        const long long tg0 = clock64();
        for (;;) {
          uint32_t pos = 0;
          while (cur_pc < c.pieces && pos < kChainRound) {
            if (cur_i == 0) {
              // whole pieces, one per lane: as many leading pieces of this batch as still fit
              const uint32_t pcl = cur_pc + lane;
              const uint32_t my_n = pcl < c.pieces ? __ldcg(cnt + pcl) : 0u;
              uint32_t inc = my_n;
#pragma unroll
              for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += o;
              }
              const uint32_t fits = __ballot_sync(0xffffffffu, inc <= kChainRound - pos);
              uint32_t k = fits == 0xffffffffu ? 32u : (uint32_t)__ffs(~fits) - 1u;  // leading lanes whose pieces fit
              k = min(k, c.pieces - cur_pc);
              if (k) {
                if (lane < k) {
                  const uint32_t* list = base + piece_slot0(c, pcl);
                  uint32_t* d0 = buf + pos + inc - my_n;
                  for (uint32_t i = 0; i < my_n; ++i) cp_async4(d0 + i, list + i);
                }
                pos += __shfl_sync(0xffffffffu, inc, k - 1);
                cur_pc += k;
                continue;
              }
            }
            // a piece that does not fit the rest of the buffer: part of it, coalesced
            const uint32_t n_pc = __ldcg(cnt + cur_pc);
            const uint32_t take = min(n_pc - cur_i, kChainRound - pos);
            const uint32_t* list = base + piece_slot0(c, cur_pc) + cur_i;
            for (uint32_t i = lane; i < take; i += 32) cp_async4(buf + pos + i, list + i);
            pos += take;
            cur_i += take;
            if (cur_i == n_pc) {
              ++cur_pc;
              cur_i = 0;
            }
          }
          if (pos == 0) break;
          nnz += pos;
          cp_async_wait_all();
          __syncwarp();
          const long long tc0 = clock64();
          if (p.dbg && e == 0 && lane == 0) p.dbg[8] = (unsigned long long)(tc0 - tg0);
          hf = pfnv::chain_entries<3>(hf, buf, pos, stream, lane);
          hs = pfnv::chain_entries<2>(hs, buf, pos, stream, lane);
          if (p.dbg && e == 0 && lane == 0) {
            p.dbg[9] = (unsigned long long)(clock64() - tc0);
            p.dbg[10] = pos;
          }
          __syncwarp();
        }
        if (lane == 0) {
          p.sig_full[e] = hf;
          p.sig_simple[e] = hs;
          if (p.nnz) p.nnz[e] = nnz;
        }
      }
    }
    if (fused) {
      newh = __reduce_add_sync(0xffffffffu, newh);
      newd = __reduce_add_sync(0xffffffffu, newd);
      if (lane == 0) {
        if (newh) atomicAdd(p.edge_counts + 0, (unsigned long long)newh);
        if (newd) atomicAdd(p.edge_counts + 1, (unsigned long long)newd);
      }
    }
    dbg_mark(p, 4);
    if (!p.do_resolve) return;
    __threadfence();
    grid.sync();
    dbg_mark(p, 5);
  }

  if (!fused) {
    // resolve half on its own: rank-ordered merge first (prior = virgin before D_rank), Admit codes zeroed
    uint32_t newh = 0, newd = 0;
    for (uint64_t v = gthread; v < c.S / 16; v += nthreads) {
      uint4 acc = reinterpret_cast<uint4*>(p.virgin)[v];
      const uint4 old = acc;
      for (uint32_t q = 0; q < p.n_ranks; ++q) {
        if (q == p.rank) reinterpret_cast<uint4*>(p.prior)[v] = acc;
        const uint4 d = reinterpret_cast<const uint4*>(p.deltas + (size_t)q * c.S)[v];
        acc.x |= d.x; acc.y |= d.y; acc.z |= d.z; acc.w |= d.w;
      }
      reinterpret_cast<uint4*>(p.virgin)[v] = acc;
      const uint32_t turned = __popc(nz_bytes(acc.x) & ~nz_bytes(old.x)) + __popc(nz_bytes(acc.y) & ~nz_bytes(old.y)) +
                              __popc(nz_bytes(acc.z) & ~nz_bytes(old.z)) + __popc(nz_bytes(acc.w) & ~nz_bytes(old.w));
      if (v * 16 < c.H) newh += turned; else newd += turned;
    }
    newh = __reduce_add_sync(0xffffffffu, newh);
    newd = __reduce_add_sync(0xffffffffu, newd);
    if (lane == 0) {
      if (newh) atomicAdd(p.edge_counts + 0, (unsigned long long)newh);
      if (newd) atomicAdd(p.edge_counts + 1, (unsigned long long)newd);
    }
    __threadfence();
    grid.sync();
    // the table against P_r (just written above), one thread per slot
    for (uint64_t s = gthread; s < c.S; s += nthreads) {
      const uint4* f = reinterpret_cast<const uint4*>(c.first + s * 8);
      resolve_slot(__ldcg(f), __ldcg(f + 1), __ldcg(p.prior + s), p.flags);
    }
    __threadfence();
    grid.sync();
  }

  // ---- phase 3: flags -> Admit codes (and the flags back to zero for the next call)
  for (uint64_t e = gthread; e < c.n_exec; e += nthreads) {
    const uint32_t f = __ldcg(p.flags + e);
    p.admit[e] = (f & 2u) ? 2 : (uint8_t)(f & 1u);
    if (f) p.flags[e] = 0;
  }
  dbg_mark(p, 6);
}

// ---------------------------------------------------------------------------
// launch plumbing

template <int ROW>
size_t scan_smem_bytes(uint32_t S, bool vsmem, int warps) {
  return (vsmem ? S : 0) + (size_t)warps * (RowCfg<ROW>::kGroup * RowCfg<ROW>::kSlot + 128) + 16;
}

template <int REC_CT, int ROW, bool VSMEM, bool CLASSED>
int launch_scan_t(hfz_ctx* ctx, const ScanParams& p) {
  auto kern = hfz_k_scan<REC_CT, ROW, VSMEM, CLASSED>;
  int warps = ROW >= 512 ? 10 : 20;  // __launch_bounds__ of the kernel
  while (warps > 1 && scan_smem_bytes<ROW>(p.S, VSMEM, warps) > (size_t)ctx->max_smem_optin) --warps;
  if (ctx->scan_warps > 0 && ctx->scan_warps < warps) warps = ctx->scan_warps;
  const size_t smem = scan_smem_bytes<ROW>(p.S, VSMEM, warps);
  HFZ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  uint64_t grid = (uint64_t)ctx->num_sms;
  const uint64_t groups = (p.n_exec + RowCfg<ROW>::kGroup - 1) / RowCfg<ROW>::kGroup;
  if (grid > groups) grid = groups;  // warp w of CTA b owns work slice w * grid + b
  kern<<<(uint32_t)grid, warps * 32, smem, ctx->stream>>>(p);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

template <int REC_CT, bool VSMEM>
int launch_scan_r(hfz_ctx* ctx, const ScanParams& p, int row) {
  const bool classed = p.classed != nullptr;
  if (row == 256)
    return classed ? launch_scan_t<REC_CT, 256, VSMEM, true>(ctx, p)
                   : launch_scan_t<REC_CT, 256, VSMEM, false>(ctx, p);
  if (row == 1024)
    return classed ? launch_scan_t<REC_CT, 1024, VSMEM, true>(ctx, p)
                   : launch_scan_t<REC_CT, 1024, VSMEM, false>(ctx, p);
  return classed ? launch_scan_t<REC_CT, 512, VSMEM, true>(ctx, p)
                 : launch_scan_t<REC_CT, 512, VSMEM, false>(ctx, p);
}

template <bool VSMEM, bool CLASSED>
int launch_scan_wpm_t(hfz_ctx* ctx, const ScanParams& p) {
  auto kern = hfz_k_scan_wpm<VSMEM, CLASSED>;
  // spread a small batch over all SMs: as few warps per CTA as cover the batch (4..16)
  int warps = (int)((p.n_exec + ctx->num_sms - 1) / ctx->num_sms);
  warps = warps < 4 ? 4 : (warps > 16 ? 16 : warps);
  const size_t smem = (VSMEM ? p.S : 0) + (size_t)warps * kListCap * 4 + 16;
  HFZ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  uint64_t grid = (p.n_exec + warps - 1) / warps;
  if (grid > (uint64_t)ctx->num_sms) grid = (uint64_t)ctx->num_sms;
  kern<<<(uint32_t)grid, warps * 32, smem, ctx->stream>>>(p);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

constexpr int kPipeP = 4;  // producer warps per team

template <int REC_CT, int ROW, bool VSMEM, bool CLASSED>
int launch_scan_pipe_t(hfz_ctx* ctx, const ScanParams& p) {
  auto kern = hfz_k_scan_pipe<REC_CT, ROW, kPipeP, VSMEM, CLASSED>;
  constexpr int SLOT = 32 * RowCfg<ROW>::kSlot + 128;
  const uint64_t groups = (p.n_exec + 31) / 32;
  int gmax = (ROW == 512 ? 320 : 640) / (32 * (1 + kPipeP));  // teams the launch bounds allow
  auto smem_for = [&](int G) { return (size_t)(VSMEM ? p.S : 0) + (size_t)G * kPipeP * SLOT + 8 * (1 + 2 * kPipeP * G) + 16; };
  while (gmax > 1 && smem_for(gmax) > (size_t)ctx->max_smem_optin) --gmax;
  int G = (int)((groups + ctx->num_sms - 1) / ctx->num_sms);
  G = G < 1 ? 1 : (G > gmax ? gmax : G);
  const size_t smem = smem_for(G);
  HFZ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const uint64_t grid = (groups + G - 1) / G;
  kern<<<(uint32_t)grid, G * (1 + kPipeP) * 32, smem, ctx->stream>>>(p, G);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

template <int REC_CT, bool VSMEM>
int launch_scan_pipe_r(hfz_ctx* ctx, const ScanParams& p, int row) {
  const bool classed = p.classed != nullptr;
  if (row == 256)
    return classed ? launch_scan_pipe_t<REC_CT, 256, VSMEM, true>(ctx, p)
                   : launch_scan_pipe_t<REC_CT, 256, VSMEM, false>(ctx, p);
  return classed ? launch_scan_pipe_t<REC_CT, 512, VSMEM, true>(ctx, p)
                 : launch_scan_pipe_t<REC_CT, 512, VSMEM, false>(ctx, p);
}

// grow-only scratch with geometric slack (no cudaFree + cudaMalloc per slightly larger batch)
template <typename T>
int grow(T*& ptr, uint64_t& cap, uint64_t need, const char* what) {
  if (cap >= need) return HFZ_OK;
  uint64_t want = cap * 2 > need ? cap * 2 : need;
  cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&ptr, want * sizeof(T));
  if (e != cudaSuccess && want > need) {
    cudaGetLastError();
    want = need;
    e = cudaMalloc(&ptr, want * sizeof(T));
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    hfz_set_error("%s: cudaMalloc of %llu bytes failed (%s)", what, (unsigned long long)(want * sizeof(T)), cudaGetErrorString(e));
    return HFZ_ENOMEM;
  }
  cap = want;
  return HFZ_OK;
}

// compact + chain for a dense batch; false when the scratch it would need is not allowed
bool two_stage_fits(const hfz_ctx* ctx, uint64_t n_exec) {
  return n_exec * (uint64_t)ctx->S <= (1ull << 30);  // <= 4 GB of u32 entries
}

int launch_scan_two_stage(hfz_ctx* ctx, const ScanParams& sp) {
  CompactParams p;
  p.raw = sp.raw;
  p.n_exec = sp.n_exec;
  p.rec_bytes = sp.rec_bytes;
  p.S = sp.S;
  p.H = sp.H;
  uint32_t piece = kTsPiece;
  while (sp.H % piece) piece >>= 1;  // H is a power of two >= 512
  p.piece = piece;
  p.host_pieces = sp.H / piece;
  p.pieces = (uint32_t)(sp.rec_bytes / piece);
  p.v0 = sp.v0;
  p.first = sp.first;
  p.classed = sp.classed;
  // grow-only scratch with geometric slack (hfz.h documents the footprint: 4 x S bytes per exec)
  int rc = grow(ctx->ts_sorted, ctx->ts_sorted_cap, sp.n_exec * (uint64_t)sp.S, "two-stage scan: piece lists");
  if (rc) return rc;
  if ((rc = grow(ctx->ts_cnt, ctx->ts_cnt_cap, sp.n_exec * (uint64_t)p.pieces, "two-stage scan: piece counts"))) return rc;
  p.sorted = ctx->ts_sorted;
  p.cnt = ctx->ts_cnt;
  const uint64_t items = sp.n_exec * p.pieces;
  uint64_t blocks = (items + 7) / 8;
  const uint64_t cap = (uint64_t)ctx->num_sms * 8;  // 64 warps per SM
  if (blocks > cap) blocks = cap;
  hfz_k_compact<<<(uint32_t)blocks, 256, 0, ctx->stream>>>(p);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  hfz_k_chain_pieces<<<(uint32_t)((sp.n_exec + 127) / 128), 128, 0, ctx->stream>>>(
      p, sp.sig_full, sp.sig_simple, sp.nnz);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

// ---- fused small step: host side
int ensure_admit_flags(hfz_ctx* ctx, uint64_t n_exec);
bool small_step_ok(hfz_ctx* ctx, uint64_t n_exec) {
  if (!ctx->small_fused || n_exec == 0) return false;
  // measured on B200 (65,536 slots, warm / cold virgin): 4,096 maps 0.21 / 0.36 ms fused vs 0.36 / 0.70 pipelined;
  // 8,192 maps 0.40 / 0.62 vs 0.40 / 1.47; 12,288 maps 0.58 / 0.90 vs 0.47 / 2.03 (pipelined wins warm from there on)
  const uint64_t limit = ctx->scan_two_stage >= 0 ? (uint64_t)ctx->scan_two_stage : 8192;
  if (n_exec > limit || !two_stage_fits(ctx, n_exec)) return false;
  if (ctx->coop_grid < 0) {  // once: cooperative launch support and the co-resident grid size
    int coop = 0, per_sm = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
    const size_t smem = kStepSmem;
    if (coop && cudaFuncSetAttribute(hfz_k_small_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hfz_k_small_step, kStepWarps * 32, smem) == cudaSuccess && per_sm >= 1)
      ctx->coop_grid = ctx->num_sms;
    else
      ctx->coop_grid = 0;
    cudaGetLastError();
  }
  return ctx->coop_grid > 0;
}

int small_step_scratch(hfz_ctx* ctx, uint64_t n_exec, uint32_t pieces) {
  int rc = ensure_admit_flags(ctx, n_exec);
  if (rc) return rc;
  if ((rc = grow(ctx->ts_sorted, ctx->ts_sorted_cap, n_exec * (uint64_t)ctx->S, "small step: piece lists"))) return rc;
  if ((rc = grow(ctx->ts_cnt, ctx->ts_cnt_cap, n_exec * (uint64_t)pieces, "small step: piece counts"))) return rc;
  if (!ctx->ss_first[0]) {  // two first-occurrence tables (all-ones between calls)
    const size_t bytes = (size_t)ctx->S * 8 * sizeof(uint32_t);
    for (int i = 0; i < 2; ++i) {
      HFZ_CUDA(cudaMalloc(&ctx->ss_first[i], bytes));
      HFZ_CUDA(cudaMemsetAsync(ctx->ss_first[i], 0xff, bytes, ctx->stream));
    }
  }
  return HFZ_OK;
}

int launch_small_step(hfz_ctx* ctx, StepParams& p) {
  void* args[] = {&p};
  HFZ_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(hfz_k_small_step), dim3((unsigned)ctx->coop_grid),
                                       dim3(kStepWarps * 32), args, kStepSmem, ctx->stream));
  ++ctx->launches;
  return HFZ_OK;
}

// scan half (and, with virgin_inout, the whole single-rank step) of a small dense batch
int small_step_scan(hfz_ctx* ctx, const uint8_t* raw, uint64_t n_exec, const uint8_t* v0, uint8_t* classed,
                    uint64_t* sig_full, uint64_t* sig_simple, uint32_t* nnz, uint8_t* delta_out,
                    uint8_t* virgin_inout, uint64_t* edge_counts, uint8_t* admit) {
  HFZ_CUDA(cudaSetDevice(ctx->device));
  StepParams p;
  CompactParams& c = p.c;
  c.raw = raw;
  c.n_exec = n_exec;
  c.rec_bytes = ctx->rec_bytes;
  c.S = ctx->S;
  c.H = ctx->H;
  // piece = what one TMA bulk copy stages for a warp (4 KB, or the whole host half of a tiny map)
  uint32_t piece = kStepPiece;
  while (ctx->H % piece) piece >>= 1;
  c.piece = piece;
  c.host_pieces = ctx->H / piece;
  c.pieces = (uint32_t)(ctx->rec_bytes / piece);
  int rc = small_step_scratch(ctx, n_exec, c.pieces);
  if (rc) return rc;
  if (classed) HFZ_CUDA(cudaMemsetAsync(classed, 0, n_exec * (size_t)ctx->S, ctx->stream));
  ctx->ss_pp ^= 1;
  c.v0 = v0;
  c.first = ctx->ss_first[ctx->ss_pp];
  c.sorted = ctx->ts_sorted;
  c.cnt = ctx->ts_cnt;
  c.classed = classed;
  p.first_prev = ctx->ss_first[ctx->ss_pp ^ 1];
  p.sig_full = sig_full;
  p.sig_simple = sig_simple;
  p.nnz = nnz;
  p.delta_out = delta_out;
  p.virgin = virgin_inout;
  p.prior = ctx->prior;
  p.edge_counts = reinterpret_cast<unsigned long long*>(edge_counts);
  p.deltas = delta_out;
  p.n_ranks = 1;
  p.rank = 0;
  p.admit = admit;
  p.flags = ctx->admit_flags;
  p.do_scan = 1;
  p.do_resolve = virgin_inout != nullptr;
  p.dbg = ctx->ss_dbg ? ctx->d_small + 8 : nullptr;
  if (p.dbg) {
    HFZ_CUDA(cudaMemsetAsync(p.dbg, 0, 16 * 8, ctx->stream));
    HFZ_CUDA(cudaMemsetAsync(p.dbg, 0xff, 8, ctx->stream));
  }
  ctx->sc_small = !p.do_resolve;  // a resolve-only launch follows (hfz_feedback_resolve)
  if (ctx->sc_small) {
    ctx->sc_step.resize(sizeof(StepParams));
    memcpy(ctx->sc_step.data(), &p, sizeof(StepParams));
  }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (ctx->time_scan) {
    HFZ_CUDA(cudaEventCreate(&ev0));
    HFZ_CUDA(cudaEventCreate(&ev1));
    HFZ_CUDA(cudaEventRecord(ev0, ctx->stream));
  }
  rc = launch_small_step(ctx, p);
  if (ctx->time_scan) {
    HFZ_CUDA(cudaEventRecord(ev1, ctx->stream));
    ctx->scan_events.emplace_back(ev0, ev1);
  }
  return rc;
}

// resolve half after small_step_scan(virgin_inout = nullptr): merge in rank order + Admit codes
int small_step_resolve(hfz_ctx* ctx, uint64_t n_exec, uint8_t* virgin_inout, uint64_t* edge_counts,
                       const uint8_t* deltas, uint32_t n_ranks, uint32_t rank, uint8_t* admit) {
  StepParams p;
  if (ctx->sc_step.size() != sizeof(StepParams)) {
    hfz_set_error("hfz_feedback_resolve: no scan to resolve");
    return HFZ_EINVAL;
  }
  memcpy(&p, ctx->sc_step.data(), sizeof(StepParams));
  if (p.c.n_exec != n_exec) {
    hfz_set_error("hfz_feedback_resolve: n_exec differs from the scan's");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  p.virgin = virgin_inout;
  p.edge_counts = reinterpret_cast<unsigned long long*>(edge_counts);
  p.deltas = deltas;
  p.n_ranks = n_ranks;
  p.rank = rank;
  p.admit = admit;
  p.flags = ctx->admit_flags;
  p.do_scan = 0;
  p.do_resolve = 1;
  return launch_small_step(ctx, p);
}

int launch_scan(hfz_ctx* ctx, const ScanParams& p) {
  // virgin copy in shared memory whenever it leaves room for the per-warp slots
  const bool vsmem = ctx->virgin_smem && p.S <= 65536u;
  // small batches: one warp per map (latency), else 32 maps per warp (pipelined, then throughput)
  const uint64_t small_limit = ctx->scan_small >= 0 ? (uint64_t)ctx->scan_small
                                                    : (uint64_t)ctx->num_sms * 10 * 65536u / p.S;
  // small and medium batches: compact + chain (two-stage)
  // measured: 65,536 slots -- wins up to ~3 k maps; 262,144 slots (virgin not in shared memory for the
  // other kernels) -- 1,024 maps 0.82 vs 1.72 ms, 4,096 maps 1.60 vs 1.72 ms
  const uint64_t ts_limit = ctx->scan_two_stage >= 0 ? (uint64_t)ctx->scan_two_stage : (p.S <= 65536u ? 3072 : 4096);
  if (p.n_exec <= ts_limit && two_stage_fits(ctx, p.n_exec)) {
    const int rc = launch_scan_two_stage(ctx, p);
    if (rc != HFZ_ENOMEM) return rc;
    cudaGetLastError();  // no room for the list scratch: the kernels below need none
  }
  if (p.n_exec <= small_limit) {
    const bool classed = p.classed != nullptr;
    if (vsmem) return classed ? launch_scan_wpm_t<true, true>(ctx, p) : launch_scan_wpm_t<true, false>(ctx, p);
    return classed ? launch_scan_wpm_t<false, true>(ctx, p) : launch_scan_wpm_t<false, false>(ctx, p);
  }
  // medium batches: pipelined lane-per-map (producer warps stream, one consumer warp per group).
  // Measured on B200, 65,536 slots, ms per step (lane-per-map / warp-per-map / pipelined):
  //   1,024: 0.61 / 0.34 / 0.37   2,048: 0.62 / 0.40 / 0.37   4,096: 0.61 / 0.71 / 0.38
  //   8,192: 0.62 / 1.36 / 0.42  12,288: 0.64 / 1.99 / 0.48  16,384: 0.65 / 2.37 / 0.78
  const uint64_t groups = (p.n_exec + 31) / 32;
  const uint64_t pipe_limit = ctx->scan_pipe >= 0 ? (uint64_t)ctx->scan_pipe : 3;  // groups per SM
  if (groups <= pipe_limit * (uint64_t)ctx->num_sms) {
    // 512-byte rows (up to 2 teams per CTA) while every SM has one group, 256-byte rows (4 teams) beyond
    int row = ctx->scan_row;
    if (row != 256 && row != 512) row = groups <= (uint64_t)ctx->num_sms ? 512 : 256;
    if (p.S == 65536u && vsmem) return launch_scan_pipe_r<163840, true>(ctx, p, row);
    if (p.S == 262144u && !vsmem) return launch_scan_pipe_r<655360, false>(ctx, p, row);
    return vsmem ? launch_scan_pipe_r<0, true>(ctx, p, row) : launch_scan_pipe_r<0, false>(ctx, p, row);
  }
  // 256-byte rows let 18 warps/SM hide the shared-memory latency of phase B (best when every SM
  // has more than 9 groups to run); 512-byte rows halve the number of rows a warp walks, which
  // wins while a batch gives each SM at most 9 groups anyway (latency-bound regime).
  // 1,024-byte rows = 16 maps per warp (lanes 16..31 idle in the chain phase): twice the warps for a batch that
  // leaves most of the grid without a 32-map group.  Measured (65,536 slots, ms per fold, 512- vs 1,024-byte rows):
  // 14,336 maps 0.617 / 0.577, 16,384: 0.627 / 0.581, 20,480: 0.705 / 0.672, 24,576: 0.765 / 1.070.
  int row = ctx->scan_row;
  if (row == 1024 && (p.H % 1024u)) row = 0;  // needs rows of 1,024 bytes in both halves
  if (row != 256 && row != 512 && row != 1024) {
    const uint64_t g32 = (p.n_exec + 31) / 32;
    row = (g32 * 2 <= (uint64_t)ctx->num_sms * 9 && p.H % 1024u == 0) ? 1024 : (g32 <= (uint64_t)ctx->num_sms * 9 ? 512 : 256);
  }
  if (p.S == 65536u && vsmem) return launch_scan_r<163840, true>(ctx, p, row);
  if (p.S == 262144u && !vsmem) return launch_scan_r<655360, false>(ctx, p, row);
  return vsmem ? launch_scan_r<0, true>(ctx, p, row) : launch_scan_r<0, false>(ctx, p, row);
}

// per-exec flags of the table resolve: zero between calls (hfz_k_admit_codes / the fused step re-zero what they read)
int ensure_admit_flags(hfz_ctx* ctx, uint64_t n_exec) {
  if (ctx->admit_cap >= n_exec) return HFZ_OK;
  if (ctx->admit_flags) cudaFree(ctx->admit_flags);
  ctx->admit_flags = nullptr;
  ctx->admit_cap = 0;
  const uint64_t cap = n_exec < 1024 ? 1024 : n_exec + n_exec / 4;
  if (cudaMalloc(&ctx->admit_flags, cap * sizeof(uint32_t)) != cudaSuccess) {
    hfz_set_error("cudaMalloc(admit flags, %llu) failed", (unsigned long long)cap * 4);
    return HFZ_ENOMEM;
  }
  HFZ_CUDA(cudaMemsetAsync(ctx->admit_flags, 0, cap * sizeof(uint32_t), ctx->stream));
  ctx->admit_cap = cap;
  return HFZ_OK;
}

}  // namespace

// delta_out = NULL: no delta kernel (hfz_feedback_fold_single follows and reads the table itself)
static int scan_dense(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec, const uint8_t* virgin_v0,
                      uint8_t* classed_out, uint64_t* sig_full_out, uint64_t* sig_simple_out, uint32_t* nnz_out,
                      uint8_t* delta_out);

extern "C" int hfz_feedback_scan(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                                 const uint8_t* virgin_v0, uint8_t* classed_out,
                                 uint64_t* sig_full_out, uint64_t* sig_simple_out,
                                 uint32_t* nnz_out, uint8_t* delta_out) {
  if (!delta_out) {
    hfz_set_error("hfz_feedback_scan: null argument");
    return HFZ_EINVAL;
  }
  return scan_dense(ctx, raw_maps, n_exec, virgin_v0, classed_out, sig_full_out, sig_simple_out, nnz_out, delta_out);
}

static int scan_dense(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec, const uint8_t* virgin_v0,
                      uint8_t* classed_out, uint64_t* sig_full_out, uint64_t* sig_simple_out, uint32_t* nnz_out,
                      uint8_t* delta_out) {
  if (!ctx || !virgin_v0 || (n_exec && (!raw_maps || !sig_full_out || !sig_simple_out))) {
    hfz_set_error("hfz_feedback_scan: null argument");
    return HFZ_EINVAL;
  }
  if (n_exec >= 0xfffffffeull) {
    hfz_set_error("hfz_feedback_scan: n_exec too large");
    return HFZ_ECAP;
  }
  if (((uintptr_t)raw_maps | (uintptr_t)virgin_v0 | (uintptr_t)delta_out) & 15) {
    hfz_set_error("hfz_feedback_scan: raw_maps/virgin/delta must be 16-byte aligned");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  if (delta_out && small_step_ok(ctx, n_exec))  // small batch: the scan half of the fused step, one launch
    return small_step_scan(ctx, raw_maps, n_exec, virgin_v0, classed_out, sig_full_out, sig_simple_out, nnz_out,
                           delta_out, nullptr, nullptr, nullptr);
  ctx->sc_small = false;
  int rc = ensure_admit_flags(ctx, n_exec);
  if (rc) return rc;
  HFZ_CUDA(cudaMemsetAsync(ctx->first, 0xff, (size_t)ctx->S * 8 * sizeof(uint32_t), ctx->stream));
  if (classed_out && n_exec)
    HFZ_CUDA(cudaMemsetAsync(classed_out, 0, n_exec * (size_t)ctx->S, ctx->stream));
  if (n_exec) {
    ScanParams p;
    p.raw = raw_maps;
    p.n_exec = n_exec;
    p.S = ctx->S;
    p.H = ctx->H;
    p.rec_bytes = ctx->rec_bytes;
    p.v0 = virgin_v0;
    p.first = ctx->first;
    p.sig_full = sig_full_out;
    p.sig_simple = sig_simple_out;
    p.nnz = nnz_out;
    p.classed = classed_out;
    p.n_groups = (uint32_t)((n_exec + 31) / 32);
    p.prefetch = ctx->scan_prefetch;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (ctx->time_scan) {
      HFZ_CUDA(cudaEventCreate(&ev0));
      HFZ_CUDA(cudaEventCreate(&ev1));
      HFZ_CUDA(cudaEventRecord(ev0, ctx->stream));
    }
    rc = launch_scan(ctx, p);
    if (ctx->time_scan) {
      HFZ_CUDA(cudaEventRecord(ev1, ctx->stream));
      ctx->scan_events.emplace_back(ev0, ev1);
    }
    if (rc) return rc;
  }
  if (delta_out) {
    hfz_k_delta<<<(ctx->S + 255) / 256, 256, 0, ctx->stream>>>(ctx->first, delta_out, ctx->S);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
  }
  return HFZ_OK;
}

// Second half of a single-rank fold after a scan with delta_out = NULL: delta, merge, edge counters and Admit
// flags in one pass over the table, then the codes.
int hfz_feedback_fold_single(hfz_ctx* ctx, uint64_t n_exec, uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                             uint8_t* admit_out) {
  if (!ctx || !virgin_inout || !edge_counts_inout || (n_exec && !admit_out)) {
    hfz_set_error("hfz_feedback_batch: null argument");
    return HFZ_EINVAL;
  }
  hfz_k_fold_single<<<(ctx->S / 4 + 255) / 256, 256, 0, ctx->stream>>>(
      ctx->first, virgin_inout, ctx->admit_flags, reinterpret_cast<unsigned long long*>(edge_counts_inout), ctx->S,
      ctx->H);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  if (n_exec) {
    hfz_k_admit_codes<<<(uint32_t)((n_exec + 255) / 256), 256, 0, ctx->stream>>>(ctx->admit_flags, admit_out, n_exec);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
  }
  return HFZ_OK;
}

bool hfz_sparse_native_ok(const hfz_ctx* c) {
  // one warp's bitmap + prefix (6 bytes per 32 slots) must fit shared memory: maps of up to 2^20 slots
  return c->sparse_native && c->S <= (1u << 20) && c->S >= 1024u;
}

int hfz_feedback_scan_sparse(hfz_ctx* ctx, const uint32_t* pairs, const uint64_t* entry_off,
                             const uint32_t* compact, const uint64_t* compact_off, uint64_t n_exec,
                             uint64_t total_pairs, const uint8_t* virgin_v0, uint8_t* classed_out,
                             uint64_t* sig_full_out, uint64_t* sig_simple_out, uint32_t* nnz_out,
                             uint8_t* delta_out, unsigned long long* bad_pairs, int packed) {
  if (n_exec >= 0xfffffffeull) {
    hfz_set_error("hfz_feedback_scan_sparse: n_exec too large");
    return HFZ_ECAP;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  int rc = ensure_admit_flags(ctx, n_exec);
  if (rc) return rc;
  if (ctx->sp_sorted_cap < total_pairs) {
    cudaFree(ctx->sp_sorted);
    ctx->sp_sorted = nullptr;
    ctx->sp_sorted_cap = 0;
    const uint64_t cap = total_pairs + total_pairs / 8 + 1024;
    HFZ_CUDA(cudaMalloc(&ctx->sp_sorted, cap * 4));
    ctx->sp_sorted_cap = cap;
  }
  if (ctx->sp_cnt_cap < n_exec) {
    cudaFree(ctx->sp_cnt);
    ctx->sp_cnt = nullptr;
    ctx->sp_cnt_cap = 0;
    HFZ_CUDA(cudaMalloc(&ctx->sp_cnt, (n_exec + 1024) * 4));
    ctx->sp_cnt_cap = n_exec + 1024;
  }
  HFZ_CUDA(cudaMemsetAsync(ctx->first, 0xff, (size_t)ctx->S * 8 * sizeof(uint32_t), ctx->stream));
  if (classed_out && n_exec) HFZ_CUDA(cudaMemsetAsync(classed_out, 0, n_exec * (size_t)ctx->S, ctx->stream));
  if (n_exec) {
    SparseParams p;
    p.pairs = reinterpret_cast<const uint2*>(pairs);
    p.off = entry_off;
    p.cpairs = compact;
    p.coff = compact_off;
    p.packed = packed;
    p.n_exec = n_exec;
    p.S = ctx->S;
    p.H = ctx->H;
    p.v0 = virgin_v0;
    p.first = ctx->first;
    p.sorted = ctx->sp_sorted;
    p.cnt = ctx->sp_cnt;
    p.classed = classed_out;
    p.bad = bad_pairs;
    const uint32_t words = ctx->S / 32;
    const size_t per_warp = rank_warp_bytes(words);
    uint64_t rank_warps = (uint64_t)ctx->max_smem_optin / per_warp;
    if (rank_warps > (uint64_t)kRankWarps) rank_warps = kRankWarps;
    if (rank_warps == 0) {
      hfz_set_error("sparse fold: a %u-slot bitmap does not fit shared memory", ctx->S);
      return HFZ_EINVAL;
    }
    const size_t smem = (size_t)rank_warps * per_warp;
    HFZ_CUDA(cudaFuncSetAttribute(hfz_k_sparse_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    uint64_t grid = (n_exec + rank_warps - 1) / rank_warps;
    if (grid > (uint64_t)ctx->num_sms) grid = (uint64_t)ctx->num_sms;
    hfz_k_sparse_rank<<<(uint32_t)grid, (uint32_t)rank_warps * 32, smem, ctx->stream>>>(p);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
    if (n_exec <= (uint64_t)ctx->num_sms * 32)  // latency regime: a warp per exec (one wave)
      hfz_k_sparse_chain_warp<<<(uint32_t)((n_exec + kChainWarps - 1) / kChainWarps), kChainWarps * 32, 0, ctx->stream>>>(
          ctx->sp_sorted, entry_off, compact_off, ctx->sp_cnt, n_exec, sig_full_out, sig_simple_out, nnz_out);
    else
      hfz_k_sparse_chain<<<(uint32_t)((n_exec + 127) / 128), 128, 0, ctx->stream>>>(
          ctx->sp_sorted, entry_off, compact_off, ctx->sp_cnt, n_exec, sig_full_out, sig_simple_out, nnz_out);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
  }
  if (delta_out) {
    hfz_k_delta<<<(ctx->S + 255) / 256, 256, 0, ctx->stream>>>(ctx->first, delta_out, ctx->S);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
  }
  return HFZ_OK;
}

extern "C" int hfz_virgin_merge(hfz_ctx* ctx, uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                                const uint8_t* deltas, uint32_t n_ranks) {
  if (!ctx || !virgin_inout || !edge_counts_inout || (n_ranks && !deltas)) {
    hfz_set_error("hfz_virgin_merge: null argument");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  hfz_k_merge<<<(ctx->S / 16 + 255) / 256, 256, 0, ctx->stream>>>(
      virgin_inout, deltas, n_ranks, 0xffffffffu, nullptr,
      reinterpret_cast<unsigned long long*>(edge_counts_inout), ctx->S, ctx->H);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

namespace {
int resolve_impl(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec, uint8_t* virgin_inout,
                 uint64_t* edge_counts_inout, const uint8_t* deltas, const PeerPtrs* peers, uint32_t n_ranks,
                 uint32_t rank, uint8_t* admit_out) {
  if (!ctx || !virgin_inout || !edge_counts_inout || (!deltas && !peers) || n_ranks == 0 || rank >= n_ranks ||
      (n_exec && !admit_out)) {
    hfz_set_error("hfz_feedback_resolve: bad argument");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  if (ctx->sc_small && n_exec) {  // the scan was the fused small step: its resolve half, one launch
    if (peers) {  // gather the peers' deltas (64 KB each) into the context's staging first
      if (!ctx->ss_deltas) HFZ_CUDA(cudaMalloc(&ctx->ss_deltas, (size_t)kMaxPeers * ctx->S));
      for (uint32_t q = 0; q < n_ranks; ++q)
        HFZ_CUDA(cudaMemcpyAsync(ctx->ss_deltas + (size_t)q * ctx->S, peers->p[q], ctx->S, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
      deltas = ctx->ss_deltas;
    }
    return small_step_resolve(ctx, n_exec, virgin_inout, edge_counts_inout, deltas, n_ranks, rank, admit_out);
  }
  if (peers)
    hfz_k_merge_peers<<<(ctx->S / 16 + 255) / 256, 256, 0, ctx->stream>>>(
        virgin_inout, *peers, n_ranks, rank, ctx->prior, reinterpret_cast<unsigned long long*>(edge_counts_inout),
        ctx->S, ctx->H);
  else
    hfz_k_merge<<<(ctx->S / 16 + 255) / 256, 256, 0, ctx->stream>>>(
        virgin_inout, deltas, n_ranks, rank, ctx->prior,
        reinterpret_cast<unsigned long long*>(edge_counts_inout), ctx->S, ctx->H);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  if (n_exec) {
    hfz_k_resolve_table<<<(ctx->S + 255) / 256, 256, 0, ctx->stream>>>(ctx->first, ctx->prior, ctx->S, ctx->admit_flags);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
    hfz_k_admit_codes<<<(uint32_t)((n_exec + 255) / 256), 256, 0, ctx->stream>>>(ctx->admit_flags, admit_out, n_exec);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
  }
  return HFZ_OK;
}
}  // namespace

extern "C" int hfz_feedback_resolve(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                                    uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                                    const uint8_t* deltas, uint32_t n_ranks, uint32_t rank,
                                    uint8_t* admit_out) {
  if (!deltas) {
    hfz_set_error("hfz_feedback_resolve: bad argument");
    return HFZ_EINVAL;
  }
  return resolve_impl(ctx, raw_maps, n_exec, virgin_inout, edge_counts_inout, deltas, nullptr, n_ranks, rank,
                      admit_out);
}

extern "C" int hfz_feedback_resolve_peers(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                                          uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                                          const uint8_t* const* delta_ptrs, uint32_t n_ranks, uint32_t rank,
                                          uint8_t* admit_out) {
  if (!delta_ptrs || n_ranks == 0 || n_ranks > (uint32_t)kMaxPeers) {
    hfz_set_error("hfz_feedback_resolve_peers: 1..%d delta pointers expected", kMaxPeers);
    return HFZ_EINVAL;
  }
  PeerPtrs peers;
  for (uint32_t q = 0; q < (uint32_t)kMaxPeers; ++q) peers.p[q] = q < n_ranks ? delta_ptrs[q] : nullptr;
  for (uint32_t q = 0; q < n_ranks; ++q)
    if (!peers.p[q] || ((uintptr_t)peers.p[q] & 15)) {
      hfz_set_error("hfz_feedback_resolve_peers: delta pointer %u is null or not 16-byte aligned", q);
      return HFZ_EINVAL;
    }
  return resolve_impl(ctx, raw_maps, n_exec, virgin_inout, edge_counts_inout, nullptr, &peers, n_ranks, rank,
                      admit_out);
}

extern "C" int hfz_feedback_batch(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                                  uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                                  uint8_t* classed_out, uint8_t* admit_out,
                                  uint64_t* sig_full_out, uint64_t* sig_simple_out,
                                  uint32_t* nnz_out) {
  if (!ctx) {
    hfz_set_error("hfz_feedback_batch: null context");
    return HFZ_EINVAL;
  }
  if (small_step_ok(ctx, n_exec)) {  // small batch: scan + resolve as ONE cooperative launch
    if (!raw_maps || !virgin_inout || !edge_counts_inout || !admit_out || !sig_full_out || !sig_simple_out) {
      hfz_set_error("hfz_feedback_batch: null argument");
      return HFZ_EINVAL;
    }
    if (((uintptr_t)raw_maps | (uintptr_t)virgin_inout) & 15) {
      hfz_set_error("hfz_feedback_batch: raw_maps/virgin must be 16-byte aligned");
      return HFZ_EINVAL;
    }
    return small_step_scan(ctx, raw_maps, n_exec, virgin_inout, classed_out, sig_full_out, sig_simple_out, nnz_out,
                           ctx->delta, virgin_inout, edge_counts_inout, admit_out);
  }
  if (!edge_counts_inout || (n_exec && !admit_out)) {
    hfz_set_error("hfz_feedback_batch: null argument");
    return HFZ_EINVAL;
  }
  int rc = scan_dense(ctx, raw_maps, n_exec, virgin_inout, classed_out, sig_full_out, sig_simple_out, nnz_out, nullptr);
  if (rc) return rc;
  return hfz_feedback_fold_single(ctx, n_exec, virgin_inout, edge_counts_inout, admit_out);
}

// ---- dev / test entry: both signatures of an ordered entry list (slot | rung << 24) by the warp-parallel
// FNV of hfz_fnv.cuh, one warp.  Not part of include/hfz.h; tests/test_feedback_gpu.py::test_warp_fnv.
namespace {
__global__ void __launch_bounds__(32) hfz_k_dbg_warp_fnv(const uint32_t* __restrict__ entries, uint64_t n,
                                                         unsigned long long* __restrict__ out) {
  __shared__ __align__(16) uint32_t buf[kChainRound];
  __shared__ __align__(16) uint8_t stream[3072 + 16];
  const int lane = threadIdx.x;
  uint64_t hf = HFZ_FNV_OFFSET, hs = HFZ_FNV_OFFSET;
  for (uint64_t i0 = 0; i0 < n; i0 += kChainRound) {
    const uint32_t m = (uint32_t)(n - i0 < kChainRound ? n - i0 : kChainRound);
    for (uint32_t i = lane; i < m; i += 32) buf[i] = entries[i0 + i];
    __syncwarp();
    hf = pfnv::chain_entries<3>(hf, buf, m, stream, lane);
    hs = pfnv::chain_entries<2>(hs, buf, m, stream, lane);
    __syncwarp();
  }
  if (lane == 0) {
    out[0] = hf;
    out[1] = hs;
  }
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int hfz_dbg_warp_fnv(const uint32_t* entries_host, uint64_t n,
                                                                       uint64_t* out2_host) {
  uint32_t* d_e = nullptr;
  unsigned long long* d_o = nullptr;
  if (cudaMalloc(&d_e, (size_t)(n + 1) * 4) != cudaSuccess || cudaMalloc(&d_o, 16) != cudaSuccess) {
    cudaFree(d_e);
    return HFZ_ENOMEM;
  }
  cudaError_t e = cudaMemcpy(d_e, entries_host, (size_t)n * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    hfz_k_dbg_warp_fnv<<<1, 32>>>(d_e, n, d_o);
    e = cudaMemcpy(out2_host, d_o, 16, cudaMemcpyDeviceToHost);
  }
  cudaFree(d_e);
  cudaFree(d_o);
  return e == cudaSuccess ? HFZ_OK : hfz_cuda_fail(e, "hfz_dbg_warp_fnv");
}
