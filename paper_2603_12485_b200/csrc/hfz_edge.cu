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
//   * one CTA owns one execution; its 32,768 x u32 counter table lives in SHARED memory
//     (warp bumps are shared-memory atomics, flushed to HBM once per exec -- no global atomic
//     per hit); maps with more than 32,768 device slots fall back to global atomics;
//   * a real warp replays one simulated warp, real lane L <-> simulated lane L:
//       fast path   all active lanes walk the same site sequence (the SIMT common case):
//                   only the lowest lane can ever bump, every event of it does;
//       general     pass 1 counts visits per (site, lane) in a per-warp shared-memory table
//                   (site -> row by hashing, one column per lane), an exclusive prefix-max
//                   over lanes turns each row into M_L(s) = max_{L'<L} count_{L'}(s), pass 2
//                   replays the events and bumps the visits with k > M_L(s).  If a warp has
//                   more distinct sites than the table holds, the sites are partitioned by
//                   hash prefix and the passes repeat per partition (splitting on overflow).
#include "hfz_common.cuh"

namespace {

constexpr int kEdgeWarps = 4;
constexpr uint32_t kTC = 128;          // table rows per warp
constexpr uint32_t kTCFill = 96;       // split the partition when more rows than this are in use
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

struct WarpTable {
  unsigned long long* keys;  // [kTC]  0 = empty, else (1<<32 | site)
  uint32_t* cnt;             // [kTC][32]
};

// find-or-insert; returns row or kTC when the table is over its fill limit
__device__ __forceinline__ uint32_t table_insert(WarpTable& t, uint32_t site, uint32_t h, uint32_t* used) {
  const unsigned long long want = (1ull << 32) | site;
  uint32_t r = h & (kTC - 1);
  for (uint32_t probe = 0; probe < kTC; ++probe) {
    unsigned long long cur = t.keys[r];
    if (cur == want) return r;
    if (cur == 0) {
      const unsigned long long old = atomicCAS(&t.keys[r], 0ull, want);
      if (old == 0) {
        atomicAdd(used, 1u);
        return r;
      }
      if (old == want) return r;
    }
    r = (r + 1) & (kTC - 1);
  }
  return kTC;
}

__device__ __forceinline__ uint32_t table_find(const WarpTable& t, uint32_t site, uint32_t h) {
  const unsigned long long want = (1ull << 32) | site;
  uint32_t r = h & (kTC - 1);
  while (t.keys[r] != want) r = (r + 1) & (kTC - 1);  // present by construction
  return r;
}

template <bool SMEM_HIST>
__global__ void __launch_bounds__(kEdgeWarps * 32, 1) hfz_k_edge_record(const EdgeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* hist = SMEM_HIST ? reinterpret_cast<uint32_t*>(smem) : nullptr;
  uint8_t* wbase = smem + (SMEM_HIST ? (size_t)p.H * 4 : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpTable tab;
  tab.keys = reinterpret_cast<unsigned long long*>(wbase + (size_t)warp * (kTC * 8 + kTC * 32 * 4 + 64));
  tab.cnt = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(tab.keys) + kTC * 8);
  uint32_t* used = tab.cnt + kTC * 32;  // [1] rows in use (+ padding)
  __shared__ unsigned long long s_events;
  uint32_t* prev_tab = p.prev_scratch + (size_t)blockIdx.x * p.prev_stride;
  const uint32_t hmask = p.H - 1;

  for (uint64_t e = blockIdx.x; e < p.n_exec; e += gridDim.x) {
    uint32_t* ghist = reinterpret_cast<uint32_t*>(p.raw + e * p.rec_bytes + p.H);
    uint32_t* counters = SMEM_HIST ? hist : ghist;
    for (uint32_t i = threadIdx.x; i < p.H; i += blockDim.x) counters[i] = 0;
    if (threadIdx.x == 0) s_events = 0;
    const uint64_t l0 = p.launch_off[e], l1 = p.launch_off[e + 1];
    // prev is carried across launches per flattened gtid (hdvm.cpp:376,426-430): only needed
    // when the exec has more than one launch
    const bool multi = l1 - l0 > 1;
    if (multi) {
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

    uint64_t my_events = 0;
    for (uint64_t l = l0; l < l1; ++l) {
      const uint32_t* d = p.dims + l * 6;
      if (launch_valid(d)) {
        const uint64_t gx = d[0], gy = d[1], bdx = d[3], bdy = d[4], bdz = d[5];
        const uint64_t tpb = bdx * bdy * bdz, blocks = gx * gy * (uint64_t)d[2];
        const uint64_t wpb = (tpb + 31) / 32;
        const uint64_t t0 = p.thread_off[l];
        for (uint64_t sw = warp; sw < blocks * wpb; sw += kEdgeWarps) {
          const uint64_t bl = sw / wpb, tl = (sw % wpb) * 32 + lane;
          const bool active = tl < tpb;
          uint64_t e0 = 0, e1 = 0, gtid = 0;
          if (active) {
            const uint64_t t = t0 + bl * tpb + tl;
            e0 = p.ev_off[t];
            e1 = p.ev_off[t + 1];
            const uint64_t bx = bl % gx, by = (bl / gx) % gy, bz = bl / (gx * gy);
            const uint64_t tx = tl % bdx, ty = (tl / bdx) % bdy, tz = tl / (bdx * bdy);
            gtid = tx + bx * bdx + ty * (bdx * gx) + by * (bdx * bdy * gx) + tz * (bdx * bdy * gx * gy) +
                   bz * (bdx * bdy * bdz * gx * gy);
          }
          const uint32_t n_ev = (uint32_t)(e1 - e0);
          uint32_t prev0 = (multi && active) ? prev_tab[gtid] : 0;
          const uint32_t amask = __ballot_sync(0xffffffffu, active);
          const int lead = __ffs(amask) - 1;  // lowest active lane (always lane 0 of the sim warp)

          // ---- fast path: every active lane walks the same sequence
          const uint32_t n_lead = __shfl_sync(0xffffffffu, n_ev, lead);
          bool same = __all_sync(0xffffffffu, !active || n_ev == n_lead);
          if (same) {
            for (uint32_t i = 0; i < n_lead; ++i) {
              const uint32_t s = active ? p.sites[e0 + i] : 0;
              const uint32_t sl = __shfl_sync(0xffffffffu, s, lead);
              if (!__all_sync(0xffffffffu, !active || s == sl)) {
                same = false;
                break;
              }
            }
          }
          if (same) {
            if (lane == lead) {
              uint32_t pv = prev0;
              for (uint32_t i = 0; i < n_lead; ++i) {
                const uint32_t s = p.sites[e0 + i];
                bump(&counters[(pv ^ s) & hmask]);
                pv = s >> 1;
              }
              my_events += n_lead;
            }
            if (multi && active && n_ev) prev_tab[gtid] = p.sites[e1 - 1] >> 1;
            continue;
          }

          // ---- general path: partitions of the site space by hash prefix, explicit stack
          uint32_t stk_prefix[34], stk_depth[34];
          int sp = 0;
          stk_prefix[0] = 0;
          stk_depth[0] = 0;
          sp = 1;
          while (sp > 0) {
            --sp;
            const uint32_t prefix = stk_prefix[sp], depth = stk_depth[sp];
            // reset table
            for (uint32_t i = lane; i < kTC; i += 32) tab.keys[i] = 0;
            for (uint32_t i = lane; i < kTC * 32 / 4; i += 32)
              reinterpret_cast<uint4*>(tab.cnt)[i] = make_uint4(0, 0, 0, 0);
            if (lane == 0) *used = 0;
            __syncwarp();
            // pass 1: count visits per (site row, lane column)
            bool overflow = false;
            for (uint32_t i = 0; i < n_ev; ++i) {
              const uint32_t s = p.sites[e0 + i];
              const uint32_t h = mix32(s);
              if (depth && (h >> (32 - depth)) != prefix) continue;
              const uint32_t r = table_insert(tab, s, h, used);
              if (r == kTC) {
                overflow = true;
                break;
              }
              tab.cnt[r * 32 + lane] += 1;
            }
            __syncwarp();
            overflow = __any_sync(0xffffffffu, overflow) || (*used > kTCFill && depth < 32);
            if (overflow) {  // split this partition in two and retry (depth 32 = a single site)
              stk_prefix[sp] = prefix * 2 + 1;
              stk_depth[sp] = depth + 1;
              stk_prefix[sp + 1] = prefix * 2;
              stk_depth[sp + 1] = depth + 1;
              sp += 2;
              __syncwarp();
              continue;
            }
            // rows in use -> exclusive prefix-max over lanes: cnt[r][L] := max_{L'<L} cnt[r][L']
            for (uint32_t r0 = 0; r0 < kTC; r0 += 32) {
              uint32_t occ = __ballot_sync(0xffffffffu, tab.keys[r0 + lane] != 0);
              while (occ) {
                const uint32_t r = r0 + __ffs(occ) - 1;
                occ &= occ - 1;
                uint32_t c = tab.cnt[r * 32 + lane];
#pragma unroll
                for (int d2 = 1; d2 < 32; d2 <<= 1) {
                  const uint32_t o = __shfl_up_sync(0xffffffffu, c, d2);
                  if (lane >= d2) c = max(c, o);
                }
                const uint32_t excl = __shfl_up_sync(0xffffffffu, c, 1);
                tab.cnt[r * 32 + lane] = lane ? excl : 0;
              }
            }
            __syncwarp();
            // pass 2: replay; the first M visits of a site by this lane do not bump
            uint32_t pv = prev0;
            for (uint32_t i = 0; i < n_ev; ++i) {
              const uint32_t s = p.sites[e0 + i];
              const uint32_t h = mix32(s);
              if (!depth || (h >> (32 - depth)) == prefix) {
                const uint32_t r = table_find(tab, s, h);
                const uint32_t m = tab.cnt[r * 32 + lane];
                if (m) {
                  tab.cnt[r * 32 + lane] = m - 1;
                } else {
                  bump(&counters[(pv ^ s) & hmask]);
                  ++my_events;
                }
              }
              pv = s >> 1;
            }
            __syncwarp();
          }
          if (multi && active && n_ev) prev_tab[gtid] = p.sites[e1 - 1] >> 1;
        }
      }
      __syncthreads();  // prev table and counters are launch-ordered
    }
    // block-reduce the event tally, flush the counters (copy, merge_device_into_map)
    if (my_events) atomicAdd(&s_events, (unsigned long long)my_events);
    __syncthreads();
    if (SMEM_HIST) {
      uint4* dst = reinterpret_cast<uint4*>(ghist);
      const uint4* src = reinterpret_cast<const uint4*>(hist);
      for (uint32_t i = threadIdx.x; i < p.H / 4; i += blockDim.x) dst[i] = src[i];
    }
    if (threadIdx.x == 0 && p.warp_events) p.warp_events[e] = s_events;
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

extern "C" int hfz_edge_record_batch(hfz_ctx* ctx, const uint64_t* launch_off, const uint32_t* dims,
                                     const uint64_t* thread_off, const uint64_t* ev_off,
                                     const uint32_t* sites, uint64_t n_exec, uint64_t n_launch,
                                     uint8_t* raw_maps, uint64_t* warp_events_out) {
  if (!ctx || (n_exec && (!launch_off || !raw_maps)) ||
      (n_launch && (!dims || !thread_off || !ev_off))) {
    hfz_set_error("hfz_edge_record_batch: null argument");
    return HFZ_EINVAL;
  }
  if (n_exec == 0) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  // size the per-CTA prev table from the launch geometry (one small D2H read)
  unsigned long long* d_mx = nullptr;
  unsigned long long mx = 0;
  HFZ_CUDA(cudaMalloc(&d_mx, sizeof(unsigned long long)));
  cudaError_t e = cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long), ctx->stream);
  if (e == cudaSuccess && n_launch) {
    hfz_k_edge_max_threads<<<64, 256, 0, ctx->stream>>>(dims, n_launch, d_mx);
    ++ctx->launches;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&mx, d_mx, sizeof(mx), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d_mx);
  if (e != cudaSuccess) return hfz_cuda_fail(e, "hfz_edge_record_batch(prepare)");

  uint32_t grid = (uint32_t)(n_exec < (uint64_t)ctx->num_sms ? n_exec : (uint64_t)ctx->num_sms);
  const uint64_t stride = mx ? mx : 1;
  uint32_t* d_prev = nullptr;
  if (cudaMalloc(&d_prev, (size_t)grid * stride * sizeof(uint32_t)) != cudaSuccess) {
    hfz_set_error("hfz_edge_record_batch: prev table allocation failed (%llu bytes)",
                  (unsigned long long)grid * stride * 4);
    return HFZ_ENOMEM;
  }
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
  const size_t wsmem = (size_t)kEdgeWarps * (kTC * 8 + kTC * 32 * 4 + 64);
  const bool smem_hist = ctx->H <= kSmemSlots;
  const size_t smem = wsmem + (smem_hist ? (size_t)ctx->H * 4 : 0);
  if (smem_hist) {
    e = cudaFuncSetAttribute(hfz_k_edge_record<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) hfz_k_edge_record<true><<<grid, kEdgeWarps * 32, smem, ctx->stream>>>(p);
  } else {
    e = cudaFuncSetAttribute(hfz_k_edge_record<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) hfz_k_edge_record<false><<<grid, kEdgeWarps * 32, smem, ctx->stream>>>(p);
  }
  ++ctx->launches;
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // d_prev must outlive the kernel
  cudaFree(d_prev);
  if (e != cudaSuccess) return hfz_cuda_fail(e, "hfz_edge_record_batch");
  return HFZ_OK;
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
