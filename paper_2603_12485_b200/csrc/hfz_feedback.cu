// hfz_feedback.cu -- K2 fused feedback scan, K2b first-occurrence resolve, K4 virgin merge.
//
// Reference semantics being reproduced (paths under /root/reference/proj):
//   classify_trace  src/coverage.cpp:58-72      trace_signature  src/coverage.cpp:89-97
//   has_new_bits    src/coverage.cpp:74-87      VirginMap::observe include/hetfuzz/coverage.hpp:166-174
//   per-exec order  src/engine.cpp:471-478
//
// Design (DESIGN.md has the long form):
//  * scan: ONE pass over the raw maps.  A warp owns 32 maps, one per lane ("lane-per-map"):
//    the FNV-1a signature is a strictly serial 64-bit chain per map, so the only way to keep
//    all 32 lanes of a warp busy on it is to run 32 independent chains.  Every lane pulls its
//    own map chunk by chunk into a padded shared-memory slot with a 1-D TMA bulk copy
//    (cp.async.bulk + mbarrier, STAGES deep), builds a non-zero bitmask of the chunk with
//    128-bit shared loads, and then only visits the ~2% non-zero slots: classify, look the
//    virgin byte up in the shared-memory copy of V0 (TMA-staged once per CTA), advance both
//    hash chains.  Nothing is written back except 21 bytes per map.
//  * exact sequential has_new_bits without a sequential pass: for every (slot, class bit) not
//    in V0 the scan records the FIRST exec that shows it (atomicMin into `first`).  An exec's
//    Admit code then only depends on whether it is that first exec (resolve kernel, runs on
//    the few candidate maps only).  Final virgin = V0 | OR of the novelty deltas (merge).
#include <stdio.h>

#include "hfz_common.cuh"

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
  uint32_t* cand_list;
  uint32_t* cand_count;
  uint64_t* sig_full;
  uint64_t* sig_simple;
  uint32_t* nnz;
  uint8_t* classed;
  uint32_t n_groups;
};

// non-zero-byte bitmask (4 bits) of a 32-bit word
__device__ __forceinline__ uint32_t nz_bytes(uint32_t w) {
  uint32_t t = (((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) & 0x80808080u;  // bit 7 of each non-zero byte
  return (t * 0x00204081u) >> 28;                                      // gather to bits 0..3
}

template <bool VSMEM, bool CLASSED>
struct Lane {
  uint64_t hf, hs;
  uint32_t nnz, novel;
  __device__ __forceinline__ void visit(uint32_t idx, uint32_t klass, const uint8_t* virgin,
                                        uint32_t* first, uint32_t e, uint8_t* classed_row) {
    const uint32_t b0 = idx & 0xffu, b1 = (idx >> 8) & 0xffu;
    hf = hfz_fnv(hfz_fnv(hfz_fnv(hf, b0), b1), klass);
    hs = hfz_fnv(hfz_fnv(hs, b0), b1);
    const uint32_t known = VSMEM ? (uint32_t)virgin[idx] : (uint32_t)__ldg(virgin + idx);
    ++nnz;
    if (klass & ~known) {
      novel = 1;
      atomicMin(first + (size_t)idx * 8 + (31 - __clz(klass)), e);
    }
    if (CLASSED) classed_row[idx] = (uint8_t)klass;
  }
};

// Process one staged chunk of CHUNK bytes belonging to this lane's map.
template <int CHUNK, bool HOST, bool VSMEM, bool CLASSED>
__device__ __forceinline__ void scan_chunk(const uint8_t* chunk, uint32_t slot_base,
                                           Lane<VSMEM, CLASSED>& st, const uint8_t* virgin,
                                           uint32_t* first, uint32_t e, uint8_t* classed_row) {
  constexpr int NV = CHUNK / 16;  // uint4 per chunk
  constexpr int NQ = CHUNK / 256; // 64-word mask registers
  static_assert(NQ == 1 || NQ == 2, "CHUNK must be 256 or 512");
  const uint4* c4 = reinterpret_cast<const uint4*>(chunk);
  const uint32_t* c1 = reinterpret_cast<const uint32_t*>(chunk);
  uint64_t mk[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = c4[q * 16 + i];
      lo |= ((v.x != 0u) | ((v.y != 0u) << 1) | ((v.z != 0u) << 2) | ((v.w != 0u) << 3)) << (4 * i);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = c4[q * 16 + 8 + i];
      hi |= ((v.x != 0u) | ((v.y != 0u) << 1) | ((v.z != 0u) << 2) | ((v.w != 0u) << 3)) << (4 * i);
    }
    mk[q] = ((uint64_t)hi << 32) | lo;
  }
  (void)NV;
  uint64_t A = mk[0], B = NQ == 2 ? mk[NQ - 1] : 0ull;
  uint32_t base = 0;
  uint32_t w = 0, bm = 0, wpos = 0;
  for (;;) {
    if (bm == 0) {
      if (NQ == 2 && A == 0) {
        A = B;
        B = 0;
        base = 64;
      }
      if (A == 0) break;
      const uint32_t p = __ffsll((long long)A) - 1;
      A &= A - 1;
      wpos = base + p;
      w = c1[wpos];
      bm = HOST ? nz_bytes(w) : 1u;
    }
    if (HOST) {
      const uint32_t j = __ffs(bm) - 1;
      bm &= bm - 1;
      const uint32_t c = (w >> (8 * j)) & 0xffu;
      st.visit(slot_base + wpos * 4 + j, hfz_class_host(c), virgin, first, e, classed_row);
    } else {
      bm = 0;
      st.visit(slot_base + wpos, hfz_class_device(w), virgin, first, e, classed_row);
    }
  }
}

template <int CHUNK, int STAGES, bool VSMEM, bool CLASSED>
__global__ void __launch_bounds__(1024, 1) hfz_k_scan(const ScanParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int SLOT = CHUNK + kPad;
  constexpr int STAGE_BYTES = 32 * SLOT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;

  uint8_t* s_virgin = smem;
  uint8_t* s_stage = smem + (VSMEM ? p.S : 0) + (size_t)warp * STAGES * STAGE_BYTES;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + (VSMEM ? p.S : 0) +
                                                (size_t)nwarps * STAGES * STAGE_BYTES);
  uint64_t* bar_virgin = s_bar;                     // [1]
  uint64_t* bar = s_bar + 1 + warp * STAGES;        // [STAGES] per warp

  if (threadIdx.x == 0) hfz_mbar_init(bar_virgin, 1);
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) hfz_mbar_init(bar + s, 1);
  hfz_fence_barrier_init();
  __syncthreads();

  if (VSMEM && threadIdx.x == 0) {
    // stage V0 in shared memory: one TMA bulk copy per 16 KB, kept in L2 for the other CTAs
    const uint64_t pol = hfz_policy_evict_last();
    hfz_mbar_expect_tx(bar_virgin, p.S);
    for (uint32_t off = 0; off < p.S; off += 16384u) {
      const uint32_t n = p.S - off < 16384u ? p.S - off : 16384u;
      hfz_bulk_g2s_stream(s_virgin + off, p.v0 + off, n, bar_virgin, pol);
    }
  }

  const uint64_t stream_pol = hfz_policy_evict_first();
  const uint32_t rows_host = p.H / CHUNK;
  const uint32_t rows = (uint32_t)(p.rec_bytes / CHUNK);
  const uint32_t total_warps = gridDim.x * nwarps;
  uint32_t it_issue = 0, it_wait = 0;  // running stage counters over the warp's lifetime
  const uint8_t* virgin = VSMEM ? s_virgin : p.v0;
  bool virgin_ready = !VSMEM;

  for (uint32_t g = blockIdx.x + gridDim.x * warp; g < p.n_groups; g += total_warps) {
    const uint64_t e64 = (uint64_t)g * 32 + lane;
    const bool valid = e64 < p.n_exec;
    const uint32_t e = (uint32_t)e64;
    const uint8_t* src = p.raw + (valid ? e64 : 0) * p.rec_bytes;
    const uint32_t n_valid = (uint32_t)min((uint64_t)32, p.n_exec - (uint64_t)g * 32);
    uint8_t* classed_row = CLASSED ? p.classed + e64 * p.S : nullptr;

    Lane<VSMEM, CLASSED> st;
    st.hf = HFZ_FNV_OFFSET;
    st.hs = HFZ_FNV_OFFSET;
    st.nnz = 0;
    st.novel = 0;

    auto issue = [&](uint32_t row) {
      const uint32_t s = it_issue % STAGES;
      if (lane == 0) hfz_mbar_expect_tx(bar + s, n_valid * CHUNK);
      __syncwarp();
      if (valid)
        hfz_bulk_g2s_stream(s_stage + s * STAGE_BYTES + lane * SLOT, src + (size_t)row * CHUNK,
                            CHUNK, bar + s, stream_pol);
      ++it_issue;
    };

    const uint32_t pre = rows < (uint32_t)(STAGES - 1) ? rows : (uint32_t)(STAGES - 1);
    for (uint32_t r = 0; r < pre; ++r) issue(r);

    if (!virgin_ready) {
      hfz_mbar_wait(bar_virgin, 0);
      virgin_ready = true;
    }

    for (uint32_t r = 0; r < rows; ++r) {
      // the stage refilled here was consumed in iteration r-1 (all lanes passed __syncwarp)
      if (r + STAGES - 1 < rows) issue(r + STAGES - 1);
      const uint32_t s = it_wait % STAGES;
      hfz_mbar_wait(bar + s, (it_wait / STAGES) & 1u);
      ++it_wait;
      if (valid) {
        const uint8_t* chunk = s_stage + s * STAGE_BYTES + lane * SLOT;
        if (r < rows_host)
          scan_chunk<CHUNK, true, VSMEM, CLASSED>(chunk, r * CHUNK, st, virgin, p.first, e,
                                                  classed_row);
        else
          scan_chunk<CHUNK, false, VSMEM, CLASSED>(chunk, p.H + (r - rows_host) * (CHUNK / 4), st,
                                                   virgin, p.first, e, classed_row);
      }
      __syncwarp();
      hfz_fence_proxy_async();
    }

    if (valid) {
      p.sig_full[e64] = st.hf;
      p.sig_simple[e64] = st.hs;
      if (p.nnz) p.nnz[e64] = st.nnz;
    }
    // warp-aggregated append of the candidate execs
    const uint32_t cm = __ballot_sync(0xffffffffu, valid && st.novel);
    if (cm) {
      uint32_t basei = 0;
      if (lane == 0) basei = atomicAdd(p.cand_count, __popc(cm));
      basei = __shfl_sync(0xffffffffu, basei, 0);
      if (valid && st.novel) p.cand_list[basei + __popc(cm & ((1u << lane) - 1u))] = e;
    }
  }
  if (!virgin_ready) hfz_mbar_wait(bar_virgin, 0);  // never leave a bulk copy in flight
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

// ---------------------------------------------------------------------------
// K2b: exact Admit codes of the candidate execs.  One warp per candidate map.
struct ResolveParams {
  const uint8_t* raw;
  uint64_t rec_bytes;
  uint32_t S, H;
  const uint8_t* prior;     // P_r
  const uint32_t* first;
  const uint32_t* cand_list;
  const uint32_t* cand_count;
  uint8_t* admit;
};

__device__ __forceinline__ uint32_t first_any(const uint32_t* first, uint32_t idx) {
  const uint4* f = reinterpret_cast<const uint4*>(first + (size_t)idx * 8);
  const uint4 a = f[0], b = f[1];
  return min(min(min(a.x, a.y), min(a.z, a.w)), min(min(b.x, b.y), min(b.z, b.w)));
}

__device__ __forceinline__ uint32_t resolve_entry(const ResolveParams& p, uint32_t idx,
                                                  uint32_t klass, uint32_t e) {
  const uint32_t pr = __ldg(p.prior + idx);
  if (!(klass & ~pr)) return 0;
  if (p.first[(size_t)idx * 8 + (31 - __clz(klass))] != e) return 0;  // an earlier exec had it
  if (pr == 0 && first_any(p.first, idx) == e) return 2;              // slot never seen before e
  return 1;
}

__global__ void __launch_bounds__(256) hfz_k_resolve(const ResolveParams p) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t total_warps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t n = *p.cand_count;
  for (uint32_t i = warp; i < n; i += total_warps) {
    const uint32_t e = p.cand_list[i];
    const uint8_t* src = p.raw + (uint64_t)e * p.rec_bytes;
    uint32_t flags = 0;
    const uint4* h4 = reinterpret_cast<const uint4*>(src);
    for (uint32_t v = lane; v < p.H / 16; v += 32) {
      const uint4 x = hfz_ldg_stream(h4 + v);
      if ((x.x | x.y | x.z | x.w) == 0u) continue;
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t bm = nz_bytes(w[k]);
        while (bm) {
          const uint32_t j = __ffs(bm) - 1;
          bm &= bm - 1;
          flags |= resolve_entry(p, v * 16 + k * 4 + j, hfz_class_host((w[k] >> (8 * j)) & 0xffu), e);
        }
      }
    }
    const uint4* d4 = reinterpret_cast<const uint4*>(src + p.H);
    for (uint32_t v = lane; v < p.H / 4; v += 32) {
      const uint4 x = hfz_ldg_stream(d4 + v);
      if ((x.x | x.y | x.z | x.w) == 0u) continue;
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (w[k]) flags |= resolve_entry(p, p.H + v * 4 + k, hfz_class_device(w[k]), e);
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0) p.admit[e] = (flags & 2u) ? 2 : ((flags & 1u) ? 1 : 0);
  }
}

// ---------------------------------------------------------------------------
// launch plumbing

template <int CHUNK, int STAGES>
size_t scan_smem_bytes(uint32_t S, bool vsmem, int warps) {
  return (vsmem ? S : 0) + (size_t)warps * STAGES * 32 * (CHUNK + kPad) + (1 + warps * STAGES) * 8;
}

template <int CHUNK, int STAGES, bool VSMEM, bool CLASSED>
int launch_scan_t(hfz_ctx* ctx, const ScanParams& p, int warps) {
  auto kern = hfz_k_scan<CHUNK, STAGES, VSMEM, CLASSED>;
  const size_t smem = scan_smem_bytes<CHUNK, STAGES>(p.S, VSMEM, warps);
  HFZ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  uint32_t grid = (uint32_t)ctx->num_sms;
  if (grid > p.n_groups) grid = p.n_groups;
  kern<<<grid, warps * 32, smem, ctx->stream>>>(p);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

template <int CHUNK, int STAGES>
int launch_scan_v(hfz_ctx* ctx, const ScanParams& p, bool vsmem, int warps) {
  const bool classed = p.classed != nullptr;
  if (vsmem)
    return classed ? launch_scan_t<CHUNK, STAGES, true, true>(ctx, p, warps)
                   : launch_scan_t<CHUNK, STAGES, true, false>(ctx, p, warps);
  return classed ? launch_scan_t<CHUNK, STAGES, false, true>(ctx, p, warps)
                 : launch_scan_t<CHUNK, STAGES, false, false>(ctx, p, warps);
}

template <int CHUNK, int STAGES>
int max_warps(const hfz_ctx* ctx, uint32_t S, bool vsmem) {
  int w = 32;
  while (w > 0 && scan_smem_bytes<CHUNK, STAGES>(S, vsmem, w) > (size_t)ctx->max_smem_optin) --w;
  return w;
}

// pick the warp count (<= cap) that wastes the least of the last wave
int pick_warps(const hfz_ctx* ctx, uint32_t n_groups, int cap) {
  if (ctx->scan_warps > 0) return ctx->scan_warps < cap ? ctx->scan_warps : cap;
  int best = cap;
  double best_eff = 0;
  for (int w = cap; w >= (cap + 1) / 2 && w >= 1; --w) {
    const double workers = (double)ctx->num_sms * w;
    const double waves = n_groups / workers;
    const double eff = waves / (double)(uint64_t)(waves + 0.999999);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = w;
    }
  }
  return best;
}

int ensure_cand(hfz_ctx* ctx, uint64_t n_exec) {
  if (ctx->cand_cap >= n_exec) return HFZ_OK;
  if (ctx->cand_list) cudaFree(ctx->cand_list);
  ctx->cand_list = nullptr;
  ctx->cand_cap = 0;
  const uint64_t cap = n_exec < 1024 ? 1024 : n_exec;
  if (cudaMalloc(&ctx->cand_list, cap * sizeof(uint32_t)) != cudaSuccess) {
    hfz_set_error("cudaMalloc(cand_list, %llu) failed", (unsigned long long)cap * 4);
    return HFZ_ENOMEM;
  }
  ctx->cand_cap = cap;
  return HFZ_OK;
}

}  // namespace

extern "C" int hfz_feedback_scan(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                                 const uint8_t* virgin_v0, uint8_t* classed_out,
                                 uint64_t* sig_full_out, uint64_t* sig_simple_out,
                                 uint32_t* nnz_out, uint8_t* delta_out) {
  if (!ctx || !virgin_v0 || !delta_out || (n_exec && (!raw_maps || !sig_full_out || !sig_simple_out))) {
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
  int rc = ensure_cand(ctx, n_exec);
  if (rc) return rc;
  HFZ_CUDA(cudaMemsetAsync(ctx->first, 0xff, (size_t)ctx->S * 8 * sizeof(uint32_t), ctx->stream));
  HFZ_CUDA(cudaMemsetAsync(ctx->cand_count, 0, sizeof(uint32_t), ctx->stream));
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
    p.cand_list = ctx->cand_list;
    p.cand_count = ctx->cand_count;
    p.sig_full = sig_full_out;
    p.sig_simple = sig_simple_out;
    p.nnz = nnz_out;
    p.classed = classed_out;
    p.n_groups = (uint32_t)((n_exec + 31) / 32);
    // virgin copy in shared memory whenever it leaves room for the staging ring
    const bool vsmem = ctx->S <= 65536u;
    int variant = ctx->scan_variant;
    if (variant == 0) variant = 1;
    int cap;
    switch (variant) {
      case 1: cap = max_warps<256, 3>(ctx, p.S, vsmem); break;
      case 2: cap = max_warps<256, 4>(ctx, p.S, vsmem); break;
      case 3: cap = max_warps<512, 2>(ctx, p.S, vsmem); break;
      case 4: cap = max_warps<512, 3>(ctx, p.S, vsmem); break;
      case 5: cap = max_warps<256, 2>(ctx, p.S, vsmem); break;
      default:
        hfz_set_error("unknown scan_variant %d", variant);
        return HFZ_EINVAL;
    }
    if (cap < 1) {
      hfz_set_error("scan: shared memory too small for map size %u", p.S);
      return HFZ_EINVAL;
    }
    const int warps = pick_warps(ctx, p.n_groups, cap);
    switch (variant) {
      case 1: rc = launch_scan_v<256, 3>(ctx, p, vsmem, warps); break;
      case 2: rc = launch_scan_v<256, 4>(ctx, p, vsmem, warps); break;
      case 3: rc = launch_scan_v<512, 2>(ctx, p, vsmem, warps); break;
      case 4: rc = launch_scan_v<512, 3>(ctx, p, vsmem, warps); break;
      case 5: rc = launch_scan_v<256, 2>(ctx, p, vsmem, warps); break;
    }
    if (rc) return rc;
  }
  hfz_k_delta<<<(ctx->S + 255) / 256, 256, 0, ctx->stream>>>(ctx->first, delta_out, ctx->S);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
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

extern "C" int hfz_feedback_resolve(hfz_ctx* ctx, const uint8_t* raw_maps, uint64_t n_exec,
                                    uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                                    const uint8_t* deltas, uint32_t n_ranks, uint32_t rank,
                                    uint8_t* admit_out) {
  if (!ctx || !virgin_inout || !edge_counts_inout || !deltas || n_ranks == 0 || rank >= n_ranks ||
      (n_exec && (!raw_maps || !admit_out))) {
    hfz_set_error("hfz_feedback_resolve: bad argument");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  hfz_k_merge<<<(ctx->S / 16 + 255) / 256, 256, 0, ctx->stream>>>(
      virgin_inout, deltas, n_ranks, rank, ctx->prior,
      reinterpret_cast<unsigned long long*>(edge_counts_inout), ctx->S, ctx->H);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  if (n_exec) {
    HFZ_CUDA(cudaMemsetAsync(admit_out, 0, n_exec, ctx->stream));
    ResolveParams p;
    p.raw = raw_maps;
    p.rec_bytes = ctx->rec_bytes;
    p.S = ctx->S;
    p.H = ctx->H;
    p.prior = ctx->prior;
    p.first = ctx->first;
    p.cand_list = ctx->cand_list;
    p.cand_count = ctx->cand_count;
    p.admit = admit_out;
    uint64_t blocks = (n_exec + 7) / 8;  // 8 warps per block, at most one warp per exec
    const uint64_t maxb = (uint64_t)ctx->num_sms * 8;
    if (blocks > maxb) blocks = maxb;
    hfz_k_resolve<<<(uint32_t)blocks, 256, 0, ctx->stream>>>(p);
    ++ctx->launches;
    HFZ_CUDA(cudaGetLastError());
  }
  return HFZ_OK;
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
  int rc = hfz_feedback_scan(ctx, raw_maps, n_exec, virgin_inout, classed_out, sig_full_out,
                             sig_simple_out, nnz_out, ctx->delta);
  if (rc) return rc;
  return hfz_feedback_resolve(ctx, raw_maps, n_exec, virgin_inout, edge_counts_inout, ctx->delta, 1,
                              0, admit_out);
}
