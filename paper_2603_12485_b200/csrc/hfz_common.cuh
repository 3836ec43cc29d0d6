// hfz_common.cuh -- shared device helpers and the context struct (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <vector>

#include "../../include/hfz.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "hfz kernels are written for sm_100a (B200) only"
#endif

// ---------------------------------------------------------------------------
// Context

struct hfz_ctx {
  int device = 0;
  uint32_t S = 0;          // logical slots
  uint32_t H = 0;          // S / 2
  uint64_t rec_bytes = 0;  // 5 * H
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  int max_smem_optin = 0;
  uint64_t launches = 0;

  // K2 scratch (owned)
  uint32_t* first = nullptr;      // [S * 8] first local exec index showing (slot, class bit); ~0u = none
  uint32_t* admit_flags = nullptr; // [admit_cap] per-exec novelty flags of the table resolve (1 = NewCounts, 2 = NewEdges); zero between calls
  uint64_t admit_cap = 0;
  uint8_t* prior = nullptr;        // [S] P_r = V0 | OR_{q<r} D_q
  uint8_t* delta = nullptr;        // [S] this rank's delta (hfz_feedback_batch)
  uint8_t* v0 = nullptr;           // [S] batch-start snapshot

  // K1 scratch (owned, grow-only)
  uint32_t* edge_prev = nullptr;
  uint64_t edge_prev_words = 0;
  unsigned long long* d_small = nullptr;  // [32] small device scalars
  // K1 flat path (hfz_edge.cu: decide + count; owned, grow-only)
  int edge_flat = 1;               // 0 = every exec through the per-exec kernel
  int64_t edge_scratch_mb = 2048;  // bump-list scratch per chunk of execs (4 bytes per trace event of the chunk)
  uint32_t* fl_nsw = nullptr;      uint64_t fl_nsw_cap = 0;
  uint64_t* fl_sw_off = nullptr;   uint64_t fl_sw_off_cap = 0;
  uint32_t* fl_l_exec = nullptr;   uint64_t fl_l_exec_cap = 0;
  uint8_t* fl_elig = nullptr;      uint64_t fl_elig_cap = 0;
  uint64_t* fl_exec_ev0 = nullptr; uint64_t fl_exec_ev0_cap = 0;
  uint64_t* fl_exec_sw0 = nullptr; uint64_t fl_exec_sw0_cap = 0;
  uint32_t* fl_inelig = nullptr;   uint64_t fl_inelig_cap = 0;
  uint32_t* fl_scratch = nullptr;  uint64_t fl_scratch_cap = 0;
  uint64_t* fl_rec_first = nullptr; uint64_t fl_rec_first_cap = 0;
  uint32_t* fl_rec_cnt = nullptr;  uint64_t fl_rec_cnt_cap = 0;
  uint32_t* fl_div = nullptr;      uint64_t fl_div_cap = 0;
  uint32_t* fl_lines = nullptr;    uint64_t fl_lines_cap = 0;

  // K3 scratch (owned, grow-only): edit lists of one chunk of slots, 528 bytes per slot (hfz_mutate.cu)
  uint64_t* hv_ops = nullptr;
  uint64_t hv_ops_cap = 0;  // slots

  // host-buffer path staging (owned, lazily allocated)
  uint8_t* stage_raw[2] = {nullptr, nullptr};
  uint64_t stage_execs = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_stream = nullptr;  // orders a new stream after the old one (hfz_ctx_set_stream)
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_done[2] = {nullptr, nullptr};
  uint8_t* d_virgin = nullptr;
  uint64_t* d_counts = nullptr;
  uint8_t* d_admit = nullptr;
  uint64_t* d_sigf = nullptr;
  uint64_t* d_sigs = nullptr;
  uint32_t* d_nnz = nullptr;
  uint8_t* d_classed = nullptr;
  uint64_t d_out_cap = 0;
  uint64_t d_classed_cap = 0;

  // sparse ingest (hfz_sparse.cu; owned, lazily allocated)
  uint8_t* sp_dense = nullptr;     // dense expansion staging, all-zero between calls
  uint64_t sp_dense_execs = 0;     // records it holds
  bool sp_dirty = false;           // an error path left entries behind: memset before reuse
  uint64_t sparse_chunk = 0;       // execs expanded per chunk (0 = ~1.25 GB of records)
  uint32_t* sp_entries = nullptr;  // device copy of host (slot, count) pairs
  uint64_t sp_entries_cap = 0;     // pairs
  uint64_t* sp_off = nullptr;
  uint64_t sp_off_cap = 0;
  uint32_t* sp_compact = nullptr;  // device copy of host compact pairs (slot | count << 16)
  uint64_t sp_compact_cap = 0;
  uint64_t* sp_coff = nullptr;
  uint64_t sp_coff_cap = 0;
  uint32_t* sp_h3 = nullptr;       // device copy of a packed host-half list (3 bytes per entry), in words
  uint64_t sp_h3_cap = 0;
  std::vector<cudaEvent_t> sp_events;  // one "entries of chunk k copied" event per chunk
  int sparse_native = 1;           // 1 = rank + chain kernels on the lists (S <= 65,536), 0 = expand to dense records
  uint32_t* sp_sorted = nullptr;   // per pair: slot | rung << 24, ascending slots inside an exec
  uint64_t sp_sorted_cap = 0;
  uint32_t* sp_cnt = nullptr;      // per exec: distinct non-zero slots
  uint64_t sp_cnt_cap = 0;

  // tuning
  int scan_warps = 0;     // 0 = as many as fit
  int scan_row = 0;       // bytes per map per row: 0 = auto, 256 (18 warps/SM), 512 (9 warps/SM) or 1024 (16 maps per warp)
  int scan_prefetch = 1;  // L2 prefetch of the row after next
  int virgin_smem = 1;    // stage V0 in shared memory when it fits
  int time_scan = 0;      // bracket scan launches with events (bench roofline)
  int64_t scan_small = -1; // batches up to this many execs use the warp-per-map kernel (-1 = auto)
  int64_t scan_pipe = -1;  // batches of up to this many 32-map groups per SM use the pipelined kernel (-1 = auto)
  int64_t scan_two_stage = -1;  // batches of up to this many execs use compact + chain (-1 = auto, 0 = off)
  uint32_t* ts_sorted = nullptr;  // two-stage scratch: [n_exec][S] entries (only the used prefix of each piece is touched)
  uint64_t ts_sorted_cap = 0;     // entries
  uint32_t* ts_cnt = nullptr;     // [n_exec][pieces] entries per piece
  uint64_t ts_cnt_cap = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> scan_events;

  // fused small step (hfz_k_small_step, hfz_feedback.cu; owned, lazily allocated)
  int small_fused = 1;            // small dense batches: the whole fold as one cooperative launch
  int coop_grid = -1;             // co-resident grid of the fused step (-1 = not probed, 0 = unsupported)
  uint32_t* ss_first[2] = {nullptr, nullptr};  // double-buffered first-occurrence tables, all-ones between calls
  int ss_pp = 0;                  // table the last call used
  uint8_t* ss_deltas = nullptr;   // staging for peer deltas (resolve_peers after a fused scan)
  int ss_dbg = 0;                 // dev probe: phase timestamps of the fused step in d_small[8..16)
  bool sc_small = false;          // last scan was the scan half of the fused step
  std::vector<uint8_t> sc_step;   // its parameters, for the resolve half
};

void hfz_set_error(const char* fmt, ...);
int hfz_cuda_fail(cudaError_t e, const char* what);
int hfz_ensure_host_common(hfz_ctx* c, uint64_t n_exec);   // hfz_api.cu
int hfz_ensure_classed_stage(hfz_ctx* c, uint64_t execs);  // hfz_api.cu
// hfz_feedback.cu: the scan half of the fold on touched-slot lists (device buffers); total_pairs =
// entry_off[n_exec] (absolute).  Pair it with hfz_feedback_resolve, or (delta_out = NULL) hfz_feedback_fold_single.
bool hfz_sparse_native_ok(const hfz_ctx* c);
// pairs / entry_off = wide {slot, count} pairs, compact / compact_off = slot | count << 16 words;
// either list may be absent (null); total_pairs = the sum of both lists' end offsets (absolute).
int hfz_feedback_scan_sparse(hfz_ctx* c, const uint32_t* pairs, const uint64_t* entry_off,
                             const uint32_t* compact, const uint64_t* compact_off, uint64_t n_exec,
                             uint64_t total_pairs, const uint8_t* virgin_v0, uint8_t* classed_out,
                             uint64_t* sig_full_out, uint64_t* sig_simple_out, uint32_t* nnz_out,
                             uint8_t* delta_out, unsigned long long* bad_pairs, int packed = 0);
// packed = 1: `pairs` / `entry_off` are the 3-byte host-half list (entries, every exec a multiple of four) and
// `compact` / `compact_off` the 17-bit-count device-half list of hfz_feedback_batch_packed_host (include/hfz.h)
// single-rank second half after a scan with delta_out = NULL: delta + merge + Admit flags in one pass over the table
int hfz_feedback_fold_single(hfz_ctx* ctx, uint64_t n_exec, uint8_t* virgin_inout, uint64_t* edge_counts_inout,
                             uint8_t* admit_out);

#define HFZ_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return hfz_cuda_fail(_e, #call); \
  } while (0)

// ---------------------------------------------------------------------------
// Arithmetic of the path

// Host ladder (src/coverage.cpp:7-19): {1}->1 {2}->2 {3}->4 {4-7}->8 {8-15}->16
// {16-31}->32 {32-127}->64 {128+}->128.  c in 1..255.
__device__ __forceinline__ uint32_t hfz_class_host(uint32_t c) {
  // rung = 0,1,2 for c = 1,2,3; else 1 + floor(log2 c) for 4..31 (3,4,5); 6 for 32..127; 7 above
  uint32_t lg = 31u - __clz(c);                   // floor(log2 c), c >= 1
  uint32_t r = c <= 3u ? c - 1u : (lg + 1u);      // 4-7 ->3, 8-15 ->4, 16-31 ->5, 32-63 ->6, 64-127 ->7, 128+ ->8
  r = c >= 32u ? (c >= 128u ? 7u : 6u) : r;
  return 1u << r;
}

// Device ladder (src/coverage.cpp:21-32): {1}->1 {2}->2 {3-511}->4 {512-4095}->8
// {4096-16383}->16 {16384-65535}->32 {65536+}->64.  c >= 1, full u32 range.
__device__ __forceinline__ uint32_t hfz_class_device(uint32_t c) {
  uint32_t r = (c >= 2u) + (c >= 3u) + (c >= 512u) + (c >= 4096u) + (c >= 16384u) + (c >= 65536u);
  return 1u << r;
}

// FNV-1a step (include/hetfuzz/coverage.hpp:208-213), P = 2^40 + 0x1b3.
__device__ __forceinline__ uint64_t hfz_fnv(uint64_t h, uint32_t byte) {
  return (h ^ (uint64_t)byte) * 1099511628211ULL;
}
#define HFZ_FNV_OFFSET 14695981039346656037ULL

// splitmix64 (include/hetfuzz/rng.hpp:15-21)
#define HFZ_GAMMA 0x9e3779b97f4a7c15ULL
__host__ __device__ __forceinline__ uint64_t hfz_sm64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier + bulk async copy (TMA, 1-D) + proxy fence

__device__ __forceinline__ uint32_t hfz_smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void hfz_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(hfz_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void hfz_fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void hfz_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void hfz_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(hfz_smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool hfz_mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(hfz_smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void hfz_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(hfz_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void hfz_mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!hfz_mbar_try_wait(bar, parity)) {
  }
}
// global -> shared::cta bulk copy, completion on an mbarrier (SASS: UBLKCP)
__device__ __forceinline__ void hfz_bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          hfz_smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(hfz_smem_u32(bar))
      : "memory");
}
// same with an L2 evict-first policy for streamed-once data
__device__ __forceinline__ void hfz_bulk_g2s_stream(void* smem_dst, const void* gsrc,
                                                    uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(hfz_smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(hfz_smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t hfz_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t hfz_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// streaming 128-bit load (ld.global.cs: evict-first, read once)
__device__ __forceinline__ uint4 hfz_ldg_stream(const uint4* p) { return __ldcs(p); }
