// hfz_sparse.cu -- sparse ingest of raw maps: per-exec touched-slot lists instead of dense records.
//
// A raw map is ~2 % dense, so shipping it dense costs 163,840 B per exec over PCIe (the e2e
// bound of hfz_feedback_batch_host) for ~1,300 non-zero counters.  The reference's own runtime
// already keeps a dirty-slot list beside its device counters (Runtime::bump_counter /
// reset_device_coverage, /root/reference/proj/src/hdvm.cpp:356-366) and classify_trace reduces
// a map to its ascending non-zero list (src/coverage.cpp:58-72).  Here the host hands over, per
// exec, the (slot, count) pairs of the slots it touched, in ANY order; the device scatters
// them into an all-zero dense staging record and runs the same K2 scan / K2b resolve / K4 merge
// on it, so results are bit-identical to the dense call by construction.  After each chunk the
// same pairs are scattered back as zeros (the staging buffer stays all-zero between calls, no
// 1.3 GB memset per chunk).
#include "hfz_common.cuh"

namespace {

// One warp per exec, lanes stride over the exec's pairs (coalesced 8-byte loads, 4 in flight).
// ZERO = true writes zeros instead of the counts (cleanup pass).
template <bool ZERO>
__global__ void __launch_bounds__(256) hfz_k_expand(const uint2* __restrict__ entries,
                                                    const uint64_t* __restrict__ off, uint64_t n_exec,
                                                    uint8_t* __restrict__ dense, uint32_t S, uint32_t H,
                                                    uint64_t rec, unsigned long long* __restrict__ bad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t nbad = 0;
  for (uint64_t e = warp; e < n_exec; e += nwarps) {
    const uint64_t b = off[e], t = off[e + 1];
    uint8_t* r = dense + e * rec;
    for (uint64_t i0 = b; i0 < t; i0 += 128) {
      uint2 x[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t i = i0 + j * 32 + lane;
        x[j] = i < t ? __ldcs(entries + i) : make_uint2(0xffffffffu, 0u);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t slot = x[j].x, c = ZERO ? 0u : x[j].y;
        if (slot < H) {
          r[slot] = (uint8_t)c;  // host half: u8 counters (CoverageMap::host_, coverage.hpp:19)
        } else if (slot < S) {
          *reinterpret_cast<uint32_t*>(r + H + (size_t)(slot - H) * 4) = c;  // device half: u32
        } else if (!ZERO && i0 + j * 32 + lane < t) {
          ++nbad;
        }
      }
    }
  }
  if (!ZERO) {
    nbad = __reduce_add_sync(0xffffffffu, nbad);
    if (lane == 0 && nbad) atomicAdd(bad, (unsigned long long)nbad);
  }
}

constexpr int kBadSlot = 4;  // ctx->d_small[4]: out-of-range pairs seen by the expand kernel

uint64_t chunk_execs(const hfz_ctx* c) {
  if (c->sparse_chunk) return c->sparse_chunk;
  uint64_t n = (1280ull << 20) / c->rec_bytes;  // 8,192 records of 163,840 B
  return n < 32 ? 32 : n / 32 * 32;
}

int ensure_dense(hfz_ctx* c, uint64_t n_exec) {
  uint64_t want = chunk_execs(c);
  if (n_exec < want) want = (n_exec + 31) / 32 * 32;
  if (want < 32) want = 32;
  if (c->sp_dense_execs < want) {
    cudaFree(c->sp_dense);
    c->sp_dense = nullptr;
    c->sp_dense_execs = 0;
    cudaError_t e = cudaMalloc(&c->sp_dense, want * c->rec_bytes);
    if (e != cudaSuccess) {
      hfz_set_error("sparse ingest: cudaMalloc of %llu staging bytes failed (%s)",
                    (unsigned long long)(want * c->rec_bytes), cudaGetErrorString(e));
      return HFZ_ENOMEM;
    }
    c->sp_dense_execs = want;
    c->sp_dirty = true;
  }
  if (c->sp_dirty) {
    HFZ_CUDA(cudaMemsetAsync(c->sp_dense, 0, c->sp_dense_execs * c->rec_bytes, c->stream));
    c->sp_dirty = false;
  }
  return HFZ_OK;
}

template <bool ZERO>
int launch_expand(hfz_ctx* c, const uint32_t* entries, const uint64_t* off, uint64_t n) {
  uint64_t blocks = (n + 7) / 8;  // 8 warps per block, one exec per warp
  const uint64_t cap = (uint64_t)c->num_sms * 8;
  if (blocks > cap) blocks = cap;
  hfz_k_expand<ZERO><<<(uint32_t)blocks, 256, 0, c->stream>>>(
      reinterpret_cast<const uint2*>(entries), off, n, c->sp_dense, c->S, c->H, c->rec_bytes,
      c->d_small + kBadSlot);
  ++c->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

// Folds execs [0, n_exec) given device pairs / offsets, chunk by chunk.  `events` (may be
// null) holds one event per chunk that the stream must wait for before touching the chunk's
// pairs; classed_host (may be null) receives the classed maps through ctx->d_classed.
// native: rank + chain kernels on the lists (total_pairs = entry_off[n_exec], absolute);
// otherwise the pairs are expanded into the dense staging buffer and scanned by K2.
int fold_chunks(hfz_ctx* c, const uint32_t* entries, const uint64_t* off, const uint32_t* compact,
                const uint64_t* coff, uint64_t n_exec, uint64_t C,
                bool native, uint64_t total_pairs, uint8_t* virgin, uint64_t* counts, uint8_t* classed_dev,
                uint8_t* classed_host, uint8_t* admit, uint64_t* sigf, uint64_t* sigs, uint32_t* nnz,
                const cudaEvent_t* events, int packed = 0) {
  if (!native) c->sp_dirty = true;  // until the last cleanup pass has been enqueued
  uint64_t k = 0;
  for (uint64_t done = 0; done < n_exec; done += C, ++k) {
    const uint64_t n = n_exec - done < C ? n_exec - done : C;
    if (events) HFZ_CUDA(cudaStreamWaitEvent(c->stream, events[k], 0));
    uint8_t* cls = classed_dev ? classed_dev + done * (uint64_t)c->S : (classed_host ? c->d_classed : nullptr);
    int rc;
    if (native) {
      rc = hfz_feedback_scan_sparse(c, entries, off ? off + done : nullptr, compact, coff ? coff + done : nullptr, n,
                                    total_pairs, virgin, cls, sigf + done, sigs + done,
                                    nnz ? nnz + done : nullptr, nullptr, c->d_small + kBadSlot, packed);
      if (rc) return rc;
      rc = hfz_feedback_fold_single(c, n, virgin, counts, admit + done);
      if (rc) return rc;
    } else {
      rc = launch_expand<false>(c, entries, off + done, n);
      if (rc) return rc;
      rc = hfz_feedback_batch(c, c->sp_dense, n, virgin, counts, cls, admit + done, sigf + done, sigs + done,
                              nnz ? nnz + done : nullptr);
      if (rc) return rc;
    }
    if (classed_host)
      HFZ_CUDA(cudaMemcpyAsync(classed_host + done * (uint64_t)c->S, c->d_classed, n * (uint64_t)c->S,
                               cudaMemcpyDeviceToHost, c->stream));
    if (!native) {
      rc = launch_expand<true>(c, entries, off + done, n);
      if (rc) return rc;
    }
  }
  if (!native) c->sp_dirty = false;
  return HFZ_OK;
}

}  // namespace

extern "C" int hfz_feedback_batch_sparse(hfz_ctx* c, const uint32_t* entries, const uint64_t* entry_off,
                                         uint64_t n_exec, uint8_t* virgin_inout,
                                         uint64_t* edge_counts_inout, uint8_t* classed_out,
                                         uint8_t* admit_out, uint64_t* sig_full_out,
                                         uint64_t* sig_simple_out, uint32_t* nnz_out) {
  if (!c || !virgin_inout || !edge_counts_inout ||
      (n_exec && (!entry_off || !admit_out || !sig_full_out || !sig_simple_out))) {
    hfz_set_error("hfz_feedback_batch_sparse: null argument");
    return HFZ_EINVAL;
  }
  if ((uintptr_t)entries & 7) {
    hfz_set_error("hfz_feedback_batch_sparse: entries must be 8-byte aligned");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(c->device));
  if (n_exec == 0) return HFZ_OK;
  HFZ_CUDA(cudaMemsetAsync(c->d_small + kBadSlot, 0, sizeof(unsigned long long), c->stream));
  if (hfz_sparse_native_ok(c)) {
    // one pass over the whole batch; the ordered-list scratch is sized from entry_off[n_exec]
    // (one 8-byte read back: this call synchronises the stream once before it enqueues)
    uint64_t total = 0;
    HFZ_CUDA(cudaMemcpyAsync(&total, entry_off + n_exec, 8, cudaMemcpyDeviceToHost, c->stream));
    HFZ_CUDA(cudaStreamSynchronize(c->stream));
    return fold_chunks(c, entries, entry_off, nullptr, nullptr, n_exec, n_exec, true, total, virgin_inout,
                       edge_counts_inout, classed_out, nullptr, admit_out, sig_full_out, sig_simple_out, nnz_out,
                       nullptr);
  }
  int rc = ensure_dense(c, n_exec);
  if (rc) return rc;
  return fold_chunks(c, entries, entry_off, nullptr, nullptr, n_exec, c->sp_dense_execs, false, 0, virgin_inout,
                     edge_counts_inout, classed_out, nullptr, admit_out, sig_full_out, sig_simple_out, nnz_out, nullptr);
}

namespace {

int grow(void** buf, uint64_t* cap, uint64_t want, uint64_t unit) {
  if (*cap >= want) return HFZ_OK;
  cudaFree(*buf);
  *buf = nullptr;
  *cap = 0;
  const uint64_t ncap = want + want / 8 + 1024;
  HFZ_CUDA(cudaMalloc(buf, ncap * unit));
  *cap = ncap;
  return HFZ_OK;
}

int check_offsets(const char* what, const uint64_t* off, uint64_t n_exec) {
  for (uint64_t e = 0; e < n_exec; ++e)
    if (off[e + 1] < off[e]) {
      hfz_set_error("%s: offsets are not non-decreasing at exec %llu", what, (unsigned long long)e);
      return HFZ_EINVAL;
    }
  return HFZ_OK;
}

// Host lists -> device, chunk by chunk on the copy stream, folded as they arrive.  wide pairs
// {slot, count} and/or compact pairs (slot | count << 16); either list may be absent.
int sparse_host_impl(hfz_ctx* c, const uint32_t* entries, const uint64_t* entry_off, const uint32_t* compact,
                     const uint64_t* compact_off, uint64_t n_exec, uint8_t* virgin, uint64_t* counts,
                     uint8_t* classed, uint8_t* admit, uint64_t* sigf, uint64_t* sigs, uint32_t* nnz) {
  const char* who = compact_off ? "hfz_feedback_batch_compact_host" : "hfz_feedback_batch_sparse_host";
  if (!c || !virgin || !counts || (n_exec && ((!entry_off && !compact_off) || !admit || !sigf || !sigs))) {
    hfz_set_error("%s: null argument", who);
    return HFZ_EINVAL;
  }
  if (n_exec == 0) return HFZ_OK;
  // offsets index their list absolutely, so a sub-range of a larger batch is folded by passing
  // off + first_exec; only pairs [off[0], off[n_exec]) are copied
  const uint64_t total = entry_off ? entry_off[n_exec] : 0;
  const uint64_t ctotal = compact_off ? compact_off[n_exec] : 0;
  if ((entry_off && total > entry_off[0] && !entries) || (compact_off && ctotal > compact_off[0] && !compact)) {
    hfz_set_error("%s: a list has pairs but its pointer is null", who);
    return HFZ_EINVAL;
  }
  int rc;
  if (entry_off && (rc = check_offsets(who, entry_off, n_exec))) return rc;
  if (compact_off && (rc = check_offsets(who, compact_off, n_exec))) return rc;
  HFZ_CUDA(cudaSetDevice(c->device));
  rc = hfz_ensure_host_common(c, n_exec);
  if (rc) return rc;
  const bool native = hfz_sparse_native_ok(c);
  if (compact_off && (!native || c->S > 65536u)) {
    hfz_set_error("%s: compact lists need the list-native fold and a 16-bit slot (map_slots <= 65536, sparse_native = 1)", who);
    return HFZ_EINVAL;
  }
  uint64_t C;
  if (native) {
    // chunks only pace the overlap of the H2D stream with the kernels (measured: 4,096 execs)
    C = c->sparse_chunk ? c->sparse_chunk : 4096;
  } else {
    rc = ensure_dense(c, n_exec);
    if (rc) return rc;
    C = c->sp_dense_execs;
  }
  const uint64_t n_chunks = (n_exec + C - 1) / C;
  if (classed && (rc = hfz_ensure_classed_stage(c, n_exec < C ? n_exec : C))) return rc;
  // the device copies keep the absolute indexing: pairs below off[0] are never read
  if (entry_off) {
    if ((rc = grow(reinterpret_cast<void**>(&c->sp_entries), &c->sp_entries_cap, total, 8))) return rc;
    if ((rc = grow(reinterpret_cast<void**>(&c->sp_off), &c->sp_off_cap, n_exec + 1, 8))) return rc;
  }
  if (compact_off) {
    if ((rc = grow(reinterpret_cast<void**>(&c->sp_compact), &c->sp_compact_cap, ctotal, 4))) return rc;
    if ((rc = grow(reinterpret_cast<void**>(&c->sp_coff), &c->sp_coff_cap, n_exec + 1, 8))) return rc;
  }
  while (c->sp_events.size() < n_chunks) {
    cudaEvent_t ev;
    HFZ_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    c->sp_events.push_back(ev);
  }
  cudaStream_t st = c->stream;
  // small inputs first: the H2D copy engine serves copies in issue order, so queueing them
  // behind the pairs would hold the first chunk's kernels back until every pair has arrived
  if (entry_off) HFZ_CUDA(cudaMemcpyAsync(c->sp_off, entry_off, (n_exec + 1) * 8, cudaMemcpyHostToDevice, st));
  if (compact_off) HFZ_CUDA(cudaMemcpyAsync(c->sp_coff, compact_off, (n_exec + 1) * 8, cudaMemcpyHostToDevice, st));
  HFZ_CUDA(cudaMemcpyAsync(c->d_virgin, virgin, c->S, cudaMemcpyHostToDevice, st));
  HFZ_CUDA(cudaMemcpyAsync(c->d_counts, counts, 16, cudaMemcpyHostToDevice, st));
  HFZ_CUDA(cudaMemsetAsync(c->d_small + kBadSlot, 0, sizeof(unsigned long long), st));
  // the pairs stream in on the copy stream, one event per chunk; everything else on `st`
  for (uint64_t k = 0; k < n_chunks; ++k) {
    const uint64_t e0 = k * C, e1 = e0 + C < n_exec ? e0 + C : n_exec;
    if (entry_off && entry_off[e1] > entry_off[e0])
      HFZ_CUDA(cudaMemcpyAsync(c->sp_entries + 2 * entry_off[e0], entries + 2 * entry_off[e0],
                               (entry_off[e1] - entry_off[e0]) * 8, cudaMemcpyHostToDevice, c->copy_stream));
    if (compact_off && compact_off[e1] > compact_off[e0])
      HFZ_CUDA(cudaMemcpyAsync(c->sp_compact + compact_off[e0], compact + compact_off[e0],
                               (compact_off[e1] - compact_off[e0]) * 4, cudaMemcpyHostToDevice, c->copy_stream));
    HFZ_CUDA(cudaEventRecord(c->sp_events[k], c->copy_stream));
  }
  rc = fold_chunks(c, c->sp_entries, entry_off ? c->sp_off : nullptr, c->sp_compact, compact_off ? c->sp_coff : nullptr,
                   n_exec, C, native, total + ctotal, c->d_virgin, c->d_counts, nullptr, classed, c->d_admit,
                   c->d_sigf, c->d_sigs, c->d_nnz, c->sp_events.data());
  if (rc) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamSynchronize(st);
    return rc;
  }
  unsigned long long bad = 0;
  HFZ_CUDA(cudaMemcpyAsync(admit, c->d_admit, n_exec, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(sigf, c->d_sigf, n_exec * 8, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(sigs, c->d_sigs, n_exec * 8, cudaMemcpyDeviceToHost, st));
  if (nnz) HFZ_CUDA(cudaMemcpyAsync(nnz, c->d_nnz, n_exec * 4, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(virgin, c->d_virgin, c->S, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(counts, c->d_counts, 16, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(&bad, c->d_small + kBadSlot, sizeof(bad), cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaStreamSynchronize(st));
  if (bad) {
    hfz_set_error("%s: %llu pairs name a slot >= %u (ignored)", who, bad, c->S);
    return HFZ_EINVAL;
  }
  return HFZ_OK;
}

// Packed lists (include/hfz.h, hfz_feedback_batch_packed_host[_v]): host half 3 bytes per entry, device half 4 bytes
// with a 17-bit count -- ~4.1 KB per exec of the bench batch against ~5.0 KB of the compact form.  Same streaming as
// above, over one batch or over several (one per packing thread of the host, folded in the order given): every list
// of every batch is queued on the copy stream up front, the folds follow chunk by chunk, ONE synchronisation at the end.
int packed_host_impl(hfz_ctx* c, uint32_t n_batches, const uint8_t* const* host3, const uint64_t* const* host3_off,
                     const uint32_t* const* dev17, const uint64_t* const* dev17_off, const uint64_t* n_exec,
                     uint8_t* virgin, uint64_t* counts, uint8_t* classed, uint8_t* admit, uint64_t* sigf, uint64_t* sigs,
                     uint32_t* nnz) {
  const char* who = n_batches == 1 ? "hfz_feedback_batch_packed_host" : "hfz_feedback_batch_packed_host_v";
  if (!c || !virgin || !counts || !host3 || !host3_off || !dev17 || !dev17_off || !n_exec) {
    hfz_set_error("%s: null argument", who);
    return HFZ_EINVAL;
  }
  uint64_t n_total = 0, h_words = 0, d_words = 0, n_chunks = 0, max_pairs = 0;
  const uint64_t C = c->sparse_chunk ? c->sparse_chunk : 4096;
  int rc;
  for (uint32_t k = 0; k < n_batches; ++k) {
    const uint64_t n = n_exec[k];
    if (n == 0) continue;
    if (!host3_off[k] || !dev17_off[k]) {
      hfz_set_error("%s: batch %u has execs but no offsets", who, k);
      return HFZ_EINVAL;
    }
    const uint64_t htotal = host3_off[k][n], dtotal = dev17_off[k][n];
    if ((htotal > host3_off[k][0] && !host3[k]) || (dtotal > dev17_off[k][0] && !dev17[k]) || ((uintptr_t)host3[k] & 3)) {
      hfz_set_error("%s: a list has entries but its pointer is null, or host3 is not 4-byte aligned", who);
      return HFZ_EINVAL;
    }
    if (htotal < host3_off[k][0] || dtotal < dev17_off[k][0] || (htotal & 3)) {
      hfz_set_error("%s: batch %u: offsets decrease, or the host list is not a multiple of four entries", who, k);
      return HFZ_EINVAL;
    }
    n_total += n;
    h_words += htotal / 4 * 3;
    d_words += dtotal;
    n_chunks += (n + C - 1) / C;
    if (htotal + dtotal > max_pairs) max_pairs = htotal + dtotal;
  }
  if (n_total == 0) return HFZ_OK;
  if (!admit || !sigf || !sigs) {
    hfz_set_error("%s: null argument", who);
    return HFZ_EINVAL;
  }
  if (classed && n_batches != 1) {
    hfz_set_error("%s: classed maps are returned by the single-batch call only", who);
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(c->device));
  if ((rc = hfz_ensure_host_common(c, n_total))) return rc;
  if (!hfz_sparse_native_ok(c) || c->S != 65536u) {
    hfz_set_error("%s: packed lists need the list-native fold and map_slots = 65536 (15-bit slots per half)", who);
    return HFZ_EINVAL;
  }
  if (classed && (rc = hfz_ensure_classed_stage(c, n_total < C ? n_total : C))) return rc;
  // device copies, batch after batch; inside a batch the absolute indexing is kept (entries below off[0] are never read)
  if ((rc = grow(reinterpret_cast<void**>(&c->sp_h3), &c->sp_h3_cap, h_words + 4, 4))) return rc;
  if ((rc = grow(reinterpret_cast<void**>(&c->sp_off), &c->sp_off_cap, n_total + n_batches, 8))) return rc;
  if ((rc = grow(reinterpret_cast<void**>(&c->sp_compact), &c->sp_compact_cap, d_words + 1, 4))) return rc;
  if ((rc = grow(reinterpret_cast<void**>(&c->sp_coff), &c->sp_coff_cap, n_total + n_batches, 8))) return rc;
  while (c->sp_events.size() < n_chunks) {
    cudaEvent_t ev;
    HFZ_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    c->sp_events.push_back(ev);
  }
  cudaStream_t st = c->stream;
  // small inputs first (the copy engine serves copies in issue order)
  {
    uint64_t ob = 0;
    for (uint32_t k = 0; k < n_batches; ++k) {
      if (!n_exec[k]) continue;
      HFZ_CUDA(cudaMemcpyAsync(c->sp_off + ob, host3_off[k], (n_exec[k] + 1) * 8, cudaMemcpyHostToDevice, st));
      HFZ_CUDA(cudaMemcpyAsync(c->sp_coff + ob, dev17_off[k], (n_exec[k] + 1) * 8, cudaMemcpyHostToDevice, st));
      ob += n_exec[k] + 1;
    }
  }
  HFZ_CUDA(cudaMemcpyAsync(c->d_virgin, virgin, c->S, cudaMemcpyHostToDevice, st));
  HFZ_CUDA(cudaMemcpyAsync(c->d_counts, counts, 16, cudaMemcpyHostToDevice, st));
  HFZ_CUDA(cudaMemsetAsync(c->d_small + kBadSlot, 0, sizeof(unsigned long long), st));
  {
    uint64_t hb = 0, db = 0, ev = 0;  // word offsets of batch k's lists in the device buffers
    for (uint32_t k = 0; k < n_batches; ++k) {
      const uint64_t n = n_exec[k];
      if (!n) continue;
      uint8_t* d_h3 = reinterpret_cast<uint8_t*>(c->sp_h3 + hb);
      for (uint64_t e0 = 0; e0 < n; e0 += C, ++ev) {
        const uint64_t e1 = e0 + C < n ? e0 + C : n;
        const uint64_t* ho = host3_off[k];
        const uint64_t* dof = dev17_off[k];
        // (every offset is validated below, while these copies are in flight; here only what keeps the copies
        // themselves inside the buffers)
        if (ho[e0] > ho[e1] || ho[e1] > ho[n] || dof[e0] > dof[e1] || dof[e1] > dof[n] || ((ho[e0] | ho[e1]) & 3)) {
          cudaStreamSynchronize(c->copy_stream);
          cudaStreamSynchronize(st);
          hfz_set_error("%s: batch %u: offsets are not non-decreasing multiples of four (host) / non-decreasing (device)", who, k);
          return HFZ_EINVAL;
        }
        if (ho[e1] > ho[e0])
          HFZ_CUDA(cudaMemcpyAsync(d_h3 + 3 * ho[e0], host3[k] + 3 * ho[e0], (ho[e1] - ho[e0]) * 3, cudaMemcpyHostToDevice,
                                   c->copy_stream));
        if (dof[e1] > dof[e0])
          HFZ_CUDA(cudaMemcpyAsync(c->sp_compact + db + dof[e0], dev17[k] + dof[e0], (dof[e1] - dof[e0]) * 4,
                                   cudaMemcpyHostToDevice, c->copy_stream));
        HFZ_CUDA(cudaEventRecord(c->sp_events[ev], c->copy_stream));
      }
      hb += host3_off[k][n] / 4 * 3;
      db += dev17_off[k][n];
    }
  }
  // the offsets of every exec, checked while the lists cross PCIe (0.15 ms of host work per 65,536 execs that
  // used to sit in front of the first copy)
  for (uint32_t k = 0; k < n_batches; ++k) {
    const uint64_t n = n_exec[k];
    if (!n) continue;
    rc = check_offsets(who, host3_off[k], n);
    if (!rc) rc = check_offsets(who, dev17_off[k], n);
    for (uint64_t e = 0; !rc && e <= n; ++e)
      if (host3_off[k][e] & 3) {
        hfz_set_error("%s: host3_off[%llu] is not a multiple of four entries (pad every exec with zero entries)", who,
                      (unsigned long long)e);
        rc = HFZ_EINVAL;
      }
    if (rc) {
      cudaStreamSynchronize(c->copy_stream);
      cudaStreamSynchronize(st);
      return rc;
    }
  }
  {
    uint64_t hb = 0, db = 0, ob = 0, eb = 0, ev = 0;
    for (uint32_t k = 0; k < n_batches; ++k) {
      const uint64_t n = n_exec[k];
      if (!n) continue;
      rc = fold_chunks(c, c->sp_h3 + hb, c->sp_off + ob, c->sp_compact + db, c->sp_coff + ob, n, C, true, max_pairs,
                       c->d_virgin, c->d_counts, nullptr, classed, c->d_admit + eb, c->d_sigf + eb, c->d_sigs + eb,
                       c->d_nnz + eb, c->sp_events.data() + ev, 1);
      if (rc) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamSynchronize(st);
        return rc;
      }
      hb += host3_off[k][n] / 4 * 3;
      db += dev17_off[k][n];
      ob += n + 1;
      eb += n;
      ev += (n + C - 1) / C;
    }
  }
  HFZ_CUDA(cudaMemcpyAsync(admit, c->d_admit, n_total, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(sigf, c->d_sigf, n_total * 8, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(sigs, c->d_sigs, n_total * 8, cudaMemcpyDeviceToHost, st));
  if (nnz) HFZ_CUDA(cudaMemcpyAsync(nnz, c->d_nnz, n_total * 4, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(virgin, c->d_virgin, c->S, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(counts, c->d_counts, 16, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaStreamSynchronize(st));
  return HFZ_OK;
}

}  // namespace

extern "C" int hfz_feedback_batch_sparse_host(hfz_ctx* c, const uint32_t* entries, const uint64_t* entry_off,
                                              uint64_t n_exec, uint8_t* virgin, uint64_t* counts,
                                              uint8_t* classed, uint8_t* admit, uint64_t* sigf,
                                              uint64_t* sigs, uint32_t* nnz) {
  if (n_exec && !entry_off) {
    hfz_set_error("hfz_feedback_batch_sparse_host: null argument");
    return HFZ_EINVAL;
  }
  return sparse_host_impl(c, entries, entry_off, nullptr, nullptr, n_exec, virgin, counts, classed, admit, sigf, sigs,
                          nnz);
}

extern "C" int hfz_feedback_batch_compact_host(hfz_ctx* c, const uint32_t* compact, const uint64_t* compact_off,
                                               const uint32_t* wide, const uint64_t* wide_off, uint64_t n_exec,
                                               uint8_t* virgin, uint64_t* counts, uint8_t* classed, uint8_t* admit,
                                               uint64_t* sigf, uint64_t* sigs, uint32_t* nnz) {
  if (n_exec && !compact_off) {
    hfz_set_error("hfz_feedback_batch_compact_host: null argument");
    return HFZ_EINVAL;
  }
  return sparse_host_impl(c, wide, wide_off, compact, compact_off, n_exec, virgin, counts, classed, admit, sigf, sigs,
                          nnz);
}

extern "C" int hfz_feedback_batch_packed_host(hfz_ctx* c, const uint8_t* host3, const uint64_t* host3_off,
                                              const uint32_t* dev17, const uint64_t* dev17_off, uint64_t n_exec,
                                              uint8_t* virgin, uint64_t* counts, uint8_t* classed, uint8_t* admit,
                                              uint64_t* sigf, uint64_t* sigs, uint32_t* nnz) {
  if (n_exec && (!host3_off || !dev17_off)) {
    hfz_set_error("hfz_feedback_batch_packed_host: null argument");
    return HFZ_EINVAL;
  }
  return packed_host_impl(c, 1, &host3, &host3_off, &dev17, &dev17_off, &n_exec, virgin, counts, classed, admit, sigf, sigs,
                          nnz);
}

extern "C" int hfz_feedback_batch_packed_host_v(hfz_ctx* c, uint32_t n_batches, const uint8_t* const* host3,
                                                const uint64_t* const* host3_off, const uint32_t* const* dev17,
                                                const uint64_t* const* dev17_off, const uint64_t* n_exec, uint8_t* virgin,
                                                uint64_t* counts, uint8_t* admit, uint64_t* sigf, uint64_t* sigs,
                                                uint32_t* nnz) {
  return packed_host_impl(c, n_batches, host3, host3_off, dev17, dev17_off, n_exec, virgin, counts, nullptr, admit, sigf,
                          sigs, nnz);
}

extern "C" int hfz_expand_sparse(hfz_ctx* c, const uint32_t* entries, const uint64_t* entry_off,
                                 uint64_t n_exec, uint8_t* raw_maps_out) {
  if (!c || (n_exec && (!entry_off || !raw_maps_out))) {
    hfz_set_error("hfz_expand_sparse: null argument");
    return HFZ_EINVAL;
  }
  if (((uintptr_t)entries & 7) || ((uintptr_t)raw_maps_out & 15)) {
    hfz_set_error("hfz_expand_sparse: entries must be 8-byte, raw_maps_out 16-byte aligned");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(c->device));
  if (n_exec == 0) return HFZ_OK;
  HFZ_CUDA(cudaMemsetAsync(raw_maps_out, 0, n_exec * c->rec_bytes, c->stream));
  uint64_t blocks = (n_exec + 7) / 8;
  const uint64_t cap = (uint64_t)c->num_sms * 8;
  if (blocks > cap) blocks = cap;
  hfz_k_expand<false><<<(uint32_t)blocks, 256, 0, c->stream>>>(
      reinterpret_cast<const uint2*>(entries), entry_off, n_exec, raw_maps_out, c->S, c->H, c->rec_bytes,
      c->d_small + kBadSlot);
  ++c->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}

// Pinned host memory for C/C++ hosts that do not link the CUDA runtime themselves.
extern "C" int hfz_host_alloc(void** out, uint64_t bytes) {
  if (!out) return HFZ_EINVAL;
  *out = nullptr;
  cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault);
  if (e != cudaSuccess) {
    hfz_set_error("hfz_host_alloc(%llu): %s", (unsigned long long)bytes, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? HFZ_ENOMEM : HFZ_ECUDA;
  }
  return HFZ_OK;
}

extern "C" int hfz_host_free(void* p) {
  if (!p) return HFZ_OK;
  HFZ_CUDA(cudaFreeHost(p));
  return HFZ_OK;
}
