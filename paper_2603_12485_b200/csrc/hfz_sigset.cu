// hfz_sigset.cu -- signature seen-sets and dispatch flags on the device.
//
// Reference semantics: Campaign::run_one keeps two std::set<uint64_t> (src/engine.cpp:319) and,
// per exec IN ORDER, reads "was this signature seen before?" and then inserts it
// (src/engine.cpp:474-478); should_sanitize (src/sanitizers.cpp:283-296) turns the two flags and
// the Admit code into the dispatch decision.
//
// Parallel formulation: an open-addressing hash set of u64 keys in device memory; every slot also
// carries a u64 tag (epoch << 32 | exec index) updated with atomicMin.  A batch inserts all its
// signatures (pass 1), then exec i was "seen before" iff the tag of its slot is not its own
// (pass 2): an older epoch or a smaller exec index got there first -- exactly count()-then-insert()
// in exec order.
#include "hfz_common.cuh"

struct hfz_sigset {
  hfz_ctx* ctx = nullptr;
  uint64_t cap = 0;             // power of two
  unsigned long long* keys = nullptr;  // [cap + 1]  stored as key ^ kScramble, 0 = empty; slot cap = the key that scrambles to 0
  unsigned long long* tags = nullptr;  // [cap + 1]  all-ones = never touched
  uint32_t* slot_tmp = nullptr;        // [tmp_cap] slot of exec i within the current call
  uint64_t tmp_cap = 0;
  uint32_t* d_count = nullptr;         // [2] {distinct keys, overflow flag}
  uint64_t inserted_ub = 0;            // host upper bound of the number of keys
  uint32_t epoch = 0;
};

namespace {
constexpr unsigned long long kScramble = 0x9e3779b97f4a7c15ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  return x;
}

__global__ void hfz_k_sigset_insert(unsigned long long* __restrict__ keys,
                                    unsigned long long* __restrict__ tags, uint64_t cap,
                                    const uint64_t* __restrict__ sigs, uint64_t n, uint32_t epoch,
                                    uint32_t* __restrict__ slot_tmp, uint32_t* __restrict__ count) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = sigs[i] ^ kScramble;
    uint64_t slot;
    if (k == 0) {
      slot = cap;  // dedicated slot for the one key that collides with the empty marker
      if (atomicCAS(&keys[cap], 0ull, 1ull) == 0ull) atomicAdd(count, 1u);
    } else {
      slot = mix64(k) & (cap - 1);
      uint64_t probes = 0;
      for (;;) {
        const unsigned long long cur = keys[slot];
        if (cur == k) break;
        if (cur == 0) {
          const unsigned long long old = atomicCAS(&keys[slot], 0ull, k);
          if (old == 0) {
            atomicAdd(count, 1u);
            break;
          }
          if (old == k) break;
        }
        slot = (slot + 1) & (cap - 1);
        if (++probes > cap) {  // table full: flagged, the host call reports HFZ_ECAP
          atomicExch(count + 1, 1u);
          slot = cap;
          break;
        }
      }
    }
    slot_tmp[i] = (uint32_t)slot;
    atomicMin(&tags[slot], ((unsigned long long)epoch << 32) | (unsigned long long)i);
  }
}

__global__ void hfz_k_sigset_seen(const unsigned long long* __restrict__ tags,
                                  const uint32_t* __restrict__ slot_tmp, uint64_t n, uint32_t epoch,
                                  uint8_t* __restrict__ seen) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    seen[i] = tags[slot_tmp[i]] != (((unsigned long long)epoch << 32) | (unsigned long long)i);
}

// should_sanitize (src/sanitizers.cpp:283-296); strategy: 0 AllTrace, 1 UniqueTrace, 2 SimpleTrace,
// 3 CoverageIncrease (enum class Strategy, include/hetfuzz/sanitizers.hpp:70-75)
__global__ void hfz_k_dispatch(const uint8_t* __restrict__ admit, const uint8_t* __restrict__ full_seen,
                               const uint8_t* __restrict__ simple_seen, uint64_t n, int strategy,
                               uint8_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t r;
    switch (strategy) {
      case 0: r = 1; break;
      case 1: r = !full_seen[i]; break;
      case 2: r = !simple_seen[i]; break;
      default: r = admit[i] != 0; break;
    }
    out[i] = r;
  }
}
}  // namespace

extern "C" int hfz_sigset_create(hfz_ctx* ctx, uint64_t capacity, hfz_sigset** out) {
  if (!ctx || !out || capacity < 1024 || (capacity & (capacity - 1)) || capacity > (1ull << 31)) {
    hfz_set_error("hfz_sigset_create: capacity must be a power of two in [1024, 2^31]");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  hfz_sigset* s = new hfz_sigset;
  s->ctx = ctx;
  s->cap = capacity;
  cudaError_t e = cudaMalloc(&s->keys, (capacity + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&s->tags, (capacity + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_count, 8);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->keys, 0, (capacity + 1) * 8, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->tags, 0xff, (capacity + 1) * 8, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->d_count, 0, 8, ctx->stream);
  if (e != cudaSuccess) {
    cudaFree(s->keys);
    cudaFree(s->tags);
    cudaFree(s->d_count);
    delete s;
    return hfz_cuda_fail(e, "hfz_sigset_create");
  }
  *out = s;
  return HFZ_OK;
}

extern "C" int hfz_sigset_destroy(hfz_sigset* s) {
  if (!s) return HFZ_OK;
  cudaSetDevice(s->ctx->device);
  cudaFree(s->keys);
  cudaFree(s->tags);
  cudaFree(s->slot_tmp);
  cudaFree(s->d_count);
  delete s;
  return HFZ_OK;
}

extern "C" int hfz_sigset_size(hfz_sigset* s, uint64_t* size_out) {
  if (!s || !size_out) return HFZ_EINVAL;
  HFZ_CUDA(cudaSetDevice(s->ctx->device));
  uint32_t h[2] = {0, 0};
  HFZ_CUDA(cudaMemcpyAsync(h, s->d_count, 8, cudaMemcpyDeviceToHost, s->ctx->stream));
  HFZ_CUDA(cudaStreamSynchronize(s->ctx->stream));
  *size_out = h[0];
  s->inserted_ub = h[0];
  if (h[1]) {
    hfz_set_error("hfz_sigset: table overflowed (capacity %llu)", (unsigned long long)s->cap);
    return HFZ_ECAP;
  }
  return HFZ_OK;
}

extern "C" int hfz_sigset_seen_insert(hfz_ctx* ctx, hfz_sigset* s, const uint64_t* sigs, uint64_t n,
                                      uint8_t* seen_out) {
  if (!ctx || !s || s->ctx != ctx || (n && (!sigs || !seen_out)) || n >= 0xffffffffull) {
    hfz_set_error("hfz_sigset_seen_insert: bad argument");
    return HFZ_EINVAL;
  }
  if (n == 0) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  // keep the load factor <= 3/4: refresh the exact size only when the bound says we might exceed it
  if (s->inserted_ub + n > s->cap / 4 * 3) {
    uint64_t sz = 0;
    int rc = hfz_sigset_size(s, &sz);
    if (rc) return rc;
    if (sz + n > s->cap / 4 * 3) {
      hfz_set_error("hfz_sigset_seen_insert: %llu keys + %llu new would exceed 3/4 of capacity %llu",
                    (unsigned long long)sz, (unsigned long long)n, (unsigned long long)s->cap);
      return HFZ_ECAP;
    }
  }
  if (s->tmp_cap < n) {
    cudaFree(s->slot_tmp);
    s->slot_tmp = nullptr;
    s->tmp_cap = 0;
    HFZ_CUDA(cudaMalloc(&s->slot_tmp, n * sizeof(uint32_t)));
    s->tmp_cap = n;
  }
  ++s->epoch;
  const uint32_t blocks = (uint32_t)((n + 255) / 256 < (uint64_t)ctx->num_sms * 8 ? (n + 255) / 256
                                                                                   : (uint64_t)ctx->num_sms * 8);
  hfz_k_sigset_insert<<<blocks, 256, 0, ctx->stream>>>(s->keys, s->tags, s->cap, sigs, n, s->epoch,
                                                       s->slot_tmp, s->d_count);
  hfz_k_sigset_seen<<<blocks, 256, 0, ctx->stream>>>(s->tags, s->slot_tmp, n, s->epoch, seen_out);
  ctx->launches += 2;
  HFZ_CUDA(cudaGetLastError());
  s->inserted_ub += n;
  return HFZ_OK;
}

extern "C" int hfz_dispatch_batch(hfz_ctx* ctx, hfz_sigset* full_set, hfz_sigset* simple_set,
                                  const uint64_t* sig_full, const uint64_t* sig_simple,
                                  const uint8_t* admit, uint64_t n, int strategy,
                                  uint8_t* full_seen_out, uint8_t* simple_seen_out,
                                  uint8_t* sanitize_out) {
  if (!ctx || !full_set || !simple_set || strategy < 0 || strategy > 3 ||
      (n && (!sig_full || !sig_simple || !admit || !full_seen_out || !simple_seen_out || !sanitize_out))) {
    hfz_set_error("hfz_dispatch_batch: bad argument");
    return HFZ_EINVAL;
  }
  int rc = hfz_sigset_seen_insert(ctx, full_set, sig_full, n, full_seen_out);
  if (rc) return rc;
  rc = hfz_sigset_seen_insert(ctx, simple_set, sig_simple, n, simple_seen_out);
  if (rc || n == 0) return rc;
  const uint32_t blocks = (uint32_t)((n + 255) / 256 < (uint64_t)ctx->num_sms * 8 ? (n + 255) / 256
                                                                                   : (uint64_t)ctx->num_sms * 8);
  hfz_k_dispatch<<<blocks, 256, 0, ctx->stream>>>(admit, full_seen_out, simple_seen_out, n, strategy,
                                                  sanitize_out);
  ++ctx->launches;
  HFZ_CUDA(cudaGetLastError());
  return HFZ_OK;
}
