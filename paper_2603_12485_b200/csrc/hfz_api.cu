// hfz_api.cu -- context management, error reporting, host-buffer front-end, Rng helpers.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "hfz_common.cuh"

static thread_local char g_err[512] = "";

void hfz_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int hfz_cuda_fail(cudaError_t e, const char* what) {
  hfz_set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
  return HFZ_ECUDA;
}

extern "C" int hfz_version(void) { return HFZ_VERSION; }
extern "C" const char* hfz_last_error(void) { return g_err; }
extern "C" uint64_t hfz_record_bytes(uint32_t map_slots) { return (uint64_t)(map_slots / 2) * 5; }

extern "C" int hfz_ctx_create(hfz_ctx** out, int device, uint32_t map_slots, void* stream) {
  if (!out) {
    hfz_set_error("hfz_ctx_create: null out");
    return HFZ_EINVAL;
  }
  *out = nullptr;
  if (map_slots < 1024u || map_slots > (1u << 24) || (map_slots & (map_slots - 1u))) {
    hfz_set_error("hfz_ctx_create: map_slots must be a power of two in [1024, 2^24], got %u",
                  map_slots);
    return HFZ_EINVAL;
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    hfz_set_error("no CUDA device available (%s); this library has no CPU fallback",
                  e != cudaSuccess ? cudaGetErrorString(e) : "device count 0");
    return HFZ_ECUDA;
  }
  if (device < 0 || device >= ndev) {
    hfz_set_error("hfz_ctx_create: device %d out of range (%d devices)", device, ndev);
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  HFZ_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0) {
    hfz_set_error("device %d is sm_%d%d; the kernels are built for sm_100a only", device,
                  prop.major, prop.minor);
    return HFZ_ECUDA;
  }
  hfz_ctx* c = new hfz_ctx;
  c->device = device;
  c->S = map_slots;
  c->H = map_slots / 2;
  c->rec_bytes = (uint64_t)c->H * 5;
  c->stream = (cudaStream_t)stream;
  c->num_sms = prop.multiProcessorCount;
  c->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
  cudaError_t a = cudaMalloc(&c->first, (size_t)map_slots * 8 * sizeof(uint32_t));
  if (a == cudaSuccess) a = cudaMalloc(&c->prior, map_slots);
  if (a == cudaSuccess) a = cudaMalloc(&c->delta, map_slots);
  if (a == cudaSuccess) a = cudaMalloc(&c->v0, map_slots);
  if (a == cudaSuccess) a = cudaMalloc(&c->d_small, 32 * sizeof(unsigned long long));
  if (a != cudaSuccess) {
    hfz_ctx_destroy(c);
    hfz_set_error("hfz_ctx_create: scratch allocation failed (%s)", cudaGetErrorString(a));
    return HFZ_ENOMEM;
  }
  *out = c;
  return HFZ_OK;
}

extern "C" int hfz_ctx_destroy(hfz_ctx* c) {
  if (!c) return HFZ_OK;
  cudaSetDevice(c->device);
  cudaFree(c->first);
  cudaFree(c->admit_flags);
  cudaFree(c->prior);
  cudaFree(c->delta);
  cudaFree(c->v0);
  cudaFree(c->d_small);
  cudaFree(c->edge_prev);
  cudaFree(c->fl_nsw);
  cudaFree(c->fl_sw_off);
  cudaFree(c->fl_l_exec);
  cudaFree(c->fl_elig);
  cudaFree(c->fl_exec_ev0);
  cudaFree(c->fl_exec_sw0);
  cudaFree(c->fl_inelig);
  cudaFree(c->fl_scratch);
  cudaFree(c->fl_rec_first);
  cudaFree(c->fl_rec_cnt);
  cudaFree(c->fl_div);
  cudaFree(c->fl_lines);
  cudaFree(c->hv_ops);
  for (int i = 0; i < 2; ++i) {
    cudaFree(c->stage_raw[i]);
    if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
    if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
  }
  for (auto& ev : c->scan_events) {
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->ev_stream) cudaEventDestroy(c->ev_stream);
  cudaFree(c->d_virgin);
  cudaFree(c->d_counts);
  cudaFree(c->d_admit);
  cudaFree(c->d_sigf);
  cudaFree(c->d_sigs);
  cudaFree(c->d_nnz);
  cudaFree(c->d_classed);
  cudaFree(c->sp_dense);
  cudaFree(c->sp_entries);
  cudaFree(c->sp_off);
  cudaFree(c->sp_compact);
  cudaFree(c->sp_coff);
  cudaFree(c->sp_h3);
  cudaFree(c->sp_sorted);
  cudaFree(c->ts_sorted);
  cudaFree(c->ts_cnt);
  cudaFree(c->sp_cnt);
  cudaFree(c->ss_first[0]);
  cudaFree(c->ss_first[1]);
  cudaFree(c->ss_deltas);
  for (cudaEvent_t ev : c->sp_events) cudaEventDestroy(ev);
  delete c;
  return HFZ_OK;
}

extern "C" int hfz_ctx_set_stream(hfz_ctx* c, void* stream) {
  if (!c) return HFZ_EINVAL;
  if (c->stream == (cudaStream_t)stream) return HFZ_OK;
  // The context's scratch (first-occurrence tables, Admit flags, prior, piece lists) is shared by
  // all calls: work already enqueued on the old stream must finish before the new stream touches it.
  HFZ_CUDA(cudaSetDevice(c->device));
  if (!c->ev_stream) HFZ_CUDA(cudaEventCreateWithFlags(&c->ev_stream, cudaEventDisableTiming));
  HFZ_CUDA(cudaEventRecord(c->ev_stream, c->stream));
  HFZ_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_stream, 0));
  c->stream = (cudaStream_t)stream;
  return HFZ_OK;
}

extern "C" int hfz_ctx_sync(hfz_ctx* c) {
  if (!c) return HFZ_EINVAL;
  HFZ_CUDA(cudaSetDevice(c->device));
  HFZ_CUDA(cudaStreamSynchronize(c->stream));
  return HFZ_OK;
}

extern "C" uint32_t hfz_ctx_map_slots(const hfz_ctx* c) { return c ? c->S : 0; }
extern "C" uint64_t hfz_ctx_launch_count(const hfz_ctx* c) { return c ? c->launches : 0; }

extern "C" int hfz_ctx_set_option(hfz_ctx* c, const char* key, int64_t value) {
  if (!c || !key) return HFZ_EINVAL;
  if (!strcmp(key, "scan_warps")) {
    if (value < 0 || value > 32) return HFZ_EINVAL;
    c->scan_warps = (int)value;
  } else if (!strcmp(key, "scan_row")) {
    if (value != 0 && value != 256 && value != 512 && value != 1024) return HFZ_EINVAL;
    c->scan_row = (int)value;
  } else if (!strcmp(key, "scan_prefetch")) {
    c->scan_prefetch = value != 0;
  } else if (!strcmp(key, "virgin_smem")) {
    c->virgin_smem = value != 0;
  } else if (!strcmp(key, "scan_small")) {
    c->scan_small = value;
  } else if (!strcmp(key, "scan_pipe")) {
    c->scan_pipe = value;
  } else if (!strcmp(key, "scan_two_stage")) {
    c->scan_two_stage = value;
  } else if (!strcmp(key, "small_fused")) {
    c->small_fused = value != 0;
  } else if (!strcmp(key, "step_probe")) {
    c->ss_dbg = value != 0;
  } else if (!strcmp(key, "edge_flat")) {
    c->edge_flat = value != 0;
  } else if (!strcmp(key, "edge_scratch_mb")) {
    if (value < 1 || value > (1 << 20)) return HFZ_EINVAL;
    c->edge_scratch_mb = value;
  } else if (!strcmp(key, "time_scan")) {
    c->time_scan = value != 0;
  } else if (!strcmp(key, "sparse_native")) {
    c->sparse_native = value != 0;
  } else if (!strcmp(key, "sparse_chunk")) {
    if (value < 0 || (value && value < 32) || c->sp_dense) return HFZ_EINVAL;
    c->sparse_chunk = (uint64_t)value / 32 * 32;
  } else if (!strcmp(key, "stage_execs")) {
    if (value < 32 || c->stage_raw[0]) return HFZ_EINVAL;
    c->stage_execs = (uint64_t)value;
  } else {
    hfz_set_error("hfz_ctx_set_option: unknown key %s", key);
    return HFZ_EINVAL;
  }
  return HFZ_OK;
}

extern "C" int hfz_ctx_get_stat(hfz_ctx* c, const char* key, double* out) {
  if (!c || !key || !out) return HFZ_EINVAL;
  HFZ_CUDA(cudaSetDevice(c->device));
  if (!strcmp(key, "scan_launches")) {
    *out = (double)c->scan_events.size();
    return HFZ_OK;
  }
  if (!strcmp(key, "scan_ms_total")) {
    HFZ_CUDA(cudaStreamSynchronize(c->stream));
    double total = 0;
    for (auto& ev : c->scan_events) {
      float ms = 0;
      HFZ_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
      total += ms;
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
    c->scan_events.clear();
    *out = total;
    return HFZ_OK;
  }
  if (!strcmp(key, "ignored_pairs")) {  // pairs with slot >= S seen by the last sparse fold (device or host call)
    unsigned long long bad = 0;
    HFZ_CUDA(cudaStreamSynchronize(c->stream));
    HFZ_CUDA(cudaMemcpy(&bad, c->d_small + 4, sizeof(bad), cudaMemcpyDeviceToHost));
    *out = (double)bad;
    return HFZ_OK;
  }
  if (!strncmp(key, "step_c", 6) && key[6] >= '0' && key[6] <= '7' && !key[7]) {  // dev probe: raw counters
    unsigned long long t[8];
    HFZ_CUDA(cudaStreamSynchronize(c->stream));
    HFZ_CUDA(cudaMemcpy(t, c->d_small + 16, sizeof(t), cudaMemcpyDeviceToHost));
    *out = (double)t[key[6] - '0'];
    return HFZ_OK;
  }
  if (!strncmp(key, "step_t", 6) && key[6] >= '1' && key[6] <= '6' && !key[7]) {
    // dev probe: microseconds from the fused step's first CTA start to the LAST CTA passing boundary k
    unsigned long long t[8];
    HFZ_CUDA(cudaStreamSynchronize(c->stream));
    HFZ_CUDA(cudaMemcpy(t, c->d_small + 8, sizeof(t), cudaMemcpyDeviceToHost));
    *out = t[key[6] - '0'] >= t[0] ? (double)(t[key[6] - '0'] - t[0]) / 1e3 : -1.0;
    return HFZ_OK;
  }
  hfz_set_error("hfz_ctx_get_stat: unknown key %s", key);
  return HFZ_EINVAL;
}

// ---------------------------------------------------------------------------
// Host-buffer front-end: chunked, double-buffered H2D overlapped with the kernels.

// copy stream, device copies of virgin / counters and per-exec outputs shared by the _host calls
int hfz_ensure_host_common(hfz_ctx* c, uint64_t n_exec) {
  // each resource on its own: a failed allocation is retried by the next call instead of leaving a
  // null pointer behind an "already initialised" flag
  if (!c->copy_stream) HFZ_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (!c->d_virgin) HFZ_CUDA(cudaMalloc(&c->d_virgin, c->S));
  if (!c->d_counts) HFZ_CUDA(cudaMalloc(&c->d_counts, 2 * sizeof(uint64_t)));
  if (c->d_out_cap < n_exec) {
    cudaFree(c->d_admit);
    cudaFree(c->d_sigf);
    cudaFree(c->d_sigs);
    cudaFree(c->d_nnz);
    c->d_admit = nullptr;
    c->d_sigf = c->d_sigs = nullptr;
    c->d_nnz = nullptr;
    c->d_out_cap = 0;
    const uint64_t cap = n_exec < 1024 ? 1024 : n_exec;
    HFZ_CUDA(cudaMalloc(&c->d_admit, cap));
    HFZ_CUDA(cudaMalloc(&c->d_sigf, cap * 8));
    HFZ_CUDA(cudaMalloc(&c->d_sigs, cap * 8));
    HFZ_CUDA(cudaMalloc(&c->d_nnz, cap * 4));
    c->d_out_cap = cap;
  }
  return HFZ_OK;
}

int hfz_ensure_classed_stage(hfz_ctx* c, uint64_t execs) {
  if (c->d_classed_cap >= execs) return HFZ_OK;
  cudaFree(c->d_classed);
  c->d_classed = nullptr;
  c->d_classed_cap = 0;
  HFZ_CUDA(cudaMalloc(&c->d_classed, execs * (uint64_t)c->S));
  c->d_classed_cap = execs;
  return HFZ_OK;
}

static int ensure_host_path(hfz_ctx* c, uint64_t n_exec, bool want_classed) {
  int rc = hfz_ensure_host_common(c, n_exec);
  if (rc) return rc;
  if (!c->stage_raw[0]) {
    if (c->stage_execs == 0) {
      // ~256 MB per staging buffer
      uint64_t se = (256ull << 20) / c->rec_bytes;
      se = se < 32 ? 32 : (se / 32) * 32;
      c->stage_execs = se;
    }
    for (int i = 0; i < 2; ++i) {
      HFZ_CUDA(cudaMalloc(&c->stage_raw[i], c->stage_execs * c->rec_bytes));
      HFZ_CUDA(cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming));
      HFZ_CUDA(cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming));
    }
  }
  if (want_classed) return hfz_ensure_classed_stage(c, c->stage_execs);
  return HFZ_OK;
}

extern "C" int hfz_feedback_batch_host(hfz_ctx* c, const uint8_t* raw, uint64_t n_exec,
                                       uint8_t* virgin, uint64_t* counts, uint8_t* classed,
                                       uint8_t* admit, uint64_t* sigf, uint64_t* sigs,
                                       uint32_t* nnz) {
  if (!c || !virgin || !counts || (n_exec && (!raw || !admit || !sigf || !sigs))) {
    hfz_set_error("hfz_feedback_batch_host: null argument");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(c->device));
  int rc = ensure_host_path(c, n_exec, classed != nullptr);
  if (rc) return rc;
  cudaStream_t st = c->stream;
  HFZ_CUDA(cudaMemcpyAsync(c->d_virgin, virgin, c->S, cudaMemcpyHostToDevice, st));
  HFZ_CUDA(cudaMemcpyAsync(c->d_counts, counts, 16, cudaMemcpyHostToDevice, st));
  uint64_t done = 0;
  int buf = 0;
  bool used[2] = {false, false};
  while (done < n_exec) {
    const uint64_t n = n_exec - done < c->stage_execs ? n_exec - done : c->stage_execs;
    if (used[buf]) HFZ_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev_done[buf], 0));
    HFZ_CUDA(cudaMemcpyAsync(c->stage_raw[buf], raw + done * c->rec_bytes, n * c->rec_bytes,
                             cudaMemcpyHostToDevice, c->copy_stream));
    HFZ_CUDA(cudaEventRecord(c->ev_copied[buf], c->copy_stream));
    HFZ_CUDA(cudaStreamWaitEvent(st, c->ev_copied[buf], 0));
    rc = hfz_feedback_batch(c, c->stage_raw[buf], n, c->d_virgin, c->d_counts,
                            classed ? c->d_classed : nullptr, c->d_admit + done, c->d_sigf + done,
                            c->d_sigs + done, c->d_nnz + done);
    if (rc) return rc;
    if (classed)
      HFZ_CUDA(cudaMemcpyAsync(classed + done * (uint64_t)c->S, c->d_classed, n * (uint64_t)c->S,
                               cudaMemcpyDeviceToHost, st));
    HFZ_CUDA(cudaEventRecord(c->ev_done[buf], st));
    used[buf] = true;
    buf ^= 1;
    done += n;
  }
  if (n_exec) {
    HFZ_CUDA(cudaMemcpyAsync(admit, c->d_admit, n_exec, cudaMemcpyDeviceToHost, st));
    HFZ_CUDA(cudaMemcpyAsync(sigf, c->d_sigf, n_exec * 8, cudaMemcpyDeviceToHost, st));
    HFZ_CUDA(cudaMemcpyAsync(sigs, c->d_sigs, n_exec * 8, cudaMemcpyDeviceToHost, st));
    if (nnz) HFZ_CUDA(cudaMemcpyAsync(nnz, c->d_nnz, n_exec * 4, cudaMemcpyDeviceToHost, st));
  }
  HFZ_CUDA(cudaMemcpyAsync(virgin, c->d_virgin, c->S, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaMemcpyAsync(counts, c->d_counts, 16, cudaMemcpyDeviceToHost, st));
  HFZ_CUDA(cudaStreamSynchronize(st));
  return HFZ_OK;
}

// ---------------------------------------------------------------------------
// Rng helpers (host arithmetic on a scalar state; include/hetfuzz/rng.hpp:11-46)

extern "C" uint64_t hfz_rng_jump(uint64_t state, uint64_t k) { return state + k * HFZ_GAMMA; }

extern "C" uint64_t hfz_rng_next(uint64_t* state) {
  *state += HFZ_GAMMA;
  return hfz_sm64_mix(*state);
}

extern "C" uint64_t hfz_rng_below(uint64_t* state, uint64_t n) {
  if (n <= 1) return 0;
  return (uint64_t)(((unsigned __int128)hfz_rng_next(state) * n) >> 64);
}

extern "C" uint64_t hfz_rng_split(uint64_t* state, uint64_t tag) {
  const uint64_t s = hfz_rng_next(state);
  return s ^ (tag * HFZ_GAMMA) ^ 0xd1b54a32d192ed03ULL;
}
