// hfz_nccl.cu -- the one exchange step of the sharded campaign batch: ncclAllGather of the
// per-rank novelty deltas, followed by the rank-ordered resolve/merge.  libnccl is dlopen()ed
// so single-GPU users do not need it at load time.
#include <dlfcn.h>
#include <string.h>

#include "hfz_common.cuh"

namespace {
typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef const char* (*nccl_errstr_fn)(int);
nccl_allgather_fn g_allgather = nullptr;
nccl_errstr_fn g_errstr = nullptr;
constexpr int kNcclUint8 = 1;  // ncclDataType_t: ncclInt8 = 0, ncclUint8 = 1

bool load_nccl() {
  if (g_allgather) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  // prefer a libnccl already mapped into the process (torch's bundled copy)
  for (const char* n : names) {
    h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);
    if (h) break;
  }
  if (!h)
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
  if (!h) return false;
  g_allgather = (nccl_allgather_fn)dlsym(h, "ncclAllGather");
  g_errstr = (nccl_errstr_fn)dlsym(h, "ncclGetErrorString");
  return g_allgather != nullptr;
}
}  // namespace

extern "C" int hfz_feedback_resolve_allgather(hfz_ctx* ctx, void* nccl_comm, const uint8_t* raw_maps,
                                              uint64_t n_exec, uint8_t* virgin_inout,
                                              uint64_t* edge_counts_inout, const uint8_t* delta_local,
                                              uint8_t* deltas_scratch, uint32_t n_ranks,
                                              uint32_t rank, uint8_t* admit_out) {
  if (!ctx || !nccl_comm || !delta_local || !deltas_scratch || n_ranks == 0 || rank >= n_ranks) {
    hfz_set_error("hfz_feedback_resolve_allgather: bad argument");
    return HFZ_EINVAL;
  }
  if (!load_nccl()) {
    hfz_set_error("hfz_feedback_resolve_allgather: libnccl.so.2 not loadable (%s)", dlerror());
    return HFZ_ENCCL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  const int rc = g_allgather(delta_local, deltas_scratch, ctx->S, kNcclUint8, nccl_comm, ctx->stream);
  if (rc != 0) {
    hfz_set_error("ncclAllGather failed: %s", g_errstr ? g_errstr(rc) : "?");
    return HFZ_ENCCL;
  }
  return hfz_feedback_resolve(ctx, raw_maps, n_exec, virgin_inout, edge_counts_inout, deltas_scratch,
                              n_ranks, rank, admit_out);
}

// ---------------------------------------------------------------------------
// Peer-visible buffers for the collective-free exchange (hfz_feedback_resolve_peers): the library
// allocates the buffer itself -- its own cudaMalloc, so the CUDA IPC handle names exactly this
// buffer at offset 0 -- and exports the 64-byte handle; the other ranks (other PROCESSES, on this or
// on a peer-accessible device) open it and pass the mapped pointer in their delta_ptrs table.
static_assert(sizeof(cudaIpcMemHandle_t) == HFZ_PEER_HANDLE_BYTES, "CUDA IPC handle size");

extern "C" int hfz_peer_alloc(hfz_ctx* ctx, uint64_t bytes, void** dev_ptr_out, uint8_t* handle_out) {
  if (!ctx || !dev_ptr_out || !handle_out || bytes == 0) {
    hfz_set_error("hfz_peer_alloc: bad argument");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    hfz_set_error("hfz_peer_alloc: cudaMalloc(%llu) failed", (unsigned long long)bytes);
    return HFZ_ENOMEM;
  }
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return hfz_cuda_fail(e, "cudaIpcGetMemHandle");
  }
  HFZ_CUDA(cudaMemsetAsync(p, 0, bytes, ctx->stream));
  memcpy(handle_out, &h, sizeof(h));
  *dev_ptr_out = p;
  return HFZ_OK;
}

extern "C" int hfz_peer_open(hfz_ctx* ctx, const uint8_t* handle, void** dev_ptr_out) {
  if (!ctx || !handle || !dev_ptr_out) {
    hfz_set_error("hfz_peer_open: bad argument");
    return HFZ_EINVAL;
  }
  HFZ_CUDA(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  HFZ_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return HFZ_OK;
}

extern "C" int hfz_peer_close(hfz_ctx* ctx, void* dev_ptr) {
  if (!ctx) return HFZ_EINVAL;
  if (!dev_ptr) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  HFZ_CUDA(cudaStreamSynchronize(ctx->stream));
  HFZ_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return HFZ_OK;
}

extern "C" int hfz_peer_free(hfz_ctx* ctx, void* dev_ptr) {
  if (!ctx) return HFZ_EINVAL;
  if (!dev_ptr) return HFZ_OK;
  HFZ_CUDA(cudaSetDevice(ctx->device));
  HFZ_CUDA(cudaStreamSynchronize(ctx->stream));
  HFZ_CUDA(cudaFree(dev_ptr));
  return HFZ_OK;
}
