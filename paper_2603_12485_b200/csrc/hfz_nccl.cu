// hfz_nccl.cu -- the one exchange step of the sharded campaign batch: ncclAllGather of the
// per-rank novelty deltas, followed by the rank-ordered resolve/merge.  libnccl is dlopen()ed
// so single-GPU users do not need it at load time.
#include <dlfcn.h>

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
