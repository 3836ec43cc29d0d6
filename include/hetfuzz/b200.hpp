// hetfuzz/b200.hpp -- C++ convenience layer over the C-ABI (include/hfz.h): RAII context,
// error translation, batched host-buffer calls.  Header-only; link with libhfz.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../hfz.h"

// Built against the reference's own tree (its include directory AFTER this one on the include
// path, so that hdvm.hpp / sanitizers.hpp / targets.hpp / engine.hpp are the reference's)?
#if defined(__has_include)
#if __has_include("hetfuzz/hdvm.hpp")
#define HETFUZZ_B200_WITH_REFERENCE 1
#endif
#endif

namespace hetfuzz {

namespace b200 {

// A failure of the library itself (CUDA error, missing GPU): the role of the reference's
// InternalError (include/hetfuzz/hdvm.hpp:16-18), which its CLI maps to exit code 3.  It is its own
// type so that this header never collides with the reference's definition when both are in one
// translation unit; without the reference on the include path hetfuzz::InternalError names it.
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc, const char* what) {
  if (rc != HFZ_OK)
    throw Error(std::string(what) + ": " + hfz_last_error() + " (hfz error " + std::to_string(rc) + ")");
}

class Context {
 public:
  explicit Context(int device = 0, std::uint32_t map_slots = 65536, void* stream = nullptr) {
    check(hfz_ctx_create(&ctx_, device, map_slots, stream), "hfz_ctx_create");
  }
  ~Context() { hfz_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  hfz_ctx* get() const { return ctx_; }
  std::uint32_t map_slots() const { return hfz_ctx_map_slots(ctx_); }

 private:
  hfz_ctx* ctx_ = nullptr;
};

// One lazily created context per host thread for the reference-named single-item calls.
inline Context& default_context(std::uint32_t map_slots = 65536) {
  thread_local Context ctx(0, map_slots);
  if (ctx.map_slots() != map_slots) throw Error("default_context: map size differs from the first use");
  return ctx;
}

struct FeedbackResult {
  std::vector<std::uint8_t> admit;
  std::vector<std::uint64_t> sig_full, sig_simple;
  std::vector<std::uint32_t> nnz;
  std::vector<std::uint8_t> classed;  // n x S when requested
};

// raw: n records of 5*S/2 bytes; virgin (S bytes) and edge_counts {host, device} are folded in place.
inline FeedbackResult feedback_batch(Context& ctx, const std::uint8_t* raw, std::uint64_t n,
                                     std::uint8_t* virgin, std::uint64_t* edge_counts,
                                     bool want_classed = false) {
  FeedbackResult r;
  r.admit.resize(n);
  r.sig_full.resize(n);
  r.sig_simple.resize(n);
  r.nnz.resize(n);
  if (want_classed) r.classed.resize(n * std::uint64_t(ctx.map_slots()));
  check(hfz_feedback_batch_host(ctx.get(), raw, n, virgin, edge_counts,
                                want_classed ? r.classed.data() : nullptr, r.admit.data(),
                                r.sig_full.data(), r.sig_simple.data(), r.nnz.data()),
        "hfz_feedback_batch_host");
  return r;
}

}  // namespace b200

#ifndef HETFUZZ_B200_WITH_REFERENCE
using InternalError = b200::Error;
#endif

}  // namespace hetfuzz
