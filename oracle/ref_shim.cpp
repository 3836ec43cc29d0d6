// ref_shim.cpp -- C entry points around the UNMODIFIED reference implementation.
//
// TEST INFRASTRUCTURE ONLY (see oracle/hfz_oracle.c header).  This file is
// compiled by oracle/build_ref.sh together with the reference's own sources
// where they lie under /root/reference/proj/src into oracle/_ref/ (git-ignored,
// shipped to the GPU box as a prebuilt .so).  It contains no algorithm: every
// function forwards to the reference's public API (include/hetfuzz/*.hpp).
//
// Used (a) to validate the plain-C restatement in hfz_oracle.c, (b) to generate
// tests/golden/ fixtures, (c) as the "reference" CPU baseline in bench.py.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hetfuzz/coverage.hpp"
#include "hetfuzz/hdvm.hpp"
#include "hetfuzz/rng.hpp"
#ifndef REF_NO_ENGINE
#include "hetfuzz/engine.hpp"
#endif

using namespace hetfuzz;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

struct MapBatch {
  std::vector<CoverageMap> maps;
};

void fill_map(CoverageMap& m, const std::uint8_t* rec) {
  const std::uint8_t* host = rec;
  const std::uint8_t* dev = rec + kHostSlots;
  for (std::uint32_t i = 0; i < kHostSlots; ++i)
    for (unsigned k = 0; k < host[i]; ++k) m.host_increment(i);  // 1..255 -> same value
  for (std::uint32_t i = 0; i < kMapSize - kHostSlots; ++i) {
    std::uint32_t c;
    std::memcpy(&c, dev + 4ull * i, 4);
    if (c) m.device_store(kDeviceIndexBase + i, c);
  }
}

std::uint64_t rng_state(const Rng& r) {
  static_assert(sizeof(Rng) == sizeof(std::uint64_t), "Rng is one u64");
  std::uint64_t s;
  std::memcpy(&s, &r, sizeof(s));
  return s;
}

}  // namespace

REF_API std::uint32_t ref_map_size() { return kMapSize; }

REF_API std::uint8_t ref_classify_host(std::uint64_t c) {
  return BucketLadder::host().classify(c);
}
REF_API std::uint8_t ref_classify_device(std::uint64_t c) {
  return BucketLadder::device().classify(c);
}
REF_API std::uint32_t ref_device_edge_index(std::uint32_t prev, std::uint32_t cur) {
  return device_edge_index(prev, cur);
}

// Build CoverageMap objects from raw records (outside any timed region).
REF_API void* ref_maps_create(const std::uint8_t* raw, std::uint64_t n_exec) {
  auto* b = new MapBatch;
  b->maps.resize(n_exec);
  const std::uint64_t rec = std::uint64_t(kHostSlots) * 5;
  for (std::uint64_t e = 0; e < n_exec; ++e) fill_map(b->maps[e], raw + e * rec);
  return b;
}
REF_API void ref_maps_free(void* h) { delete static_cast<MapBatch*>(h); }

// The per-exec sequence of src/engine.cpp:471-478 over maps [first, first+count)
// folded in order into one VirginMap seeded from virgin_inout.
REF_API int ref_feedback_run(void* h, std::uint64_t first, std::uint64_t count,
                             std::uint8_t* virgin_inout, std::uint64_t* edge_counts_inout,
                             std::uint8_t* classed_out, std::uint8_t* admit_out,
                             std::uint64_t* sig_full_out, std::uint64_t* sig_simple_out,
                             std::uint32_t* nnz_out) {
  auto* b = static_cast<MapBatch*>(h);
  VirginMap virgin;
  for (std::uint32_t i = 0; i < kMapSize; ++i)
    if (virgin_inout[i]) virgin.observe(i, virgin_inout[i]);
  const std::uint64_t h0 = virgin.host_edges(), d0 = virgin.device_edges();
  for (std::uint64_t e = 0; e < count; ++e) {
    ClassedTrace trace = classify_trace(b->maps[first + e]);
    std::uint64_t full = trace_signature(trace, SignatureMode::Full);
    std::uint64_t simple = trace_signature(trace, SignatureMode::Simple);
    Admit adm = has_new_bits(trace, virgin);
    if (admit_out) admit_out[e] = static_cast<std::uint8_t>(adm);
    if (sig_full_out) sig_full_out[e] = full;
    if (sig_simple_out) sig_simple_out[e] = simple;
    if (nnz_out) nnz_out[e] = static_cast<std::uint32_t>(trace.nonzero.size());
    if (classed_out)
      std::memcpy(classed_out + e * std::uint64_t(kMapSize), trace.classed.data(), kMapSize);
  }
  for (std::uint32_t i = 0; i < kMapSize; ++i) virgin_inout[i] = virgin.at(i);
  edge_counts_inout[0] += virgin.host_edges() - h0;
  edge_counts_inout[1] += virgin.device_edges() - d0;
  return 0;
}

REF_API int ref_feedback_batch(const std::uint8_t* raw, std::uint64_t n_exec,
                               std::uint8_t* virgin_inout, std::uint64_t* edge_counts_inout,
                               std::uint8_t* classed_out, std::uint8_t* admit_out,
                               std::uint64_t* sig_full_out, std::uint64_t* sig_simple_out,
                               std::uint32_t* nnz_out) {
  void* h = ref_maps_create(raw, n_exec);
  int rc = ref_feedback_run(h, 0, n_exec, virgin_inout, edge_counts_inout, classed_out,
                            admit_out, sig_full_out, sig_simple_out, nnz_out);
  ref_maps_free(h);
  return rc;
}

// ---- rng -------------------------------------------------------------------

REF_API std::uint64_t ref_rng_next(std::uint64_t* state) {
  Rng r(*state);
  std::uint64_t v = r.next();
  *state = rng_state(r);
  return v;
}
REF_API std::uint64_t ref_rng_below(std::uint64_t* state, std::uint64_t n) {
  Rng r(*state);
  std::uint64_t v = r.below(n);
  *state = rng_state(r);
  return v;
}
REF_API std::uint64_t ref_rng_split(std::uint64_t* state, std::uint64_t tag) {
  Rng r(*state);
  Rng c = r.split(tag);
  *state = rng_state(r);
  return rng_state(c);
}

// ---- host edges --------------------------------------------------------------

REF_API int ref_host_edge_record(const std::uint16_t* sites, std::uint64_t n,
                                 std::uint8_t* host_half_out, std::uint64_t* violations) {
  CoverageMap map;
  HostEdgeState st;
  for (std::uint64_t i = 0; i < n; ++i) host_edge_update(st, sites[i], map);
  std::memcpy(host_half_out, map.host_half().data(), kHostSlots);
  if (violations) *violations = map.host_partition_violations();
  return 0;
}

// ---- device edge recording through the real runtime ---------------------------
// A lambda replay target (as tests/test_hdvm.cpp:66-85 builds them): kernel l's
// body replays the site list of the thread currently being simulated.  Threads
// run sequentially in (block, linear-in-block) order, so a running counter
// identifies the thread.
REF_API int ref_edge_record_exec(const std::uint32_t* dims, std::uint32_t n_launch,
                                 const std::uint64_t* ev_off, const std::uint32_t* sites,
                                 std::uint32_t* counters_out, std::uint64_t* warp_events) {
  using namespace hetfuzz::hdvm;
  TargetProgram tp;
  tp.name = "replay";
  std::vector<LaunchConfig> cfgs(n_launch);
  auto cursor = std::make_shared<std::uint64_t>(0);
  for (std::uint32_t l = 0; l < n_launch; ++l) {
    cfgs[l].grid = Dim3{dims[l * 6 + 0], dims[l * 6 + 1], dims[l * 6 + 2]};
    cfgs[l].block = Dim3{dims[l * 6 + 3], dims[l * 6 + 4], dims[l * 6 + 5]};
    KernelDescriptor kd;
    kd.name = "k" + std::to_string(l);
    kd.arg_count = 0;
    kd.body = [cursor, ev_off, sites](DeviceThreadCtx& d) {
      const std::uint64_t t = (*cursor)++;
      for (std::uint64_t e = ev_off[t]; e < ev_off[t + 1]; ++e) d.edge(sites[e]);
    };
    tp.kernels.push_back(kd);
  }
  tp.host_proc = [cfgs, n_launch](HostCtx& h) {
    for (std::uint32_t l = 0; l < n_launch; ++l) h.launch("k" + std::to_string(l), cfgs[l], {});
  };
  tp.persistent_proc = wrap_persistent(tp.host_proc);
  tp.input_format = "none";
  ExecutionReport rep = execute(tp, {});
  if (rep.exit.kind != ExitKind::Clean) return 10;
  if (!rep.api_failures.empty()) return 11;
  std::memcpy(counters_out, rep.raw_map.device_half().data(),
              std::uint64_t(kMapSize - kHostSlots) * 4);
  if (warp_events) *warp_events = rep.warp_edge_events;
  return 0;
}

// ---- mutators ------------------------------------------------------------------
#ifndef REF_NO_ENGINE

REF_API int ref_havoc(const std::uint8_t* in, std::uint64_t in_len, std::uint64_t* state,
                      std::uint8_t* out, std::uint64_t* out_len) {
  Rng rng(*state);
  std::vector<std::uint8_t> v(in, in + in_len);
  std::vector<std::uint8_t> r = havoc_mutant(v, rng);
  *state = rng_state(rng);
  if (!r.empty()) std::memcpy(out, r.data(), r.size());
  *out_len = r.size();
  return 0;
}

REF_API int ref_splice(const std::uint8_t* a, std::uint64_t a_len, const std::uint8_t* b,
                       std::uint64_t b_len, std::uint64_t* state, std::uint8_t* out,
                       std::uint64_t* out_len) {
  Rng rng(*state);
  std::vector<std::uint8_t> va(a, a + a_len), vb(b, b + b_len);
  std::vector<std::uint8_t> r = splice_mutant(va, vb, rng);
  *state = rng_state(rng);
  if (!r.empty()) std::memcpy(out, r.data(), r.size());
  *out_len = r.size();
  return 0;
}

REF_API std::uint64_t ref_deterministic(const std::uint8_t* in, std::uint64_t in_len,
                                        std::uint8_t* out) {
  std::vector<std::uint8_t> v(in, in + in_len);
  auto ms = deterministic_mutants(v);
  if (out)
    for (std::size_t i = 0; i < ms.size(); ++i)
      if (in_len) std::memcpy(out + i * in_len, ms[i].data(), in_len);
  return ms.size();
}

#endif  // REF_NO_ENGINE
