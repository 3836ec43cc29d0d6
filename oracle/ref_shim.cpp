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
#include <cstdio>
#include <cstring>
#include <iterator>
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

// execs [first, first+count) of a trace batch in hfz_edge_record_batch layout, each through
// hdvm::execute as above; raw (records of S/2*5 bytes: the device half is written) and
// warp_events are indexed by exec.  One call per host thread = the CPU baseline leg of bench.py.
REF_API int ref_edge_record_range(const std::uint64_t* launch_off, const std::uint32_t* dims,
                                  const std::uint64_t* thread_off, const std::uint64_t* ev_off,
                                  const std::uint32_t* sites, std::uint64_t first, std::uint64_t count,
                                  std::uint8_t* raw, std::uint64_t* warp_events) {
  const std::uint64_t rec = std::uint64_t(kHostSlots) * 5;
  for (std::uint64_t e = first; e < first + count; ++e) {
    const std::uint64_t l0 = launch_off[e], l1 = launch_off[e + 1];
    std::uint64_t ev = 0;
    int rc = ref_edge_record_exec(dims + l0 * 6, static_cast<std::uint32_t>(l1 - l0),
                                  ev_off + (l1 > l0 ? thread_off[l0] : 0), sites,
                                  reinterpret_cast<std::uint32_t*>(raw + e * rec + kHostSlots), &ev);
    if (rc) return rc;
    if (warp_events) warp_events[e] = ev;
  }
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

// slots [first, first+count): slot j reads in[in_off[j] .. in_off[j+1]), writes at out + out_off[j]
REF_API int ref_havoc_batch(const std::uint8_t* in, const std::uint64_t* in_off, std::uint64_t first,
                            std::uint64_t count, std::uint64_t* state_inout, std::uint8_t* out,
                            const std::uint64_t* out_off, std::uint64_t* out_len) {
  for (std::uint64_t j = first; j < first + count; ++j) {
    Rng rng(state_inout[j]);
    std::vector<std::uint8_t> v(in + in_off[j], in + in_off[j + 1]);
    std::vector<std::uint8_t> r = havoc_mutant(v, rng);
    state_inout[j] = rng_state(rng);
    if (!r.empty()) std::memcpy(out + out_off[j], r.data(), r.size());
    out_len[j] = r.size();
  }
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


// ---- campaign + single executions (checker for the batch-aware campaign loop) ----
// ref_campaign_run forwards to run_campaign (engine.hpp:105); ref_execute / ref_shadow forward to
// hdvm::execute with the ExecOptions Campaign uses (engine.cpp:346-348, 396-399) plus
// derive_crash_finding / run_all_tools / dedup_key.  A test drives include/hetfuzz/campaign.hpp
// with these as its Executor and compares every field with the reference's own campaign.

namespace {

struct RefCampaign {
  CampaignConfig cfg;
  CampaignResult res;
  std::vector<std::string> texts;  // crash_report_text per crash, in map order
  std::string json, csv;
};

// findings as text: one per record-separator, fields split by unit-separator:
// key(hex16) US tool US kind US detail US site frames split by group-separator
void append_finding(std::string& out, const Finding& f) {
  char key[17];
  std::snprintf(key, sizeof key, "%016llx", static_cast<unsigned long long>(dedup_key(f)));
  out += key;
  out += '\x1f';
  out += to_string(f.tool);
  out += '\x1f';
  out += to_string(f.kind);
  out += '\x1f';
  out += f.detail;
  out += '\x1f';
  for (std::size_t i = 0; i < f.site.size(); ++i) {
    if (i) out += '\x1d';
    out += f.site[i];
  }
  out += '\x1e';
}

int copy_text(const std::string& s, char* out, std::uint64_t cap) {
  if (s.size() + 1 > cap) return 20;
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = 0;
  return 0;
}

}  // namespace

REF_API void* ref_campaign_run(const char* target, const std::uint8_t* seeds_blob,
                               const std::uint64_t* seed_off, std::uint32_t n_seeds, std::uint64_t rng_seed,
                               int strategy, int sanitizers, int device_coverage, int budget_kind,
                               std::uint64_t budget, int sequential_queue, int workers,
                               std::uint64_t stats_every, const char* out_dir) {
  auto* c = new RefCampaign;
  c->cfg.target = target;
  for (std::uint32_t i = 0; i < n_seeds; ++i)
    c->cfg.seeds.emplace_back(seeds_blob + seed_off[i], seeds_blob + seed_off[i + 1]);
  c->cfg.rng_seed = rng_seed;
  c->cfg.strategy = static_cast<Strategy>(strategy);
  c->cfg.sanitizers = sanitizers != 0;
  c->cfg.device_coverage = device_coverage != 0;
  c->cfg.budget_kind = static_cast<BudgetKind>(budget_kind);
  c->cfg.budget = budget;
  c->cfg.sequential_queue = sequential_queue != 0;
  c->cfg.workers = workers;
  c->cfg.stats_every = stats_every;
  c->cfg.out_dir = out_dir ? out_dir : "";
  try {
    c->res = run_campaign(c->cfg);
  } catch (const std::exception&) {
    delete c;
    return nullptr;
  }
  for (const auto& kv : c->res.crashes) c->texts.push_back(crash_report_text(kv.second));
  c->json = campaign_json(c->cfg, c->res);
  c->csv = plot_data_csv(c->res.stats);
  return c;
}
REF_API void ref_campaign_free(void* h) { delete static_cast<RefCampaign*>(h); }

// out[9]: execs, virtual_time, sanitizer_execs, queue size, host_edges, device_edges,
// partition_violations, crashes, stats rows
REF_API void ref_campaign_totals(void* h, std::uint64_t* out) {
  const CampaignResult& r = static_cast<RefCampaign*>(h)->res;
  out[0] = r.execs;
  out[1] = r.virtual_time;
  out[2] = r.sanitizer_execs;
  out[3] = r.queue.size();
  out[4] = r.virgin.host_edges();
  out[5] = r.virgin.device_edges();
  out[6] = r.partition_violations;
  out[7] = r.crashes.size();
  out[8] = r.stats.size();
}
// meta[7]: id, full_sig, simple_sig, admit_reason, discovered_at, parent (~0 = none), exec_cost
REF_API void ref_campaign_queue_entry(void* h, std::uint64_t i, std::uint64_t* meta,
                                      const std::uint8_t** data, std::uint64_t* len) {
  const QueueEntry& e = static_cast<RefCampaign*>(h)->res.queue[i];
  meta[0] = e.id;
  meta[1] = e.full_sig;
  meta[2] = e.simple_sig;
  meta[3] = static_cast<std::uint64_t>(e.admit_reason);
  meta[4] = e.discovered_at;
  meta[5] = e.parent ? *e.parent : ~0ull;
  meta[6] = e.exec_cost;
  *data = e.input.data();
  *len = e.input.size();
}
REF_API void ref_campaign_stats_row(void* h, std::uint64_t i, std::uint64_t* row) {
  const StatsRow& r = static_cast<RefCampaign*>(h)->res.stats[i];
  row[0] = r.virtual_time;
  row[1] = r.execs;
  row[2] = r.host_edges;
  row[3] = r.device_edges;
  row[4] = r.unique_inputs;
  row[5] = r.crashes;
  row[6] = r.sanitizer_execs;
}
// meta[4]: key, first_exposed, hits, false_positive; *text = crash_report_text
REF_API void ref_campaign_crash(void* h, std::uint64_t i, std::uint64_t* meta, const char** text) {
  auto* c = static_cast<RefCampaign*>(h);
  auto it = c->res.crashes.begin();
  std::advance(it, i);
  meta[0] = it->first;
  meta[1] = it->second.first_exposed;
  meta[2] = it->second.hits;
  meta[3] = it->second.false_positive ? 1 : 0;
  *text = c->texts[i].c_str();
}
REF_API void ref_campaign_virgin(void* h, std::uint8_t* out) {
  const VirginMap& v = static_cast<RefCampaign*>(h)->res.virgin;
  for (std::uint32_t i = 0; i < kMapSize; ++i) out[i] = v.at(i);
}
REF_API const char* ref_campaign_json(void* h) { return static_cast<RefCampaign*>(h)->json.c_str(); }
REF_API const char* ref_campaign_csv(void* h) { return static_cast<RefCampaign*>(h)->csv.c_str(); }

// The target's canonical seed corpus (TargetInfo::seeds, targets.hpp:27).
REF_API int ref_target_seeds(const char* target, std::uint8_t* blob, std::uint64_t blob_cap,
                             std::uint64_t* off, std::uint32_t* n) {
  const TargetInfo* info = find_target(target);
  if (!info) return 21;
  std::uint64_t pos = 0;
  off[0] = 0;
  *n = static_cast<std::uint32_t>(info->seeds.size());
  for (std::size_t i = 0; i < info->seeds.size(); ++i) {
    if (pos + info->seeds[i].size() > blob_cap) return 20;
    std::memcpy(blob + pos, info->seeds[i].data(), info->seeds[i].size());
    pos += info->seeds[i].size();
    off[i + 1] = pos;
  }
  return 0;
}

// One plain execution as Campaign::run_one performs it (whole-program mode, fresh process).
// raw_out: the raw record in the library layout.  out[4]: virtual_cost, partition violations,
// exit clean?, has crash finding?; text: the crash finding (see append_finding) or empty.
REF_API int ref_execute(const char* target, const std::uint8_t* in, std::uint64_t len,
                        int device_coverage, std::uint8_t* raw_out, std::uint64_t* out, char* text,
                        std::uint64_t text_cap) {
  const TargetInfo* info = find_target(target);
  if (!info) return 21;
  hdvm::ExecOptions opts;
  opts.host_coverage = true;
  opts.device_coverage = device_coverage != 0;
  opts.shadow = false;
  hdvm::ExecutionReport rep = hdvm::execute(info->program, std::vector<std::uint8_t>(in, in + len), opts);
  std::memcpy(raw_out, rep.raw_map.host_half().data(), kHostSlots);
  std::memcpy(raw_out + kHostSlots, rep.raw_map.device_half().data(), std::uint64_t(kMapSize - kHostSlots) * 4);
  out[0] = rep.virtual_cost;
  out[1] = rep.raw_map.host_partition_violations() + rep.raw_map.device_partition_violations();
  out[2] = rep.exit.kind == hdvm::ExitKind::Clean ? 1 : 0;
  out[3] = 0;
  std::string t;
  if (rep.exit.kind != hdvm::ExitKind::Clean) {
    if (auto crash = derive_crash_finding(rep)) {
      out[3] = 1;
      append_finding(t, *crash);
    }
  }
  return copy_text(t, text, text_cap);
}

// One shadow execution + all four tools (Campaign::drain_sanitizers, engine.cpp:396-417).
// out[2]: virtual_cost + records_examined, number of findings.
REF_API int ref_shadow(const char* target, const std::uint8_t* in, std::uint64_t len, std::uint64_t* out,
                       char* text, std::uint64_t text_cap) {
  const TargetInfo* info = find_target(target);
  if (!info) return 21;
  hdvm::ExecOptions opts;
  opts.host_coverage = false;
  opts.device_coverage = false;
  opts.shadow = true;
  hdvm::ExecutionReport rep = hdvm::execute(info->program, std::vector<std::uint8_t>(in, in + len), opts);
  SanitizerSweep sweep = run_all_tools(rep);
  out[0] = rep.virtual_cost + sweep.records_examined;
  out[1] = sweep.findings.size();
  std::string t;
  for (const Finding& f : sweep.findings) append_finding(t, f);
  return copy_text(t, text, text_cap);
}

#endif  // REF_NO_ENGINE
