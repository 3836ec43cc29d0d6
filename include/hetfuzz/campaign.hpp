// hetfuzz/campaign.hpp -- batch-aware campaign loop and on-disk formats.
//
// The reference's Campaign (proj/src/engine.cpp:306-593) runs ONE input at a time:
// mutate -> execute -> classify / signatures / has_new_bits -> admit -> crash / sanitizer dispatch
// -> stats.  Here the same loop runs a whole mutation stage of a queue entry as one batch --
// the deterministic stage (engine.cpp:552-558), the 48 x mult havoc mutants (:561-562), the
// 16 x mult splices (:563-566) -- with the mutators (K3) and the coverage feedback (K2, sparse
// host form) on the GPU, and produces EXACTLY the serial campaign's results: the same queue
// (inputs, signatures, reasons, parents, discovery times), the same stats rows, crash records,
// totals and output files, byte for byte.  What makes that possible:
//   * the GPU fold returns the sequential Admit codes of a batch;
//   * the havoc stage consumes the campaign's single Rng exactly like the serial loop
//     (hfz_havoc_serial_host: a length-only dry run yields every mutant's start state);
//   * a splice partner is drawn from the CURRENT queue (engine.cpp:564), so a splice batch is
//     generated speculatively for the queue as it stands and is cut at the first admission:
//     the virgin map is rolled back to the cut (64 KB host copy + re-fold of the prefix), the
//     Rng to the state after that mutant, and the rest of the stage is regenerated;
//   * a stats row needs the edge counters after one particular exec (engine.cpp:503-506), so a
//     fold never straddles a stats boundary (sub-range folds through entry_off + k).
// Target execution is NOT part of this library (the reference's simulator is out of scope):
// the caller supplies an Executor.  The queue scheduling, admission, crash bookkeeping and
// sanitizer dispatch below are host logic restated from engine.cpp with the lines cited.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <deque>
#include <filesystem>
#include <fstream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "coverage.hpp"
#include "engine.hpp"
#include "rng.hpp"

namespace hetfuzz {
namespace b200 {

using Bytes = std::vector<std::uint8_t>;

// ---- what the caller's executor reports ----------------------------------------------------

// A sanitizer / crash finding as the campaign needs it (Finding, sanitizers.hpp:36-45): the
// dedup key (sanitizers.cpp:189-198) is computed by whoever owns the analysis tools.
struct FindingInfo {
  std::uint64_t key = 0;
  std::string tool, kind, detail;
  std::vector<std::string> site;
};

struct ExecOutcome {                        // of hdvm::execute / PersistentSession::run
  std::uint64_t virtual_cost = 0;           // ExecutionReport::virtual_cost
  std::uint64_t partition_violations = 0;   // host + device partition violations of the raw map
  std::optional<FindingInfo> crash;         // derive_crash_finding() for a non-clean exit
  bool violates_invariants = false;         // launch_violates_invariants (kernel-level mode)
};

struct ShadowOutcome {                      // of one shadow execution + run_all_tools
  std::uint64_t cost = 0;                   // virtual_cost + records_examined (engine.cpp:416-417)
  std::vector<FindingInfo> findings;
  bool violates_invariants = false;
};

// CONTRACT: execute() must be a PURE function of its input -- same map, cost and outcome whatever
// was executed before (the reference's fresh-process mode, hdvm::execute).  BatchCampaign executes a
// whole mutation stage before it folds the coverage, so after a splice cut or a virtual-time stop
// inside a fold a few inputs have been executed that the serial campaign never runs; with a pure
// executor those surplus executions are invisible.  A stateful executor (the reference's
// PersistentSession: start-up cost charged once per process, iterations counted, runtime dropped
// on a crash) would see its later virtual costs shift, so CampaignConfig::persistent is rejected.
class Executor {
 public:
  virtual ~Executor() = default;
  // Runs one input; fills `map` (handed over reset) through host_increment / device_store.
  virtual ExecOutcome execute(const Bytes& input, CoverageMap& map) = 0;
  virtual ShadowOutcome shadow(const Bytes& input) = 0;
  virtual std::uint64_t persistent_processes() const { return 0; }
};

// ---- campaign types (engine.hpp:39-101, same names and meaning) -------------------------------

enum class AdmitReason : std::uint8_t { Seed, NewEdges, NewCounts };
inline const char* to_string(AdmitReason r) {  // engine.cpp:206-216
  return r == AdmitReason::Seed ? "seed" : r == AdmitReason::NewEdges ? "new-edges" : "new-counts";
}
enum class Strategy : std::uint8_t { AllTrace, UniqueTrace, SimpleTrace, CoverageIncrease };
inline const char* to_string(Strategy s) {  // sanitizers.cpp:261-273
  static const char* n[] = {"all-trace", "unique-trace", "simple-trace", "coverage-increase"};
  return n[static_cast<int>(s)];
}
inline bool should_sanitize(Strategy s, Admit admit, bool full_seen, bool simple_seen) {  // sanitizers.cpp:283-296
  switch (s) {
    case Strategy::AllTrace: return true;
    case Strategy::UniqueTrace: return !full_seen;
    case Strategy::SimpleTrace: return !simple_seen;
    case Strategy::CoverageIncrease: return admit != Admit::None;
  }
  return false;
}
enum class Mode : std::uint8_t { WholeProgram, KernelLevel };
enum class BudgetKind : std::uint8_t { Execs, VirtualTime };

struct CampaignConfig {  // engine.hpp:45-62
  std::string target;
  std::vector<Bytes> seeds;
  std::uint64_t rng_seed = 1;
  Strategy strategy = Strategy::SimpleTrace;
  Mode mode = Mode::WholeProgram;
  std::string kernel;
  bool sanitizers = true;
  bool device_coverage = true;
  bool persistent = false;
  std::uint64_t persistent_loop = 1000;
  BudgetKind budget_kind = BudgetKind::Execs;
  std::uint64_t budget = 10000;
  bool sequential_queue = false;
  int workers = 1;
  std::string out_dir;
  std::uint64_t stats_every = 100;
};

struct QueueEntry {  // engine.hpp:64-73
  std::uint64_t id = 0;
  Bytes input;
  std::uint64_t full_sig = 0, simple_sig = 0;
  AdmitReason admit_reason = AdmitReason::Seed;
  std::uint64_t discovered_at = 0;
  std::optional<std::uint64_t> parent;
  std::uint64_t exec_cost = 0;
};

struct CrashRecord {  // engine.hpp:75-81
  FindingInfo finding;
  std::uint64_t input_ref = 0, vtime = 0;  // Finding::input_ref / vtime of the first exposure
  Bytes input;
  std::uint64_t first_exposed = 0, hits = 1;
  bool false_positive = false;
};

struct StatsRow {  // engine.hpp:83-91
  std::uint64_t virtual_time = 0, execs = 0, host_edges = 0, device_edges = 0, unique_inputs = 0,
                crashes = 0, sanitizer_execs = 0;
};

struct CampaignResult {  // engine.hpp:93-103
  std::vector<QueueEntry> queue;
  std::map<std::uint64_t, CrashRecord> crashes;
  std::vector<StatsRow> stats;
  VirginMap virgin;
  std::uint64_t execs = 0, virtual_time = 0, sanitizer_execs = 0, partition_violations = 0,
                persistent_processes = 0;
  // batching telemetry (not part of the reference's result)
  std::uint64_t folds = 0, rollbacks = 0, splice_cuts = 0, gpu_mutants = 0;
};

inline std::uint64_t hash_input(const Bytes& input) {  // sanitizers.cpp:298-300
  return fnv1a_bytes(kFnvOffset, input.data(), input.size());
}

// ---- the loop ---------------------------------------------------------------------------------

class BatchCampaign {
 public:
  BatchCampaign(const CampaignConfig& cfg, Executor& exec, Context& ctx)
      : cfg_(cfg), exec_(exec), ctx_(ctx), rng_(cfg.rng_seed), next_stats_(cfg.stats_every) {
    if (ctx.map_slots() != kMapSize) throw Error("BatchCampaign: context map size != kMapSize");
    if (cfg.persistent)
      throw Error("BatchCampaign: persistent mode is not supported -- stages are executed speculatively, which is "
                          "only exact for an executor that is a pure function of its input (see Executor)");
  }

  CampaignResult run() {  // engine.cpp:569-584
    std::set<std::uint64_t> seed_hashes;
    std::vector<Bytes> seeds;
    for (const Bytes& s : cfg_.seeds)
      if (seed_hashes.insert(hash_input(s)).second) seeds.push_back(s);
    run_batch(seeds, std::nullopt, /*force_admit=*/true, /*cut_on_admit=*/false);
    while (!stop_ && !res_.queue.empty()) fuzz_entry(pick_entry());
    drain_sanitizers();
    emit_stats();
    res_.persistent_processes = exec_.persistent_processes();
    return std::move(res_);
  }

 private:
  bool budget_spent() const {  // engine.cpp:353-357
    return cfg_.budget_kind == BudgetKind::Execs ? res_.execs >= cfg_.budget : res_.virtual_time >= cfg_.budget;
  }

  void record_finding(const FindingInfo& f, const Bytes& input, std::uint64_t vtime, bool false_positive) {
    auto it = res_.crashes.find(f.key);  // engine.cpp:367-385
    if (it == res_.crashes.end()) {
      CrashRecord rec;
      rec.finding = f;
      rec.input_ref = hash_input(input);
      rec.vtime = vtime;
      rec.input = input;
      rec.first_exposed = vtime;
      rec.false_positive = false_positive;
      res_.crashes.emplace(f.key, std::move(rec));
    } else {
      ++it->second.hits;
      if (!false_positive) it->second.false_positive = false;
    }
  }

  void drain_sanitizers() {  // engine.cpp:387-424; results land in dispatch order
    for (const auto& job : pending_) {
      ShadowOutcome s = exec_.shadow(job.first);
      ++res_.sanitizer_execs;
      res_.virtual_time += s.cost;
      for (const FindingInfo& f : s.findings) record_finding(f, job.first, job.second, s.violates_invariants);
    }
    pending_.clear();
  }

  void emit_stats() {  // engine.cpp:426-437
    drain_sanitizers();
    StatsRow row;
    row.virtual_time = res_.virtual_time;
    row.execs = res_.execs;
    row.host_edges = res_.virgin.host_edges();
    row.device_edges = res_.virgin.device_edges();
    row.unique_inputs = res_.queue.size();
    row.crashes = res_.crashes.size();
    row.sanitizer_execs = res_.sanitizer_execs;
    res_.stats.push_back(row);
  }

  void admit(const Bytes& input, std::uint64_t full, std::uint64_t simple, AdmitReason reason,
             std::optional<std::uint64_t> parent, std::uint64_t cost) {  // engine.cpp:439-454
    QueueEntry e;
    e.id = res_.queue.size();
    e.input = input;
    e.full_sig = full;
    e.simple_sig = simple;
    e.admit_reason = reason;
    e.discovered_at = res_.virtual_time;
    e.parent = parent;
    e.exec_cost = cost;
    res_.queue.push_back(std::move(e));
    det_done_.push_back(false);
    fresh_.push_back(res_.queue.size() - 1);
  }

  // Everything run_one does after the execution (engine.cpp:465-507), from batch results.
  // Returns true when the input was admitted.
  bool account(const Bytes& input, const ExecOutcome& o, Admit adm, std::uint64_t full, std::uint64_t simple,
               std::optional<std::uint64_t> parent, bool force_admit) {
    ++res_.execs;
    res_.virtual_time += o.virtual_cost;
    res_.partition_violations += o.partition_violations;
    const bool full_seen = full_sigs_.count(full) > 0, simple_seen = simple_sigs_.count(simple) > 0;
    full_sigs_.insert(full);
    simple_sigs_.insert(simple);
    bool admitted = true;
    if (force_admit)
      admit(input, full, simple, AdmitReason::Seed, parent, o.virtual_cost);
    else if (adm == Admit::NewEdges)
      admit(input, full, simple, AdmitReason::NewEdges, parent, o.virtual_cost);
    else if (adm == Admit::NewCounts)
      admit(input, full, simple, AdmitReason::NewCounts, parent, o.virtual_cost);
    else
      admitted = false;
    if (o.crash) record_finding(*o.crash, input, res_.virtual_time, o.violates_invariants);
    if (cfg_.sanitizers && should_sanitize(cfg_.strategy, adm, full_seen, simple_seen)) {
      pending_.emplace_back(input, res_.virtual_time);
      if (pending_.size() >= static_cast<std::size_t>(std::max(1, cfg_.workers))) drain_sanitizers();
    }
    if (res_.execs >= next_stats_) {
      emit_stats();
      next_stats_ += cfg_.stats_every;
    }
    return admitted;
  }

  // Runs `inputs` in order exactly like consecutive run_one calls.  Returns how many were
  // consumed: all of them, fewer when the budget ran out (stop_ set) or -- with cut_on_admit --
  // up to and including the first admitted input (the caller regenerates the rest).
  std::size_t run_batch(const std::vector<Bytes>& inputs, std::optional<std::uint64_t> parent, bool force_admit,
                        bool cut_on_admit) {
    std::size_t n = inputs.size();
    if (n == 0 || stop_) return 0;
    if (budget_spent()) {  // engine.cpp:460-463
      stop_ = true;
      return 0;
    }
    if (cfg_.budget_kind == BudgetKind::Execs && cfg_.budget - res_.execs < n)
      n = static_cast<std::size_t>(cfg_.budget - res_.execs);  // never execute past an exec budget
    if (cfg_.budget_kind == BudgetKind::VirtualTime && n > kTimeBudgetBatch) {
      // a time budget can run out anywhere: bound how far past it the executor may run by
      // handing a long stage over in pieces (consecutive run_one calls either way)
      std::size_t done = 0;
      while (done < inputs.size() && !stop_) {
        const std::size_t m = std::min(kTimeBudgetBatch, inputs.size() - done);
        const std::vector<Bytes> piece(inputs.begin() + done, inputs.begin() + done + m);
        const std::size_t used = run_batch(piece, parent, force_admit, cut_on_admit);
        done += used;
        if (used < m) break;  // stopped, or cut at an admission
      }
      return done;
    }
    batch_.clear();
    std::vector<ExecOutcome> out(n);
    for (std::size_t i = 0; i < n; ++i) {
      map_.reset();
      out[i] = exec_.execute(inputs[i], map_);
      out[i].partition_violations += map_.host_partition_violations() + map_.device_partition_violations();
      batch_.append(map_);
    }
    std::size_t p = 0;
    while (p < n) {
      if (budget_spent()) {  // engine.cpp:460-463
        stop_ = true;
        return p;
      }
      // a fold must not straddle a stats row: it ends with the exec that reaches next_stats
      std::size_t end = n;
      if (next_stats_ <= res_.execs)
        end = p + 1;
      else if (next_stats_ - res_.execs < end - p)
        end = p + static_cast<std::size_t>(next_stats_ - res_.execs);
      const bool may_cut = cut_on_admit || cfg_.budget_kind == BudgetKind::VirtualTime;
      if (may_cut) save_virgin();
      FeedbackResult fb = fold(p, end);
      for (std::size_t i = p; i < end; ++i) {
        if (i > p && budget_spent()) {  // only a virtual-time budget can run out inside a fold
          refold(p, i);
          stop_ = true;
          return i;
        }
        const bool admitted = account(inputs[i], out[i], static_cast<Admit>(fb.admit[i - p]), fb.sig_full[i - p],
                                      fb.sig_simple[i - p], parent, force_admit);
        if (cut_on_admit && admitted && i + 1 < inputs.size()) {  // later mutants were drawn for a shorter queue
          ++res_.splice_cuts;
          if (i + 1 < end) refold(p, i + 1);
          return i + 1;
        }
      }
      p = end;
    }
    if (n < inputs.size()) stop_ = true;  // the next run_one call finds the exec budget spent
    return n;
  }

  FeedbackResult fold(std::size_t first, std::size_t last) {
    ++res_.folds;
    FeedbackResult r;
    const std::uint64_t n = last - first;
    r.admit.resize(n);
    r.sig_full.resize(n);
    r.sig_simple.resize(n);
    check(hfz_feedback_batch_compact_host(ctx_.get(), batch_.compact(), batch_.compact_offsets() + first,
                                          batch_.wide(), batch_.wide_offsets() + first, n, res_.virgin.data(),
                                          res_.virgin.edge_counts(), nullptr, r.admit.data(), r.sig_full.data(),
                                          r.sig_simple.data(), nullptr),
          "hfz_feedback_batch_compact_host");
    return r;
  }
  void save_virgin() {
    saved_bits_.assign(res_.virgin.data(), res_.virgin.data() + kMapSize);
    saved_edges_[0] = res_.virgin.edge_counts()[0];
    saved_edges_[1] = res_.virgin.edge_counts()[1];
  }
  void refold(std::size_t first, std::size_t last) {  // virgin := state after exec last-1
    ++res_.rollbacks;
    std::copy(saved_bits_.begin(), saved_bits_.end(), res_.virgin.data());
    res_.virgin.edge_counts()[0] = saved_edges_[0];
    res_.virgin.edge_counts()[1] = saved_edges_[1];
    if (last > first) fold(first, last);
  }

  void refresh_medians() {  // engine.cpp:510-528
    if (have_medians_ && res_.execs - medians_at_execs_ < 4096 && res_.queue.size() - medians_at_queue_ < 64) return;
    std::vector<std::uint64_t> lens, costs;
    for (const auto& e : res_.queue) {
      lens.push_back(e.input.size());
      costs.push_back(e.exec_cost);
    }
    std::sort(lens.begin(), lens.end());
    std::sort(costs.begin(), costs.end());
    len_median_ = lens[(lens.size() - 1) / 2];
    cost_median_ = costs[(costs.size() - 1) / 2];
    have_medians_ = true;
    medians_at_execs_ = res_.execs;
    medians_at_queue_ = res_.queue.size();
  }
  bool favored(std::size_t idx) {  // engine.cpp:530-534
    refresh_medians();
    return res_.queue[idx].input.size() <= len_median_ && res_.queue[idx].exec_cost <= cost_median_;
  }
  std::size_t pick_entry() {  // engine.cpp:536-545
    if (!cfg_.sequential_queue && !fresh_.empty()) {
      const std::size_t idx = fresh_.front();
      fresh_.pop_front();
      return idx;
    }
    const std::size_t idx = cursor_ % res_.queue.size();
    ++cursor_;
    return idx;
  }

  void fuzz_entry(std::size_t idx) {  // engine.cpp:547-567
    const Bytes input = res_.queue[idx].input;
    const std::uint64_t id = res_.queue[idx].id;
    if (!det_done_[idx]) {
      det_done_[idx] = true;
      std::vector<Bytes> det = deterministic_mutants(input);  // K3, RNG-free
      res_.gpu_mutants += det.size();
      run_batch(det, id, false, false);
      if (stop_) return;
    }
    const int mult = favored(idx) ? 2 : 1;
    if (!stop_) {  // 48 x mult havoc mutants off the campaign's single Rng
      std::vector<Bytes> hv = havoc_stage(input, 48 * mult);
      run_batch(hv, id, false, false);
    }
    int done = 0;
    while (done < 16 * mult && !stop_) {  // splices: regenerate after every admission
      std::vector<std::uint64_t> state_after;
      std::vector<Bytes> sp = splice_stage(input, 16 * mult - done, state_after);
      const std::size_t used = run_batch(sp, id, false, true);
      if (stop_) break;
      rng_.set_state(state_after[used - 1]);  // mutants past the cut were never drawn
      done += static_cast<int>(used);
    }
  }

  std::vector<Bytes> havoc_stage(const Bytes& input, int n) {
    std::vector<std::uint64_t> in_off(n + 1), out_off(n + 1, 0), out_len(n);
    const std::uint64_t cap = (hfz_havoc_max_out(input.size()) + 15) & ~std::uint64_t(15);
    Bytes blob;
    blob.reserve(input.size() * n + 16);
    for (int j = 0; j < n; ++j) {
      in_off[j] = blob.size();
      blob.insert(blob.end(), input.begin(), input.end());
      out_off[j + 1] = out_off[j] + cap;
    }
    in_off[n] = blob.size();
    blob.resize(blob.size() + 16);
    Bytes out(out_off[n] + 16);
    std::uint64_t state = rng_.state();
    check(hfz_havoc_serial_host(ctx_.get(), blob.data(), in_off.data(), n, &state, out.data(), out_off.data(),
                                out_len.data()),
          "hfz_havoc_serial_host");
    rng_.set_state(state);
    res_.gpu_mutants += n;
    std::vector<Bytes> res(n);
    for (int j = 0; j < n; ++j) res[j].assign(out.begin() + out_off[j], out.begin() + out_off[j] + out_len[j]);
    return res;
  }

  // n splices against the queue as it stands (engine.cpp:563-566).  Per mutant the serial loop
  // draws the partner (below(queue size)) and then splice_mutant draws two cut points
  // (engine.cpp:195-204; below(n <= 1) draws nothing): the host walks those draws to get each
  // mutant's start state, the device cuts and joins (K3 splice).
  std::vector<Bytes> splice_stage(const Bytes& input, int n, std::vector<std::uint64_t>& state_after) {
    std::vector<std::uint32_t> a_idx(n, 0), b_idx(n);
    std::vector<std::uint64_t> state(n), out_off(n + 1, 0), out_len(n);
    std::map<std::size_t, std::uint32_t> slot_of;  // queue index -> packed input index
    std::vector<std::uint64_t> in_off{0, input.size()};
    Bytes blob(input);
    state_after.resize(n);
    for (int j = 0; j < n; ++j) {
      const std::size_t other = rng_.below(res_.queue.size());
      auto it = slot_of.find(other);
      if (it == slot_of.end()) {
        const Bytes& ob = res_.queue[other].input;
        blob.insert(blob.end(), ob.begin(), ob.end());
        in_off.push_back(blob.size());
        it = slot_of.emplace(other, static_cast<std::uint32_t>(in_off.size() - 2)).first;
      }
      b_idx[j] = it->second;
      const std::uint64_t blen = res_.queue[other].input.size();
      state[j] = rng_.state();
      rng_.jump((input.size() + 1 > 1 ? 1 : 0) + (blen + 1 > 1 ? 1 : 0));
      state_after[j] = rng_.state();
      std::uint64_t cap = input.size() + blen;
      if (cap > kMaxInputBytes) cap = kMaxInputBytes;
      out_off[j + 1] = out_off[j] + ((cap + 15) & ~std::uint64_t(15));
    }
    blob.resize(blob.size() + 16);
    Bytes out(out_off[n] + 16);
    check(hfz_splice_batch_host(ctx_.get(), blob.data(), in_off.data(), in_off.size() - 1, a_idx.data(), b_idx.data(), n,
                                state.data(), out.data(), out_off.data(), out_len.data()),
          "hfz_splice_batch_host");
    for (int j = 0; j < n; ++j)
      if (state[j] != state_after[j]) throw Error("splice_stage: draw count differs from the device's");
    res_.gpu_mutants += n;
    std::vector<Bytes> res(n);
    for (int j = 0; j < n; ++j) res[j].assign(out.begin() + out_off[j], out.begin() + out_off[j] + out_len[j]);
    return res;
  }

  static constexpr std::size_t kTimeBudgetBatch = 256;
  const CampaignConfig& cfg_;
  Executor& exec_;
  Context& ctx_;
  Rng rng_;
  CampaignResult res_;
  std::set<std::uint64_t> full_sigs_, simple_sigs_;
  std::vector<bool> det_done_;
  std::deque<std::size_t> fresh_;
  std::size_t cursor_ = 0;
  std::vector<std::pair<Bytes, std::uint64_t>> pending_;  // SanJob: input, dispatch vtime
  std::uint64_t next_stats_;
  bool stop_ = false;
  std::uint64_t len_median_ = 0, cost_median_ = 0, medians_at_execs_ = 0;
  bool have_medians_ = false;
  std::size_t medians_at_queue_ = 0;
  CoverageMap map_;
  CompactBatch batch_;
  std::vector<std::uint8_t> saved_bits_;
  std::uint64_t saved_edges_[2] = {0, 0};
};

// ---- on-disk formats (engine.cpp:626-737) ---------------------------------------------------------

inline std::string crash_key_hex(std::uint64_t key) {
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(key));
  return buf;
}

inline std::string plot_data_csv(const std::vector<StatsRow>& rows) {
  std::ostringstream os;
  os << "virtual_time,execs,host_edges,device_edges,unique_inputs,crashes,sanitizer_execs\n";
  for (const auto& r : rows)
    os << r.virtual_time << ',' << r.execs << ',' << r.host_edges << ',' << r.device_edges << ','
       << r.unique_inputs << ',' << r.crashes << ',' << r.sanitizer_execs << '\n';
  return os.str();
}

inline std::string crash_report_text(const CrashRecord& rec) {
  std::ostringstream os;
  os << "tool: " << rec.finding.tool << '\n' << "kind: " << rec.finding.kind << '\n' << "site:";
  for (const auto& frame : rec.finding.site) os << ' ' << frame;
  os << '\n' << "detail: " << rec.finding.detail << '\n';
  os << "input_ref: " << crash_key_hex(rec.input_ref) << '\n';
  os << "virtual_time: " << rec.first_exposed << '\n' << "hits: " << rec.hits << '\n';
  os << "false_positive: " << (rec.false_positive ? "yes" : "no") << '\n';
  return os.str();
}

namespace detail {
// Just enough JSON to reproduce nlohmann::json::dump(2) for campaign.json: objects print their
// keys in sorted order, one member per line; arrays one element per line; [] and {} when empty.
struct Json {
  enum Kind { Obj, Arr, Str, U64, Bool } kind = Obj;
  std::map<std::string, Json> obj;
  std::vector<Json> arr;
  std::string str;
  std::uint64_t u = 0;
  bool b = false;
  static Json S(const std::string& s) { Json j; j.kind = Str; j.str = s; return j; }
  static Json U(std::uint64_t v) { Json j; j.kind = U64; j.u = v; return j; }
  static Json B(bool v) { Json j; j.kind = Bool; j.b = v; return j; }
  static Json A() { Json j; j.kind = Arr; return j; }
  Json& operator[](const std::string& k) { return obj[k]; }
  static void quote(std::ostream& os, const std::string& s) {
    os << '"';
    for (unsigned char c : s) {
      switch (c) {
        case '"': os << "\\\""; break;
        case '\\': os << "\\\\"; break;
        case '\b': os << "\\b"; break;
        case '\f': os << "\\f"; break;
        case '\n': os << "\\n"; break;
        case '\r': os << "\\r"; break;
        case '\t': os << "\\t"; break;
        default:
          if (c < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\u%04x", c);
            os << buf;
          } else {
            os << static_cast<char>(c);
          }
      }
    }
    os << '"';
  }
  void dump(std::ostream& os, int indent, int cur = 0) const {
    const std::string pad(cur + indent, ' '), close(cur, ' ');
    switch (kind) {
      case Str: quote(os, str); break;
      case U64: os << u; break;
      case Bool: os << (b ? "true" : "false"); break;
      case Arr:
        if (arr.empty()) { os << "[]"; break; }
        os << "[\n";
        for (std::size_t i = 0; i < arr.size(); ++i) {
          os << pad;
          arr[i].dump(os, indent, cur + indent);
          os << (i + 1 < arr.size() ? ",\n" : "\n");
        }
        os << close << ']';
        break;
      case Obj: {
        if (obj.empty()) { os << "{}"; break; }
        os << "{\n";
        std::size_t i = 0;
        for (const auto& kv : obj) {
          os << pad;
          quote(os, kv.first);
          os << ": ";
          kv.second.dump(os, indent, cur + indent);
          os << (++i < obj.size() ? ",\n" : "\n");
        }
        os << close << '}';
        break;
      }
    }
  }
};
}  // namespace detail

inline std::string campaign_json(const CampaignConfig& cfg, const CampaignResult& res) {  // engine.cpp:659-703
  using detail::Json;
  Json j;
  j["target"] = Json::S(cfg.target);
  j["mode"] = Json::S(cfg.mode == Mode::KernelLevel ? "kernel-level" : "whole-program");
  if (cfg.mode == Mode::KernelLevel) j["kernel"] = Json::S(cfg.kernel);
  j["strategy"] = Json::S(to_string(cfg.strategy));
  j["rng_seed"] = Json::U(cfg.rng_seed);
  j["budget"]["kind"] = Json::S(cfg.budget_kind == BudgetKind::Execs ? "execs" : "virtual-time");
  j["budget"]["value"] = Json::U(cfg.budget);
  j["sanitizers"] = Json::B(cfg.sanitizers);
  j["device_coverage"] = Json::B(cfg.device_coverage);
  j["persistent"]["enabled"] = Json::B(cfg.persistent);
  j["persistent"]["loop"] = Json::U(cfg.persistent_loop);
  j["sequential_queue"] = Json::B(cfg.sequential_queue);
  j["workers"] = Json::U(static_cast<std::uint64_t>(cfg.workers));
  Json& t = j["totals"];
  t["execs"] = Json::U(res.execs);
  t["virtual_time"] = Json::U(res.virtual_time);
  t["sanitizer_execs"] = Json::U(res.sanitizer_execs);
  t["unique_inputs"] = Json::U(res.queue.size());
  t["host_edges"] = Json::U(res.virgin.host_edges());
  t["device_edges"] = Json::U(res.virgin.device_edges());
  t["partition_violations"] = Json::U(res.partition_violations);
  t["persistent_processes"] = Json::U(res.persistent_processes);
  std::map<std::string, std::uint64_t> per_tool;
  Json crashes = Json::A();
  for (const auto& [key, rec] : res.crashes) {
    ++per_tool[rec.finding.tool];
    Json c;
    c["key"] = Json::S(crash_key_hex(key));
    c["tool"] = Json::S(rec.finding.tool);
    c["kind"] = Json::S(rec.finding.kind);
    Json site = Json::A();
    for (const auto& f : rec.finding.site) site.arr.push_back(Json::S(f));
    c["site"] = site;
    c["first_exposed"] = Json::U(rec.first_exposed);
    c["hits"] = Json::U(rec.hits);
    c["false_positive"] = Json::B(rec.false_positive);
    crashes.arr.push_back(c);
  }
  j["crashes"] = crashes;
  Json& pt = j["findings_per_tool"];
  pt.kind = Json::Obj;
  for (const auto& kv : per_tool) pt[kv.first] = Json::U(kv.second);
  std::ostringstream os;
  j.dump(os, 2);
  os << '\n';
  return os.str();
}

inline void write_out_dir(const std::string& dir, const CampaignConfig& cfg, const CampaignResult& res) {
  namespace fs = std::filesystem;  // engine.cpp:705-737
  fs::create_directories(fs::path(dir) / "queue");
  fs::create_directories(fs::path(dir) / "crashes");
  for (const auto& e : res.queue) {
    char name[32];
    std::snprintf(name, sizeof name, "id_%06llu.bin", static_cast<unsigned long long>(e.id));
    std::ofstream f(fs::path(dir) / "queue" / name, std::ios::binary);
    f.write(reinterpret_cast<const char*>(e.input.data()), static_cast<std::streamsize>(e.input.size()));
  }
  for (const auto& [key, rec] : res.crashes) {
    const fs::path cdir = fs::path(dir) / "crashes" / crash_key_hex(key);
    fs::create_directories(cdir);
    {
      std::ofstream f(cdir / "input.bin", std::ios::binary);
      f.write(reinterpret_cast<const char*>(rec.input.data()), static_cast<std::streamsize>(rec.input.size()));
    }
    std::ofstream f(cdir / "report.txt");
    f << crash_report_text(rec);
  }
  {
    std::ofstream f(fs::path(dir) / "plot_data.csv");
    f << plot_data_csv(res.stats);
  }
  std::ofstream f(fs::path(dir) / "campaign.json");
  f << campaign_json(cfg, res);
}

// run_campaign (engine.cpp:586-593) over a caller-supplied executor.
inline CampaignResult run_campaign(const CampaignConfig& cfg, Executor& exec, Context& ctx) {
  if (cfg.seeds.empty() || cfg.seeds.size() > 5) throw std::invalid_argument("campaign needs 1 to 5 seeds");
  BatchCampaign c(cfg, exec, ctx);
  CampaignResult res = c.run();
  if (!cfg.out_dir.empty()) write_out_dir(cfg.out_dir, cfg, res);
  return res;
}

}  // namespace b200
}  // namespace hetfuzz
