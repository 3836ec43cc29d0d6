// Batch-aware campaign loop (include/hetfuzz/campaign.hpp) against the
// reference's own serial campaign.  The reference library (oracle/_ref/libhetfuzz_ref.so, the
// UNMODIFIED reference + oracle/ref_shim.cpp) is dlopen()ed: it runs run_campaign as the
// expectation AND serves as this test's Executor (target execution is out of scope for the
// library under test).  Every field of the result must match: queue entries, stats rows,
// totals, crash records, virgin map, plot_data.csv, campaign.json and the output directory.
//
//   campaign_test <libhetfuzz_ref.so> <out_dir>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hetfuzz/campaign.hpp"

using namespace hetfuzz;
using namespace hetfuzz::b200;

static int g_fail = 0;
static unsigned long long g_splice_cuts = 0, g_rollbacks = 0;
#define REQUIRE(c)                                               \
  do {                                                           \
    if (!(c)) {                                                  \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                  \
    }                                                            \
  } while (0)

struct RefLib {
  void* h = nullptr;
  void* (*campaign_run)(const char*, const std::uint8_t*, const std::uint64_t*, std::uint32_t, std::uint64_t, int, int,
                        int, int, std::uint64_t, int, int, std::uint64_t, const char*);
  void (*campaign_free)(void*);
  void (*campaign_totals)(void*, std::uint64_t*);
  void (*campaign_queue_entry)(void*, std::uint64_t, std::uint64_t*, const std::uint8_t**, std::uint64_t*);
  void (*campaign_stats_row)(void*, std::uint64_t, std::uint64_t*);
  void (*campaign_crash)(void*, std::uint64_t, std::uint64_t*, const char**);
  void (*campaign_virgin)(void*, std::uint8_t*);
  const char* (*campaign_json)(void*);
  const char* (*campaign_csv)(void*);
  int (*target_seeds)(const char*, std::uint8_t*, std::uint64_t, std::uint64_t*, std::uint32_t*);
  int (*execute)(const char*, const std::uint8_t*, std::uint64_t, int, std::uint8_t*, std::uint64_t*, char*,
                 std::uint64_t);
  int (*shadow)(const char*, const std::uint8_t*, std::uint64_t, std::uint64_t*, char*, std::uint64_t);
  template <class F>
  void sym(F& f, const char* name) {
    f = reinterpret_cast<F>(dlsym(h, name));
    if (!f) {
      std::printf("missing symbol %s\n", name);
      std::exit(2);
    }
  }
  explicit RefLib(const char* path) {
    h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      std::printf("dlopen(%s): %s\n", path, dlerror());
      std::exit(2);
    }
    sym(campaign_run, "ref_campaign_run");
    sym(campaign_free, "ref_campaign_free");
    sym(campaign_totals, "ref_campaign_totals");
    sym(campaign_queue_entry, "ref_campaign_queue_entry");
    sym(campaign_stats_row, "ref_campaign_stats_row");
    sym(campaign_crash, "ref_campaign_crash");
    sym(campaign_virgin, "ref_campaign_virgin");
    sym(campaign_json, "ref_campaign_json");
    sym(campaign_csv, "ref_campaign_csv");
    sym(target_seeds, "ref_target_seeds");
    sym(execute, "ref_execute");
    sym(shadow, "ref_shadow");
  }
};

static std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::size_t p = 0;
  for (;;) {
    const std::size_t q = s.find(sep, p);
    if (q == std::string::npos) {
      out.push_back(s.substr(p));
      return out;
    }
    out.push_back(s.substr(p, q - p));
    p = q + 1;
  }
}

static std::vector<FindingInfo> parse_findings(const std::string& text) {
  std::vector<FindingInfo> out;
  for (const std::string& rec : split(text, '\x1e')) {
    if (rec.empty()) continue;
    const std::vector<std::string> f = split(rec, '\x1f');
    FindingInfo fi;
    fi.key = std::strtoull(f[0].c_str(), nullptr, 16);
    fi.tool = f[1];
    fi.kind = f[2];
    fi.detail = f[3];
    if (f.size() > 4 && !f[4].empty()) fi.site = split(f[4], '\x1d');
    out.push_back(fi);
  }
  return out;
}

// Executor backed by the reference's simulator.
class RefExecutor : public Executor {
 public:
  RefExecutor(RefLib& lib, std::string target, bool device_coverage)
      : lib_(lib), target_(std::move(target)), devcov_(device_coverage), raw_(std::size_t(kHostSlots) * 5),
        text_(1 << 16) {}
  ExecOutcome execute(const Bytes& input, CoverageMap& map) override {
    std::uint64_t o[4];
    const int rc = lib_.execute(target_.c_str(), input.data(), input.size(), devcov_ ? 1 : 0, raw_.data(), o,
                                text_.data(), text_.size());
    if (rc) {
      std::printf("ref_execute failed: %d\n", rc);
      std::exit(2);
    }
    for (std::uint32_t i = 0; i < kHostSlots; ++i)
      if (raw_[i]) map.host_assign(i, raw_[i]);
    for (std::uint32_t i = 0; i < kHostSlots; ++i) {
      std::uint32_t c;
      std::memcpy(&c, &raw_[kHostSlots + std::size_t(i) * 4], 4);
      if (c) map.device_store(kDeviceIndexBase + i, c);
    }
    ExecOutcome out;
    out.virtual_cost = o[0];
    out.partition_violations = o[1];
    if (o[3]) out.crash = parse_findings(text_.data())[0];
    ++execs;
    return out;
  }
  ShadowOutcome shadow(const Bytes& input) override {
    std::uint64_t o[2];
    const int rc = lib_.shadow(target_.c_str(), input.data(), input.size(), o, text_.data(), text_.size());
    if (rc) {
      std::printf("ref_shadow failed: %d\n", rc);
      std::exit(2);
    }
    ShadowOutcome out;
    out.cost = o[0];
    out.findings = parse_findings(text_.data());
    return out;
  }
  std::uint64_t execs = 0;

 private:
  RefLib& lib_;
  std::string target_;
  bool devcov_;
  std::vector<std::uint8_t> raw_;
  std::vector<char> text_;
};

struct Case {
  const char* target;
  std::uint64_t rng_seed, budget;
  Strategy strategy;
  bool sanitizers, sequential_queue;
  BudgetKind budget_kind;
  std::uint64_t stats_every;
  int workers;
};

static void run_case(RefLib& lib, Context& ctx, const Case& cs, const std::string& out_root, int index) {
  CampaignConfig cfg;
  cfg.target = cs.target;
  cfg.rng_seed = cs.rng_seed;
  cfg.budget = cs.budget;
  cfg.budget_kind = cs.budget_kind;
  cfg.strategy = cs.strategy;
  cfg.sanitizers = cs.sanitizers;
  cfg.sequential_queue = cs.sequential_queue;
  cfg.stats_every = cs.stats_every;
  cfg.workers = cs.workers;
  std::vector<std::uint8_t> blob(1 << 20);
  std::uint64_t off[8];
  std::uint32_t n_seeds = 0;
  if (lib.target_seeds(cs.target, blob.data(), blob.size(), off, &n_seeds)) {
    std::printf("no such target %s\n", cs.target);
    ++g_fail;
    return;
  }
  for (std::uint32_t i = 0; i < n_seeds; ++i) cfg.seeds.emplace_back(blob.begin() + off[i], blob.begin() + off[i + 1]);
  const std::string ref_dir = out_root + "/case" + std::to_string(index) + "_ref";
  cfg.out_dir = out_root + "/case" + std::to_string(index) + "_b200";

  void* ref = lib.campaign_run(cs.target, blob.data(), off, n_seeds, cfg.rng_seed, static_cast<int>(cfg.strategy),
                               cfg.sanitizers, cfg.device_coverage, static_cast<int>(cfg.budget_kind), cfg.budget,
                               cfg.sequential_queue, cfg.workers, cfg.stats_every, ref_dir.c_str());
  REQUIRE(ref != nullptr);
  if (!ref) return;

  RefExecutor exec(lib, cs.target, cfg.device_coverage);
  CampaignResult res = run_campaign(cfg, exec, ctx);

  std::uint64_t t[9];
  lib.campaign_totals(ref, t);
  std::printf("case %d %-20s budget %llu: execs %llu queue %zu crashes %zu stats %zu | folds %llu rollbacks %llu "
              "splice cuts %llu gpu mutants %llu executor calls %llu\n",
              index, cs.target, (unsigned long long)cs.budget, (unsigned long long)res.execs, res.queue.size(),
              res.crashes.size(), res.stats.size(), (unsigned long long)res.folds, (unsigned long long)res.rollbacks,
              (unsigned long long)res.splice_cuts, (unsigned long long)res.gpu_mutants, (unsigned long long)exec.execs);
  REQUIRE(res.execs == t[0]);
  REQUIRE(res.virtual_time == t[1]);
  REQUIRE(res.sanitizer_execs == t[2]);
  REQUIRE(res.queue.size() == t[3]);
  REQUIRE(res.virgin.host_edges() == t[4]);
  REQUIRE(res.virgin.device_edges() == t[5]);
  REQUIRE(res.partition_violations == t[6]);
  REQUIRE(res.crashes.size() == t[7]);
  REQUIRE(res.stats.size() == t[8]);
  int bad = 0;
  for (std::uint64_t i = 0; i < t[3] && i < res.queue.size(); ++i) {
    std::uint64_t m[7], len;
    const std::uint8_t* data;
    lib.campaign_queue_entry(ref, i, m, &data, &len);
    const QueueEntry& e = res.queue[i];
    const bool same = e.id == m[0] && e.full_sig == m[1] && e.simple_sig == m[2] &&
                      static_cast<std::uint64_t>(e.admit_reason) == m[3] && e.discovered_at == m[4] &&
                      (e.parent ? *e.parent : ~0ull) == m[5] && e.exec_cost == m[6] && e.input.size() == len &&
                      (len == 0 || std::memcmp(e.input.data(), data, len) == 0);
    if (!same && bad++ < 3) std::printf("  queue entry %llu differs\n", (unsigned long long)i);
  }
  REQUIRE(bad == 0);
  bad = 0;
  for (std::uint64_t i = 0; i < t[8] && i < res.stats.size(); ++i) {
    std::uint64_t r[7];
    lib.campaign_stats_row(ref, i, r);
    const StatsRow& s = res.stats[i];
    const bool same = s.virtual_time == r[0] && s.execs == r[1] && s.host_edges == r[2] && s.device_edges == r[3] &&
                      s.unique_inputs == r[4] && s.crashes == r[5] && s.sanitizer_execs == r[6];
    if (!same && bad++ < 3) std::printf("  stats row %llu differs\n", (unsigned long long)i);
  }
  REQUIRE(bad == 0);
  std::uint64_t ci = 0;
  for (const auto& kv : res.crashes) {
    if (ci >= t[7]) break;
    std::uint64_t m[4];
    const char* text;
    lib.campaign_crash(ref, ci++, m, &text);
    REQUIRE(kv.first == m[0]);
    REQUIRE(kv.second.first_exposed == m[1]);
    REQUIRE(kv.second.hits == m[2]);
    REQUIRE((kv.second.false_positive ? 1u : 0u) == m[3]);
    REQUIRE(crash_report_text(kv.second) == text);
  }
  std::vector<std::uint8_t> rv(kMapSize);
  lib.campaign_virgin(ref, rv.data());
  REQUIRE(std::memcmp(rv.data(), res.virgin.data(), kMapSize) == 0);
  REQUIRE(plot_data_csv(res.stats) == lib.campaign_csv(ref));
  REQUIRE(campaign_json(cfg, res) == lib.campaign_json(ref));
  if (campaign_json(cfg, res) != lib.campaign_json(ref))
    std::printf("--- ours\n%s--- reference\n%s", campaign_json(cfg, res).c_str(), lib.campaign_json(ref));
  REQUIRE(exec.execs >= res.execs);  // speculation may execute a few extra mutants
  g_splice_cuts += res.splice_cuts;
  g_rollbacks += res.rollbacks;
  lib.campaign_free(ref);
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::printf("usage: campaign_test <libhetfuzz_ref.so> <out_dir> [case index]\n");
    return 2;
  }
  RefLib lib(argv[1]);
  Context ctx(0, kMapSize);
  const Case cases[] = {
      // crashes + sanitizer findings, default strategy, stats every 100 execs
      {"vecadd-offbyone", 1, 2500, Strategy::SimpleTrace, true, false, BudgetKind::Execs, 100, 1},
      // clean target, no sanitizers, sequential queue, odd stats period (folds straddle it)
      {"clean-pipeline", 7, 3000, Strategy::SimpleTrace, false, true, BudgetKind::Execs, 37, 1},
      // every input sanitized, two workers (dispatch order must not change anything)
      {"shared-race", 3, 1200, Strategy::AllTrace, true, false, BudgetKind::Execs, 100, 2},
      // virtual-time budget: the stop falls inside a fold
      {"boxfilter-guardless", 11, 4000000, Strategy::CoverageIncrease, true, false, BudgetKind::VirtualTime, 100, 1},
      // unique-trace strategy on a device-heavy target
      {"seamcarve-nocheck", 5, 1500, Strategy::UniqueTrace, true, false, BudgetKind::Execs, 250, 1},
      // longer runs on the remaining targets: admissions inside splice stages (speculation cut + rollback)
      {"urng-headertrust", 2, 6000, Strategy::SimpleTrace, true, false, BudgetKind::Execs, 100, 1},
      {"uninit-sum", 9, 6000, Strategy::SimpleTrace, false, false, BudgetKind::Execs, 64, 1},
      {"seamcarve-nocheck", 21, 8000, Strategy::SimpleTrace, false, false, BudgetKind::Execs, 100, 1},
      {"boxfilter-guardless", 4, 8000, Strategy::SimpleTrace, false, false, BudgetKind::Execs, 1000, 1},
      {"clean-pipeline", 13, 9000000, Strategy::SimpleTrace, true, false, BudgetKind::VirtualTime, 100, 1},
  };
  const int n_cases = static_cast<int>(sizeof(cases) / sizeof(cases[0]));
  const int only = argc > 3 ? std::atoi(argv[3]) : -1;
  if (only < 0) {  // the Executor contract: a persistent (stateful) campaign is refused, not run inexactly
    struct Dummy : Executor {
      ExecOutcome execute(const Bytes&, CoverageMap&) override { return {}; }
      ShadowOutcome shadow(const Bytes&) override { return {}; }
    } dummy;
    CampaignConfig pc;
    pc.persistent = true;
    bool refused = false;
    try {
      BatchCampaign bc(pc, dummy, ctx);
    } catch (const hetfuzz::InternalError&) {
      refused = true;
    }
    REQUIRE(refused);
  }
  for (int i = 0; i < n_cases; ++i)
    if (only < 0 || only == i) run_case(lib, ctx, cases[i], argv[2], i);
  if (g_fail) {
    std::printf("%d check(s) failed\n", g_fail);
    return 1;
  }
  std::printf("splice cuts %llu, rollbacks %llu over all cases\n", g_splice_cuts, g_rollbacks);
  std::printf("campaign_test: all checks passed\n");
  return 0;
}
