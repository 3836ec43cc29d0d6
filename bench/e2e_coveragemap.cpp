// bench/e2e_coveragemap.cpp -- end to end FROM THE REFERENCE'S OWN HOST TYPE.
//
// What a host loop written against the reference holds after an execution is a hetfuzz::CoverageMap
// (Campaign::run_one, src/engine.cpp:464-471).  This harness builds N of them from the synthetic
// campaign recipe (the same one bench.py uses, paper_2603_12485_b200/synth.py::maps_campaign) and times,
// as ONE region per step:
//     PackedBatch::append(map) x N   (touched-slot lists into pinned memory, 3 / 4 bytes per slot; 1 or T host threads)
//   + feedback_batch(ctx, batch, virgin, counts)   (H2D, rank + chain + resolve kernels, D2H)
//   + the results back in host vectors
// and, in the same process, the reference's own loop over the SAME maps -- classify_trace, both
// trace_signature calls, has_new_bits, exactly src/engine.cpp:471-478 -- on one host thread (the
// reference campaign is single-threaded), through the unmodified reference build
// oracle/_ref/libhetfuzz_ref.so (dlopen).  Every output of the two is compared: Admit codes in order,
// both signatures, nnz, the final virgin map and both edge counters.
//
// A third leg, "streaming", is how a fuzzing loop actually meets the call: every worker thread owns ONE
// CoverageMap, and after each execution (here: fill_map, untimed in every leg) it appends the still
// cache-hot map to its batch and resets it for the next execution (PackedBatch::take).  Timed: the take calls
// (summed per worker, maximum over workers) + the fold + the results back in host vectors.
//
// Prints one JSON object.  Test/bench infrastructure: the oracle is used as the checker and as the
// timed CPU leg, never by the product path.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hetfuzz/coverage.hpp"

using namespace hetfuzz;
using Batch = b200::PackedBatch;  // the densest host form (3 / 4 bytes per touched slot)
using b200::Context;
using b200::FeedbackResult;

namespace {

constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;
inline std::uint64_t sm64(std::uint64_t seed, std::uint64_t k) {  // k-th output of splitmix64(seed), synth.py::sm64
  std::uint64_t z = seed + (k + 1) * kGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline std::uint64_t below32(std::uint64_t x, std::uint64_t n) { return ((x >> 32) * n) >> 32; }

const std::uint32_t kHostTable[8] = {1, 2, 3, 5, 9, 20, 40, 200};
const std::uint32_t kDevTable[7] = {1, 2, 100, 600, 5000, 20000, 70000};

struct Program {  // the fixed "program" of synth.maps_campaign: slots E and their favourite rungs
  std::vector<std::uint32_t> E, fav;
  explicit Program(std::uint64_t seed) {
    const std::uint32_t nE = 1311;  // round(0.02 * 65536)
    E.resize(nE);
    fav.resize(nE);
    for (std::uint32_t j = 0; j < nE; ++j) {
      E[j] = static_cast<std::uint32_t>(below32(sm64(seed, 2ull * j), kMapSize));
      fav[j] = static_cast<std::uint32_t>(below32(sm64(seed, 2ull * j + 1), 7));
    }
  }
};

// one execution's map, exactly synth.maps_campaign(seed=43, p_extra=256, p_rare=512) for exec index e
void fill_map(const Program& pr, std::uint64_t seed, std::uint64_t e, CoverageMap& m) {
  const std::uint32_t nE = static_cast<std::uint32_t>(pr.E.size());
  const std::uint64_t es = sm64(seed ^ 0xD1B54A32D192ED03ull, e);
  std::uint64_t dx[4];
  for (int k = 0; k < 4; ++k) dx[k] = sm64(es, nE + k);
  const bool rare_on = below32(dx[0], 512) == 0;
  const std::uint32_t rare_j = static_cast<std::uint32_t>(below32(dx[1], nE));
  for (std::uint32_t j = 0; j < nE; ++j) {
    const bool is_host = pr.E[j] < kHostSlots;
    const std::uint32_t ntab = is_host ? 8 : 7;
    bool hit = below32(sm64(es, j), 10) < 9;
    const bool alt = below32(sm64(es ^ 0xA17ull, j), 100) >= 97;
    std::uint32_t rung = alt ? (pr.fav[j] + 1) % ntab : pr.fav[j];
    if (rare_on && j == rare_j) {
      rung = (pr.fav[j] + 3) % ntab;
      hit = true;
    }
    if (!hit) continue;
    if (is_host)
      m.host_assign(pr.E[j], static_cast<std::uint8_t>(kHostTable[rung]));
    else
      m.device_store(pr.E[j], kDevTable[rung]);
  }
  if (below32(dx[2], 256) == 0) {
    const std::uint32_t s = static_cast<std::uint32_t>(below32(dx[3], kMapSize));
    if (m.count_at(s) == 0) {
      if (s < kHostSlots) m.host_assign(s, 1); else m.device_store(s, 1);
    }
  }
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct RefLib {  // the unmodified reference (oracle/_ref/libhetfuzz_ref.so): checker + timed CPU leg
  void* h = nullptr;
  void* (*maps_create)(const std::uint8_t*, std::uint64_t) = nullptr;
  void (*maps_free)(void*) = nullptr;
  int (*feedback_run)(void*, std::uint64_t, std::uint64_t, std::uint8_t*, std::uint64_t*, std::uint8_t*, std::uint8_t*,
                      std::uint64_t*, std::uint64_t*, std::uint32_t*) = nullptr;
  bool open(const std::string& path) {
    h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!h) return false;
    maps_create = reinterpret_cast<decltype(maps_create)>(dlsym(h, "ref_maps_create"));
    maps_free = reinterpret_cast<decltype(maps_free)>(dlsym(h, "ref_maps_free"));
    feedback_run = reinterpret_cast<decltype(feedback_run)>(dlsym(h, "ref_feedback_run"));
    return maps_create && maps_free && feedback_run;
  }
};

std::uint64_t fnv_bytes(const std::uint8_t* p, std::size_t n) {
  std::uint64_t h = kFnvOffset;
  for (std::size_t i = 0; i < n; ++i) h = (h ^ p[i]) * kFnvPrime;
  return h;
}

}  // namespace

int main(int argc, char** argv) {
  std::uint64_t n = 65536, steps = 5, warm = 4096;
  unsigned threads = std::max(1u, std::thread::hardware_concurrency());
  bool gen_only = false;
  std::string ref_path;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() { return i + 1 < argc ? argv[++i] : "0"; };
    if (a == "--execs") n = std::strtoull(val(), nullptr, 10);
    else if (a == "--steps") steps = std::strtoull(val(), nullptr, 10);
    else if (a == "--threads") threads = static_cast<unsigned>(std::strtoul(val(), nullptr, 10));
    else if (a == "--ref") ref_path = val();
    else if (a == "--gen-only") gen_only = true;   // print the checksum of the first 8 generated records and exit (no GPU)
  }
  if (ref_path.empty()) {
    std::string self = argv[0];
    const std::size_t slash = self.find_last_of('/');
    ref_path = (slash == std::string::npos ? std::string(".") : self.substr(0, slash)) + "/../oracle/_ref/libhetfuzz_ref.so";
  }
  const std::uint64_t seed = 43, rec = std::uint64_t(kHostSlots) * 5;
  const Program prog(seed);
  if (gen_only) {
    std::vector<std::uint8_t> recs(8 * rec);
    for (std::uint64_t e = 0; e < 8; ++e) {
      CoverageMap m;
      fill_map(prog, seed, e, m);
      m.pack(recs.data() + e * rec);
    }
    std::printf("{\"first8_fnv\": \"%016llx\"}\n", static_cast<unsigned long long>(fnv_bytes(recs.data(), recs.size())));
    return 0;
  }

  // ---- data: N CoverageMap objects (as the reference arm builds them before its timed region)
  const double t_gen0 = now();
  std::vector<CoverageMap> maps(n), warm_maps(warm);
  {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < threads; ++t)
      th.emplace_back([&, t] {
        for (std::uint64_t e = t; e < n; e += threads) fill_map(prog, seed, e, maps[e]);
        for (std::uint64_t e = t; e < warm; e += threads) fill_map(prog, seed, (1ull << 24) + e, warm_maps[e]);
      });
    for (auto& x : th) x.join();
  }
  const double gen_s = now() - t_gen0;

  Context ctx(0, kMapSize);
  VirginMap v0;
  {
    Batch wb;
    for (const CoverageMap& m : warm_maps) wb.append(m);
    b200::feedback_batch(ctx, wb, v0.data(), v0.edge_counts());
  }

  // ---- GPU leg: pack (1 thread, then T threads) + fold + results, one timed region per step
  auto run_gpu = [&](unsigned pack_threads, std::vector<double>& total, std::vector<double>& pack, FeedbackResult& last,
                     VirginMap& v_out) {
    const unsigned T = std::max(1u, pack_threads);
    std::vector<Batch> batches(T);
    for (std::uint64_t s = 0; s <= steps; ++s) {  // step 0 is the warm-up (pinned buffers grow once)
      VirginMap v = v0;
      FeedbackResult all;
      all.admit.resize(n);
      all.sig_full.resize(n);
      all.sig_simple.resize(n);
      all.nnz.resize(n);
      const double t0 = now();
      if (T == 1) {
        batches[0].clear();
        for (std::uint64_t e = 0; e < n; ++e) batches[0].append(maps[e]);
      } else {  // worker t packs the contiguous exec range [t*n/T, (t+1)*n/T): folds stay in exec order
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t)
          th.emplace_back([&, t] {
            batches[t].clear();
            for (std::uint64_t e = n * t / T; e < n * (t + 1) / T; ++e) batches[t].append(maps[e]);
          });
        for (auto& x : th) x.join();
      }
      const double t1 = now();
      {  // the workers' batches in exec order, ONE device call (batch k + 1 crosses PCIe under the fold of batch k)
        std::vector<const std::uint8_t*> h3;
        std::vector<const std::uint64_t*> hoff, doff;
        std::vector<const std::uint32_t*> d17;
        std::vector<std::uint64_t> cnts;
        for (unsigned t = 0; t < T; ++t) {
          h3.push_back(batches[t].host3());
          hoff.push_back(batches[t].host3_offsets());
          d17.push_back(batches[t].dev17());
          doff.push_back(batches[t].dev17_offsets());
          cnts.push_back(batches[t].size());
        }
        b200::check(hfz_feedback_batch_packed_host_v(ctx.get(), T, h3.data(), hoff.data(), d17.data(), doff.data(), cnts.data(),
                                                     v.data(), v.edge_counts(), all.admit.data(), all.sig_full.data(),
                                                     all.sig_simple.data(), all.nnz.data()),
                    "hfz_feedback_batch_packed_host_v");
      }
      const double t2 = now();
      if (s) {
        total.push_back(t2 - t0);
        pack.push_back(t1 - t0);
      }
      last = std::move(all);
      v_out = v;
    }
  };
  std::vector<double> tot1, pack1, totT, packT;
  FeedbackResult r1, rT;
  VirginMap v1, vT;
  run_gpu(1, tot1, pack1, r1, v1);
  run_gpu(threads, totT, packT, rT, vT);

  // ---- streaming leg: one reused map per worker, appended right after the execution that filled it
  std::vector<double> totS, packS;
  FeedbackResult rS;
  VirginMap vS;
  {
    const unsigned T = threads;
    std::vector<Batch> batches(T);
    for (std::uint64_t s = 0; s <= steps; ++s) {
      VirginMap v = v0;
      FeedbackResult all;
      all.admit.resize(n);
      all.sig_full.resize(n);
      all.sig_simple.resize(n);
      all.nnz.resize(n);
      std::vector<double> worker_s(T, 0.0);
      std::vector<std::thread> th;
      for (unsigned t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          CoverageMap m;  // this worker's map, as a fuzzing loop would hold it
          batches[t].clear();
          double acc = 0;
          for (std::uint64_t e = n * t / T; e < n * (t + 1) / T; ++e) {
            fill_map(prog, seed, e, m);  // the execution (untimed, as in the other legs)
            const double a0 = now();
            batches[t].take(m);  // append + reset in one walk
            acc += now() - a0;
          }
          worker_s[t] = acc;
        });
      for (auto& x : th) x.join();
      const double pack_s = *std::max_element(worker_s.begin(), worker_s.end());
      const double t1 = now();
      {  // the workers' batches in exec order, ONE device call (batch k + 1 crosses PCIe under the fold of batch k)
        std::vector<const std::uint8_t*> h3;
        std::vector<const std::uint64_t*> hoff, doff;
        std::vector<const std::uint32_t*> d17;
        std::vector<std::uint64_t> cnts;
        for (unsigned t = 0; t < T; ++t) {
          h3.push_back(batches[t].host3());
          hoff.push_back(batches[t].host3_offsets());
          d17.push_back(batches[t].dev17());
          doff.push_back(batches[t].dev17_offsets());
          cnts.push_back(batches[t].size());
        }
        b200::check(hfz_feedback_batch_packed_host_v(ctx.get(), T, h3.data(), hoff.data(), d17.data(), doff.data(), cnts.data(),
                                                     v.data(), v.edge_counts(), all.admit.data(), all.sig_full.data(),
                                                     all.sig_simple.data(), all.nnz.data()),
                    "hfz_feedback_batch_packed_host_v");
      }
      const double fold_s = now() - t1;
      if (s) {
        totS.push_back(pack_s + fold_s);
        packS.push_back(pack_s);
      }
      rS = std::move(all);
      vS = v;
    }
  }

  // ---- reference leg: engine.cpp:471-478 over the same maps, one thread, in chunks of 2,048 maps
  RefLib ref;
  double ref_s = -1;
  bool equal = false, have_ref = ref.open(ref_path);
  if (have_ref) {
    std::vector<std::uint8_t> ref_v(kMapSize, 0);
    std::uint64_t ref_c[2] = {0, 0};
    {
      std::vector<std::uint8_t> recs(warm * rec);
      for (std::uint64_t e = 0; e < warm; ++e) warm_maps[e].pack(recs.data() + e * rec);
      void* h = ref.maps_create(recs.data(), warm);
      ref.feedback_run(h, 0, warm, ref_v.data(), ref_c, nullptr, nullptr, nullptr, nullptr, nullptr);
      ref.maps_free(h);
    }
    equal = std::memcmp(ref_v.data(), v0.data(), kMapSize) == 0 && ref_c[0] == v0.host_edges() && ref_c[1] == v0.device_edges();
    std::vector<std::uint8_t> adm(n);
    std::vector<std::uint64_t> sf(n), ss(n);
    std::vector<std::uint32_t> nz(n);
    const std::uint64_t chunk = 2048;
    std::vector<std::uint8_t> recs(chunk * rec);
    ref_s = 0;
    for (std::uint64_t e0 = 0; e0 < n; e0 += chunk) {
      const std::uint64_t m = std::min(chunk, n - e0);
      for (std::uint64_t e = 0; e < m; ++e) maps[e0 + e].pack(recs.data() + e * rec);
      void* h = ref.maps_create(recs.data(), m);  // the reference's CoverageMap objects: outside its timed region
      const double t0 = now();
      ref.feedback_run(h, 0, m, ref_v.data(), ref_c, nullptr, adm.data() + e0, sf.data() + e0, ss.data() + e0, nz.data() + e0);
      ref_s += now() - t0;
      ref.maps_free(h);
    }
    for (const FeedbackResult* r : {&r1, &rT, &rS})
      equal = equal && r->admit == adm && r->sig_full == sf && r->sig_simple == ss && r->nnz == nz;
    for (VirginMap* v : {&v1, &vT, &vS})
      equal = equal && std::memcmp(ref_v.data(), v->data(), kMapSize) == 0 && ref_c[0] == v->host_edges() &&
              ref_c[1] == v->device_edges();
  }

  auto stats = [](std::vector<double> v, double& mn, double& med, double& mean) {
    std::sort(v.begin(), v.end());
    mn = v.front();
    med = v[v.size() / 2];
    mean = 0;
    for (double x : v) mean += x;
    mean /= v.size();
  };
  double mn1, med1, mean1, pmn1, pmed1, pmean1, mnT, medT, meanT, pmnT, pmedT, pmeanT, mnS, medS, meanS, pmnS, pmedS, pmeanS;
  stats(tot1, mn1, med1, mean1);
  stats(pack1, pmn1, pmed1, pmean1);
  stats(totT, mnT, medT, meanT);
  stats(packT, pmnT, pmedT, pmeanT);
  stats(totS, mnS, medS, meanS);
  stats(packS, pmnS, pmedS, pmeanS);
  std::uint64_t pairs = 0;
  for (const CoverageMap& m : maps) pairs += m.touched().size();
  std::printf(
      "{\"api\": \"hetfuzz::CoverageMap -> b200::PackedBatch::append x N (one batch per packing thread) -> hfz_feedback_batch_packed_host_v (one call) -> host vectors\", "
      "\"execs\": %llu, \"steps\": %llu, \"touched_slots_per_exec\": %.1f, \"gen_seconds\": %.2f, "
      "\"value\": %.1f, \"unit\": \"evals/s\", \"pack_threads\": %u, "
      "\"seconds\": {\"mean\": %.6f, \"median\": %.6f, \"min\": %.6f, \"pack_mean\": %.6f, \"fold_and_readback_mean\": %.6f}, "
      "\"one_pack_thread\": {\"value\": %.1f, \"unit\": \"evals/s\", \"seconds\": {\"mean\": %.6f, \"median\": %.6f, \"min\": %.6f, "
      "\"pack_mean\": %.6f, \"fold_and_readback_mean\": %.6f}}, "
      "\"streaming\": {\"value\": %.1f, \"unit\": \"evals/s\", \"pack_threads\": %u, \"seconds\": {\"mean\": %.6f, \"median\": %.6f, "
      "\"min\": %.6f, \"pack_mean\": %.6f, \"fold_and_readback_mean\": %.6f}, \"what\": \"one reused CoverageMap per worker: PackedBatch::take (append + reset in one walk) right "
      "after the execution that filled it (cache-hot map); timed = take summed per worker, max over workers, + fold + results\"}, "
      "\"reference_same_maps\": {\"available\": %s, \"threads\": 1, \"seconds\": %.4f, \"value\": %.1f, \"unit\": \"evals/s\", "
      "\"what\": \"classify_trace + 2 x trace_signature + has_new_bits per map (src/engine.cpp:471-478), unmodified reference build, same process\"}, "
      "\"equals_reference\": %s, \"compared\": \"all execs: Admit codes in order, both signatures, nnz; final virgin map; both edge counters; "
      "for the 1-thread, the T-thread and the streaming packing\"}\n",
      (unsigned long long)n, (unsigned long long)steps, double(pairs) / double(n), gen_s, double(n) / meanT, threads, meanT, medT, mnT,
      pmeanT, meanT - pmeanT, double(n) / mean1, mean1, med1, mn1, pmean1, mean1 - pmean1, double(n) / meanS, threads, meanS, medS,
      mnS, pmeanS, meanS - pmeanS, have_ref ? "true" : "false", ref_s,
      ref_s > 0 ? double(n) / ref_s : 0.0, have_ref ? (equal ? "true" : "false") : "null");
  return have_ref && !equal ? 1 : 0;
}
