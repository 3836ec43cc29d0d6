// The reference's C++ API (namespace hetfuzz) on top of libhfz.so: restated cases of
// proj/tests/test_coverage.cpp and proj/tests/test_engine.cpp, written against include/hetfuzz/.
// Built and run by tests/test_cpp_shim_gpu.py on the GPU box.  Exit code 0 = all checks passed.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

#include "hetfuzz/coverage.hpp"
#include "hetfuzz/engine.hpp"
#include "hetfuzz/rng.hpp"

using namespace hetfuzz;

static int g_fail = 0;
#define REQUIRE(c)                                                \
  do {                                                            \
    if (!(c)) {                                                   \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);  \
      ++g_fail;                                                   \
    }                                                             \
  } while (0)

static std::uint64_t fnv(const std::vector<std::uint8_t>& b) {
  std::uint64_t h = 14695981039346656037ULL;
  for (auto x : b) { h ^= x; h *= 1099511628211ULL; }
  return h;
}

int main() {
  {  // test_coverage.cpp:157-175
    CoverageMap map;
    map.host_increment(10);
    for (int i = 0; i < 5; ++i) map.host_increment(500);
    map.device_store(kDeviceIndexBase + 3, 700);
    map.device_store(kMapSize - 1, 2);
    ClassedTrace t = classify_trace(map);
    std::vector<std::uint32_t> want = {10, 500, kDeviceIndexBase + 3, kMapSize - 1};
    REQUIRE(t.nonzero == want);
    REQUIRE(t.classed[10] == 1 && t.classed[500] == 8 && t.classed[kDeviceIndexBase + 3] == 8 && t.classed[kMapSize - 1] == 2);
  }
  {  // test_coverage.cpp:177-221
    VirginMap virgin;
    auto mk = [](std::initializer_list<std::pair<std::uint32_t, int>> hits) {
      CoverageMap m;
      for (auto& h : hits) for (int i = 0; i < h.second; ++i) m.host_increment(h.first);
      return classify_trace(m);
    };
    ClassedTrace t1 = mk({{42, 1}});
    REQUIRE(has_new_bits(t1, virgin) == Admit::NewEdges);
    REQUIRE(virgin.host_edges() == 1 && virgin.device_edges() == 0);
    REQUIRE(has_new_bits(t1, virgin) == Admit::None);
    REQUIRE(has_new_bits(mk({{42, 2}}), virgin) == Admit::NewCounts);
    REQUIRE(has_new_bits(mk({{42, 4}}), virgin) == Admit::NewCounts);
    REQUIRE(has_new_bits(mk({{42, 5}}), virgin) == Admit::None);
    REQUIRE(has_new_bits(mk({{42, 3}, {43, 1}}), virgin) == Admit::NewEdges);
    REQUIRE(virgin.host_edges() == 2);
    CoverageMap m7;
    m7.device_store(kDeviceIndexBase + 9, 1);
    REQUIRE(has_new_bits(classify_trace(m7), virgin) == Admit::NewEdges);
    REQUIRE(virgin.device_edges() == 1);
    REQUIRE(virgin.at(42) == (1 | 2 | 4 | 8));
  }
  {  // test_coverage.cpp:239-259
    CoverageMap map;
    for (int i = 0; i < 3; ++i) map.host_increment(5);
    map.device_store(40000, 700);
    ClassedTrace t = classify_trace(map);
    REQUIRE(trace_signature(t, SignatureMode::Simple) == fnv({5, 0, 40000 & 0xff, 40000 >> 8}));
    REQUIRE(trace_signature(t, SignatureMode::Full) == fnv({5, 0, 4, 40000 & 0xff, 40000 >> 8, 8}));
    CoverageMap empty;
    REQUIRE(trace_signature(classify_trace(empty), SignatureMode::Simple) == 14695981039346656037ULL);
  }
  {  // rng + mutators: test_engine.cpp:128-169 and the survey's known answers
    Rng a(99), b(99);
    for (int i = 0; i < 100; ++i) REQUIRE(a.next() == b.next());
    std::vector<std::uint8_t> base(16);
    for (int i = 0; i < 16; ++i) base[i] = static_cast<std::uint8_t>(i);
    Rng r1(1);
    std::vector<std::uint8_t> h = havoc_mutant(base, r1);
    const std::uint8_t want[] = {0xbc, 0xff, 0xbc, 0xbc, 0x00, 0x03, 0x01};
    REQUIRE(h == std::vector<std::uint8_t>(want, want + 7));
    Rng r1b(1);
    r1b.jump(117);
    REQUIRE(r1.state() == r1b.state());  // 117 draws consumed
    Rng r7(7), r8(8);
    std::vector<std::uint8_t> z(64, 0);
    REQUIRE(havoc_mutant(z, r7) != havoc_mutant(z, r8));
    Rng r3(3);
    REQUIRE(!havoc_mutant({}, r3).empty());
    Rng rs(7);
    std::vector<std::uint8_t> A(8, 'A'), B(8, 'B');
    std::vector<std::uint8_t> s = splice_mutant(A, B, rs);
    REQUIRE(std::string(s.begin(), s.end()) == "AAABBBBBBBB");
    auto det = deterministic_mutants(std::vector<std::uint8_t>(8, 0));
    REQUIRE(det.size() == 1638);
    REQUIRE(det[0][0] == 0x80 && det[1][0] == 0x40 && det[64][0] == 1 && det[65][0] == 0xff);
    std::vector<Rng> rr = {Rng(1), Rng(2)};
    auto hb = havoc_batch({base, base}, rr);
    REQUIRE(hb[0] == h && hb[1].size() == 32);
  }
  {  // sparse host form: SparseBatch of CoverageMaps == the dense records of the same maps
    Rng rng(0x5151);
    const int n = 200;
    std::vector<CoverageMap> maps(n);
    std::vector<std::uint8_t> raw(std::size_t(n) * kHostSlots * 5);
    b200::SparseBatch batch;
    b200::CompactBatch cbatch;
    for (int e = 0; e < n; ++e) {
      const int hits = e == 7 ? 0 : 200 + int(rng.below(800));  // exec 7 touches nothing
      for (int i = 0; i < hits; ++i) {
        if (rng.chance(1, 2)) {
          const std::uint32_t idx = std::uint32_t(rng.below(64) * 97 + rng.below(3)) % kHostSlots;
          const int reps = 1 + int(rng.below(300));  // wraps past 255 now and then
          for (int k = 0; k < reps; ++k) maps[e].host_increment(idx);
        } else {
          const std::uint32_t idx = kDeviceIndexBase + std::uint32_t(rng.below(64) * 131 + rng.below(3)) % kHostSlots;
          maps[e].device_store(idx, std::uint32_t(rng.below(3) == 0 ? 0 : 1 + rng.below(100000)));
        }
      }
      maps[e].pack(&raw[std::size_t(e) * kHostSlots * 5]);
      batch.append(maps[e]);
      cbatch.append(maps[e]);
    }
    REQUIRE(batch.size() == std::uint64_t(n));
    VirginMap va, vb;
    b200::FeedbackResult a = b200::feedback_batch(b200::default_context(), raw.data(), n, va.data(), va.edge_counts(), true);
    b200::FeedbackResult b = b200::feedback_batch(b200::default_context(), batch, vb.data(), vb.edge_counts(), true);
    REQUIRE(a.admit == b.admit);
    REQUIRE(a.sig_full == b.sig_full);
    REQUIRE(a.sig_simple == b.sig_simple);
    REQUIRE(a.nnz == b.nnz);
    REQUIRE(a.classed == b.classed);
    REQUIRE(a.nnz[7] == 0 && a.sig_full[7] == 14695981039346656037ULL);
    VirginMap vc;
    b200::FeedbackResult cc = b200::feedback_batch(b200::default_context(), cbatch, vc.data(), vc.edge_counts(), true);
    REQUIRE(a.admit == cc.admit && a.sig_full == cc.sig_full && a.sig_simple == cc.sig_simple);
    REQUIRE(a.nnz == cc.nnz && a.classed == cc.classed);
    REQUIRE(va.host_edges() == vc.host_edges() && va.device_edges() == vc.device_edges());
    REQUIRE(va.host_edges() == vb.host_edges() && va.device_edges() == vb.device_edges());
    bool same = true;
    for (std::uint32_t i = 0; i < kMapSize; ++i) same = same && va.at(i) == vb.at(i);
    REQUIRE(same);
    REQUIRE(va.host_edges() > 0 && va.device_edges() > 0);
    // the packed form (3-byte host entries, 17-bit device counts): the same results again
    b200::PackedBatch pbatch;
    for (int e = 0; e < n; ++e) pbatch.append(maps[e]);
    VirginMap vp;
    b200::FeedbackResult pp = b200::feedback_batch(b200::default_context(), pbatch, vp.data(), vp.edge_counts(), true);
    REQUIRE(a.admit == pp.admit && a.sig_full == pp.sig_full && a.sig_simple == pp.sig_simple && a.nnz == pp.nnz);
    REQUIRE(a.classed == pp.classed);
    REQUIRE(va.host_edges() == vp.host_edges() && va.device_edges() == vp.device_edges());
    {  // the same execs as three packed batches (one of them empty) folded by ONE call
      b200::PackedBatch p0, p1, p2, p3;
      for (int e = 0; e < n; ++e) (e < 70 ? p0 : (e < 71 ? p2 : p3)).append(maps[e]);
      VirginMap vq;
      b200::FeedbackResult qq = b200::feedback_batch(b200::default_context(), {&p0, &p1, &p2, &p3}, vq.data(), vq.edge_counts());
      REQUIRE(a.admit == qq.admit && a.sig_full == qq.sig_full && a.sig_simple == qq.sig_simple && a.nnz == qq.nnz);
      REQUIRE(va.host_edges() == vq.host_edges() && va.device_edges() == vq.device_edges());
      bool same_v = true;
      for (std::uint32_t i = 0; i < kMapSize; ++i) same_v = same_v && va.at(i) == vq.at(i);
      REQUIRE(same_v);
    }
    // take() = append() + reset() in one walk: the same batch, and the maps end up all-zero and reusable
    b200::CompactBatch tbatch;
    for (int e = 0; e < n; ++e) tbatch.take(maps[e]);
    VirginMap vd;
    b200::FeedbackResult dd = b200::feedback_batch(b200::default_context(), tbatch, vd.data(), vd.edge_counts(), true);
    REQUIRE(a.admit == dd.admit && a.sig_full == dd.sig_full && a.sig_simple == dd.sig_simple && a.nnz == dd.nnz);
    REQUIRE(va.host_edges() == vd.host_edges() && va.device_edges() == vd.device_edges());
    bool zero = true;
    for (int e = 0; e < n; ++e) {
      zero = zero && maps[e].touched().empty();
      for (std::uint32_t i = 0; i < kHostSlots && zero; ++i) zero = maps[e].host_at(i) == 0 && maps[e].device_at(kDeviceIndexBase + i) == 0;
    }
    REQUIRE(zero);
  }
  if (g_fail) {
    std::printf("%d check(s) failed\n", g_fail);
    return 1;
  }
  std::printf("shim_test: all checks passed\n");
  return 0;
}
