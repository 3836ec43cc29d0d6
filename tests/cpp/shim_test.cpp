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
  if (g_fail) {
    std::printf("%d check(s) failed\n", g_fail);
    return 1;
  }
  std::printf("shim_test: all checks passed\n");
  return 0;
}
