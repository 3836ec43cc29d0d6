// hetfuzz/rng.hpp -- the reference's Rng (proj/include/hetfuzz/rng.hpp:11-46) as a thin value
// type over the C-ABI's scalar splitmix64 helpers.  Same member names and meaning; two
// additions make the O(1) jump-ahead of the batched mutators visible: state() and jump().
#pragma once

#include <cstdint>

#include "../hfz.h"

namespace hetfuzz {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : s_(seed) {}

  std::uint64_t next() { return hfz_rng_next(&s_); }
  // [0, n); n <= 1 yields 0 and consumes no draw
  std::uint64_t below(std::uint64_t n) { return hfz_rng_below(&s_, n); }
  // [lo, hi]
  std::uint64_t between(std::uint64_t lo, std::uint64_t hi) { return lo + below(hi - lo + 1); }
  bool chance(std::uint64_t num, std::uint64_t den) { return below(den) < num; }
  // independent child stream; advances this stream by one draw
  Rng split(std::uint64_t tag) { return Rng(hfz_rng_split(&s_, tag)); }

  // --- additions
  std::uint64_t state() const { return s_; }
  void set_state(std::uint64_t s) { s_ = s; }
  void jump(std::uint64_t draws) { s_ = hfz_rng_jump(s_, draws); }

 private:
  std::uint64_t s_;
};

}  // namespace hetfuzz
