// hetfuzz/engine.hpp -- the mutation part of the reference's engine.hpp
// (proj/include/hetfuzz/engine.hpp:17-35) running on the B200 (K3).
//
// Two ways to use it:
//  * on its own (only this repository's include/ on the include path): hetfuzz::havoc_mutant,
//    splice_mutant, deterministic_mutants and kMaxInputBytes are declared here with the reference's
//    signatures and run on the device;
//  * in front of the reference's tree (-I <this>/include -I <reference>/proj/include): this header
//    steps aside -- #include_next pulls in the reference's own engine.hpp, so src/engine.cpp,
//    python/bindings.cpp and the tests compile unchanged (their coverage types and functions come
//    from this repository's coverage.hpp, i.e. from the GPU) -- and only ADDS the device mutators
//    under hetfuzz::b200:: (the reference defines the hetfuzz:: ones itself in src/engine.cpp;
//    INTEGRATION.md shows the three forwarding lines that swap them).
#pragma once

#include <cstdint>
#include <vector>

#include "b200.hpp"
#include "rng.hpp"

#ifdef HETFUZZ_B200_WITH_REFERENCE
#include_next "hetfuzz/engine.hpp"
#endif

namespace hetfuzz {

#ifndef HETFUZZ_B200_WITH_REFERENCE
inline constexpr std::size_t kMaxInputBytes = 1 << 20;
#endif

namespace b200 {
// One stacked-havoc variant; advances rng exactly like the reference (src/engine.cpp:119-193).
inline std::vector<std::uint8_t> havoc_mutant(const std::vector<std::uint8_t>& input, Rng& rng) {
  const std::uint64_t in_off[2] = {0, input.size()};
  const std::uint64_t cap = hfz_havoc_max_out(input.size());
  const std::uint64_t out_off[2] = {0, cap};
  std::vector<std::uint8_t> out(cap ? cap : 1);
  std::uint64_t state = rng.state(), out_len = 0;
  check(hfz_havoc_batch_host(default_context().get(), input.data(), in_off, 1, &state,
                                   out.data(), out_off, &out_len, nullptr),
              "hfz_havoc_batch_host");
  rng.set_state(state);
  out.resize(out_len);
  return out;
}

// Batched form: slot j mutates inputs[j] with its own stream rngs[j].
inline std::vector<std::vector<std::uint8_t>> havoc_batch(const std::vector<std::vector<std::uint8_t>>& inputs,
                                                          std::vector<Rng>& rngs) {
  const std::uint64_t n = inputs.size();
  std::vector<std::uint64_t> in_off(n + 1, 0), out_off(n + 1, 0), state(n), out_len(n);
  for (std::uint64_t j = 0; j < n; ++j) {
    in_off[j + 1] = in_off[j] + inputs[j].size();
    out_off[j + 1] = out_off[j] + ((hfz_havoc_max_out(inputs[j].size()) + 15) & ~std::uint64_t(15));
    state[j] = rngs[j].state();
  }
  std::vector<std::uint8_t> blob(in_off[n] + 1), out(out_off[n] + 1);
  for (std::uint64_t j = 0; j < n; ++j)
    std::copy(inputs[j].begin(), inputs[j].end(), blob.begin() + in_off[j]);
  check(hfz_havoc_batch_host(default_context().get(), blob.data(), in_off.data(), n, state.data(),
                                   out.data(), out_off.data(), out_len.data(), nullptr),
              "hfz_havoc_batch_host");
  std::vector<std::vector<std::uint8_t>> res(n);
  for (std::uint64_t j = 0; j < n; ++j) {
    res[j].assign(out.begin() + out_off[j], out.begin() + out_off[j] + out_len[j]);
    rngs[j].set_state(state[j]);
  }
  return res;
}

inline std::vector<std::uint8_t> splice_mutant(const std::vector<std::uint8_t>& a,
                                               const std::vector<std::uint8_t>& b, Rng& rng) {
  const std::uint64_t in_off[3] = {0, a.size(), a.size() + b.size()};
  std::vector<std::uint8_t> blob(a);
  blob.insert(blob.end(), b.begin(), b.end());
  blob.push_back(0);
  std::uint64_t cap = a.size() + b.size();
  if (cap > kMaxInputBytes) cap = kMaxInputBytes;
  const std::uint64_t out_off[2] = {0, cap};
  const std::uint32_t ai = 0, bi = 1;
  std::vector<std::uint8_t> out(cap + 1);
  std::uint64_t state = rng.state(), out_len = 0;
  check(hfz_splice_batch_host(default_context().get(), blob.data(), in_off, 2, &ai, &bi, 1, &state,
                                    out.data(), out_off, &out_len),
              "hfz_splice_batch_host");
  rng.set_state(state);
  out.resize(out_len);
  return out;
}

inline std::vector<std::vector<std::uint8_t>> deterministic_mutants(const std::vector<std::uint8_t>& input) {
  const std::uint64_t count = hfz_deterministic_count(input.data(), input.size());
  std::vector<std::uint8_t> flat(count * input.size() + 1);
  check(hfz_deterministic_host(default_context().get(), input.data(), input.size(), flat.data(), count),
              "hfz_deterministic_host");
  std::vector<std::vector<std::uint8_t>> out(count);
  for (std::uint64_t m = 0; m < count; ++m)
    out[m].assign(flat.begin() + m * input.size(), flat.begin() + (m + 1) * input.size());
  return out;
}

}  // namespace b200

#ifndef HETFUZZ_B200_WITH_REFERENCE
using b200::deterministic_mutants;
using b200::havoc_batch;
using b200::havoc_mutant;
using b200::splice_mutant;
#endif

}  // namespace hetfuzz
