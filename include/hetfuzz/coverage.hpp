// hetfuzz/coverage.hpp -- source-compatible stand-in for the reference header of the same name
// (proj/include/hetfuzz/coverage.hpp) whose data-parallel functions run on the B200:
//   classify_trace / has_new_bits / trace_signature  -> K2 (hfz_feedback_batch_host)
// The containers are plain host value types like the reference's; each single-item call is a
// batch-of-one device call (latency-bound, kept for API parity) -- fuzzers should use
// hetfuzz::b200::feedback_batch.  Header-only; link with libhfz.so.  No CPU implementation of
// the classify / novelty / signature path exists here.
#pragma once

#include <cstddef>
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "b200.hpp"

namespace hetfuzz {

inline constexpr std::uint32_t kMapSize = 65536;
inline constexpr std::uint32_t kHostSlots = kMapSize / 2;
inline constexpr std::uint32_t kDeviceIndexBase = kHostSlots;

// One execution's raw map: u8 never-zero host counters + u32 device warp counters.
class CoverageMap {
 public:
  CoverageMap() : host_(kHostSlots, 0), device_(kMapSize - kHostSlots, 0) {}

  void host_increment(std::uint32_t idx) {
    if (idx >= kHostSlots) {  // audited, then folded into the host half
      ++host_violations_;
      idx &= kHostSlots - 1;
    }
    if (host_[idx] == 0) touched_.push_back(idx);
    const std::uint8_t next = static_cast<std::uint8_t>(host_[idx] + 1);
    host_[idx] = next == 0 ? 1 : next;  // a wrap never reads as "unvisited"
  }
  void device_store(std::uint32_t logical_idx, std::uint32_t count) {
    if (logical_idx < kDeviceIndexBase || logical_idx >= kMapSize) {
      ++device_violations_;
      logical_idx = kDeviceIndexBase + logical_idx % (kMapSize - kHostSlots);
    }
    std::uint32_t& d = device_[logical_idx - kDeviceIndexBase];
    if (d == 0 && count != 0) touched_.push_back(logical_idx);
    d = count;
  }
  std::uint8_t host_at(std::uint32_t idx) const { return host_[idx]; }
  std::uint32_t device_at(std::uint32_t logical_idx) const { return device_[logical_idx - kDeviceIndexBase]; }
  std::uint64_t count_at(std::uint32_t logical_idx) const {
    return logical_idx < kHostSlots ? host_[logical_idx] : device_[logical_idx - kDeviceIndexBase];
  }
  const std::vector<std::uint8_t>& host_half() const { return host_; }
  const std::vector<std::uint32_t>& device_half() const { return device_; }
  std::uint64_t host_partition_violations() const { return host_violations_; }
  std::uint64_t device_partition_violations() const { return device_violations_; }

  // --- additions for batched hosts
  // Back to the all-zero map in O(touched slots): the reference's runtime resets its device
  // counters the same way (reset_device_coverage, src/hdvm.cpp:356-360).
  void reset() {
    for (std::uint32_t s : touched_) {
      if (s < kHostSlots) host_[s] = 0; else device_[s - kDeviceIndexBase] = 0;
    }
    touched_.clear();
    host_violations_ = device_violations_ = 0;
  }
  // reset() that hands every touched slot's count to f(slot, count) on the way: one visit of each counter's
  // cache line instead of two (b200::CompactBatch::take).
  template <class F>
  void drain(F&& f) {
    for (std::uint32_t s : touched_) {
      if (s < kHostSlots) {
        f(s, static_cast<std::uint32_t>(host_[s]));
        host_[s] = 0;
      } else {
        f(s, device_[s - kDeviceIndexBase]);
        device_[s - kDeviceIndexBase] = 0;
      }
    }
    touched_.clear();
    host_violations_ = device_violations_ = 0;
  }
  // Sets a host counter to a final value (importing a map recorded elsewhere).
  void host_assign(std::uint32_t idx, std::uint8_t value) {
    if (host_[idx] == 0 && value != 0) touched_.push_back(idx);
    host_[idx] = value;
  }
  // Logical slots in first-touch order: the dirty list the reference's runtime keeps beside its
  // device counters (src/hdvm.cpp:356-366), here for both halves.  Feeds b200::SparseBatch.
  const std::vector<std::uint32_t>& touched() const { return touched_; }

  // raw record in the library's layout: [host u8 x H][device u32 x H]
  void pack(std::uint8_t* rec) const {
    std::memcpy(rec, host_.data(), kHostSlots);
    std::memcpy(rec + kHostSlots, device_.data(), std::size_t(kMapSize - kHostSlots) * 4);
  }

 private:
  std::vector<std::uint8_t> host_;
  std::vector<std::uint32_t> device_;
  std::vector<std::uint32_t> touched_;
  std::uint64_t host_violations_ = 0, device_violations_ = 0;
};

namespace b200 {

namespace detail {
// growable array in page-locked host memory (hfz_host_alloc): full PCIe speed for the H2D stream
template <class T>
class PinnedVec {
 public:
  PinnedVec() = default;
  PinnedVec(const PinnedVec&) = delete;
  PinnedVec& operator=(const PinnedVec&) = delete;
  ~PinnedVec() { hfz_host_free(buf_); }
  void push_back(T v) {
    if (n_ == cap_) reserve(n_ + 1);
    buf_[n_++] = v;
  }
  void reserve(std::uint64_t want) {
    if (want <= cap_) return;
    std::uint64_t ncap = cap_ ? cap_ : 4096;
    while (ncap < want) ncap *= 2;
    void* nb = nullptr;
    check(hfz_host_alloc(&nb, ncap * sizeof(T)), "hfz_host_alloc");
    if (n_) std::memcpy(nb, buf_, n_ * sizeof(T));
    hfz_host_free(buf_);
    buf_ = static_cast<T*>(nb);
    cap_ = ncap;
  }
  void clear() { n_ = 0; }
  std::uint64_t size() const { return n_; }
  const T* data() const { return buf_; }
  T* data() { return buf_; }
  // unchecked tail writes after a reserve(): tail()[0 .. k) then advance(k)
  T* tail() { return buf_ + n_; }
  void advance(std::uint64_t k) { n_ += k; }

 private:
  T* buf_ = nullptr;
  std::uint64_t cap_ = 0, n_ = 0;
};
}  // namespace detail

// A batch of executions in the sparse host form of include/hfz.h: per exec the (slot, count)
// pairs of the slots its CoverageMap touched, packed back to back in page-locked memory.
// append() right after an execution costs one ~10 KB copy while the map is still cache-hot;
// the batch then crosses PCIe at ~10 KB per exec instead of 163,840 B.
class SparseBatch {
 public:
  SparseBatch() { off_.push_back(0); }
  void append(const CoverageMap& m) {
    const std::vector<std::uint32_t>& t = m.touched();
    pairs_.reserve(pairs_.size() + 2 * t.size());
    for (std::uint32_t slot : t) {
      pairs_.push_back(slot);
      pairs_.push_back(static_cast<std::uint32_t>(m.count_at(slot)));
    }
    off_.push_back(pairs_.size() / 2);
  }
  void clear() {
    pairs_.clear();
    off_.clear();
    off_.push_back(0);
  }
  std::uint64_t size() const { return off_.size() - 1; }
  std::uint64_t pairs() const { return pairs_.size() / 2; }
  const std::uint32_t* entries() const { return pairs_.data(); }
  const std::uint64_t* offsets() const { return off_.data(); }

 private:
  detail::PinnedVec<std::uint32_t> pairs_;
  detail::PinnedVec<std::uint64_t> off_;
};

// The same batch at four bytes per pair (include/hfz.h, hfz_feedback_batch_compact_host): counts
// below 65,536 go into `slot | count << 16` words, the rare larger device counters into wide
// {slot, count} pairs.  kMapSize = 65,536 slots fit the 16-bit slot field exactly.
class CompactBatch {
 public:
  CompactBatch() {
    coff_.push_back(0);
    woff_.push_back(0);
  }
  void append(const CoverageMap& m) {
    for (std::uint32_t slot : m.touched()) {
      const std::uint32_t c = static_cast<std::uint32_t>(m.count_at(slot));
      if (c < 65536u) {
        compact_.push_back(slot | (c << 16));
      } else {
        wide_.push_back(slot);
        wide_.push_back(c);
      }
    }
    coff_.push_back(compact_.size());
    woff_.push_back(wide_.size() / 2);
  }
  // append(m) + m.reset() in one walk: what a fuzzing loop does with its one map after every execution
  void take(CoverageMap& m) {
    m.drain([this](std::uint32_t slot, std::uint32_t c) {
      if (c < 65536u) {
        compact_.push_back(slot | (c << 16));
      } else {
        wide_.push_back(slot);
        wide_.push_back(c);
      }
    });
    coff_.push_back(compact_.size());
    woff_.push_back(wide_.size() / 2);
  }
  void clear() {
    compact_.clear();
    wide_.clear();
    coff_.clear();
    woff_.clear();
    coff_.push_back(0);
    woff_.push_back(0);
  }
  std::uint64_t size() const { return coff_.size() - 1; }
  const std::uint32_t* compact() const { return compact_.data(); }
  const std::uint64_t* compact_offsets() const { return coff_.data(); }
  const std::uint32_t* wide() const { return wide_.data(); }
  const std::uint64_t* wide_offsets() const { return woff_.data(); }

 private:
  detail::PinnedVec<std::uint32_t> compact_, wide_;
  detail::PinnedVec<std::uint64_t> coff_, woff_;
};

// The densest host form (include/hfz.h, hfz_feedback_batch_packed_host): three bytes per host-half slot -- slot lo,
// slot hi, count; every exec padded with zero entries to a multiple of four -- and four per device-half slot,
// (slot - kHostSlots) | min(count, 65536) << 15 (the device ladder's last rung starts at 65,536: the clip keeps
// every class).  ~4.1 KB per exec at 2 % density against ~5.0 KB of CompactBatch; the call is PCIe-bound.
class PackedBatch {
  static_assert(kMapSize == 65536, "packed lists carry 15-bit slots per half");

 public:
  PackedBatch() {
    hoff_.push_back(0);
    doff_.push_back(0);
  }
  void append(const CoverageMap& m) {
    begin(m.touched().size());
    for (std::uint32_t slot : m.touched()) put(slot, static_cast<std::uint32_t>(m.count_at(slot)));
    finish();
  }
  // append(m) + m.reset() in one walk (see CompactBatch::take)
  void take(CoverageMap& m) {
    begin(m.touched().size());
    m.drain([this](std::uint32_t slot, std::uint32_t c) { put(slot, c); });
    finish();
  }
  void clear() {
    host_.clear();
    dev_.clear();
    hoff_.clear();
    doff_.clear();
    hoff_.push_back(0);
    doff_.push_back(0);
  }
  std::uint64_t size() const { return hoff_.size() - 1; }
  const std::uint8_t* host3() const { return host_.data(); }
  const std::uint64_t* host3_offsets() const { return hoff_.data(); }
  const std::uint32_t* dev17() const { return dev_.data(); }
  const std::uint64_t* dev17_offsets() const { return doff_.data(); }

 private:
  // room for one map's entries (all of them could land in either list) + the padding: put() writes unchecked
  void begin(std::uint64_t touched) {
    host_.reserve(host_.size() + 3 * touched + 12);
    dev_.reserve(dev_.size() + touched);
    h_ = host_.tail();
    d_ = dev_.tail();
  }
  void put(std::uint32_t slot, std::uint32_t c) {
    if (slot < kHostSlots) {
      h_[0] = static_cast<std::uint8_t>(slot);
      h_[1] = static_cast<std::uint8_t>(slot >> 8);
      h_[2] = static_cast<std::uint8_t>(c);
      h_ += 3;
    } else {
      *d_++ = (slot - kHostSlots) | ((c < 65536u ? c : 65536u) << 15);
    }
  }
  void finish() {
    host_.advance(static_cast<std::uint64_t>(h_ - host_.tail()));
    dev_.advance(static_cast<std::uint64_t>(d_ - dev_.tail()));
    while (host_.size() % 12) host_.push_back(0);  // whole groups of four 3-byte entries
    hoff_.push_back(host_.size() / 3);
    doff_.push_back(dev_.size());
  }
  std::uint8_t* h_ = nullptr;
  std::uint32_t* d_ = nullptr;
  detail::PinnedVec<std::uint8_t> host_;
  detail::PinnedVec<std::uint32_t> dev_;
  detail::PinnedVec<std::uint64_t> hoff_, doff_;
};

// Folds the batch into virgin / edge_counts in exec order (engine.cpp:471-478 per exec).
inline FeedbackResult feedback_batch(Context& ctx, const SparseBatch& batch, std::uint8_t* virgin,
                                     std::uint64_t* edge_counts, bool want_classed = false) {
  const std::uint64_t n = batch.size();
  FeedbackResult r;
  r.admit.resize(n);
  r.sig_full.resize(n);
  r.sig_simple.resize(n);
  r.nnz.resize(n);
  if (want_classed) r.classed.resize(n * std::uint64_t(ctx.map_slots()));
  check(hfz_feedback_batch_sparse_host(ctx.get(), batch.entries(), batch.offsets(), n, virgin, edge_counts,
                                       want_classed ? r.classed.data() : nullptr, r.admit.data(),
                                       r.sig_full.data(), r.sig_simple.data(), r.nnz.data()),
        "hfz_feedback_batch_sparse_host");
  return r;
}

inline FeedbackResult feedback_batch(Context& ctx, const CompactBatch& batch, std::uint8_t* virgin,
                                     std::uint64_t* edge_counts, bool want_classed = false) {
  const std::uint64_t n = batch.size();
  FeedbackResult r;
  r.admit.resize(n);
  r.sig_full.resize(n);
  r.sig_simple.resize(n);
  r.nnz.resize(n);
  if (want_classed) r.classed.resize(n * std::uint64_t(ctx.map_slots()));
  check(hfz_feedback_batch_compact_host(ctx.get(), batch.compact(), batch.compact_offsets(), batch.wide(),
                                        batch.wide_offsets(), n, virgin, edge_counts,
                                        want_classed ? r.classed.data() : nullptr, r.admit.data(),
                                        r.sig_full.data(), r.sig_simple.data(), r.nnz.data()),
        "hfz_feedback_batch_compact_host");
  return r;
}

inline FeedbackResult feedback_batch(Context& ctx, const PackedBatch& batch, std::uint8_t* virgin,
                                     std::uint64_t* edge_counts, bool want_classed = false) {
  const std::uint64_t n = batch.size();
  FeedbackResult r;
  r.admit.resize(n);
  r.sig_full.resize(n);
  r.sig_simple.resize(n);
  r.nnz.resize(n);
  if (want_classed) r.classed.resize(n * std::uint64_t(ctx.map_slots()));
  check(hfz_feedback_batch_packed_host(ctx.get(), batch.host3(), batch.host3_offsets(), batch.dev17(),
                                       batch.dev17_offsets(), n, virgin, edge_counts,
                                       want_classed ? r.classed.data() : nullptr, r.admit.data(),
                                       r.sig_full.data(), r.sig_simple.data(), r.nnz.data()),
        "hfz_feedback_batch_packed_host");
  return r;
}

// Several packed batches (one per packing thread, say) folded in the order given by ONE device call: batch k + 1
// crosses PCIe under the fold of batch k.  The results hold the execs of all batches, in batch order.
inline FeedbackResult feedback_batch(Context& ctx, const std::vector<const PackedBatch*>& batches, std::uint8_t* virgin,
                                     std::uint64_t* edge_counts) {
  std::vector<const std::uint8_t*> h3;
  std::vector<const std::uint64_t*> hoff, doff;
  std::vector<const std::uint32_t*> d17;
  std::vector<std::uint64_t> n;
  std::uint64_t total = 0;
  for (const PackedBatch* b : batches) {
    h3.push_back(b->host3());
    hoff.push_back(b->host3_offsets());
    d17.push_back(b->dev17());
    doff.push_back(b->dev17_offsets());
    n.push_back(b->size());
    total += b->size();
  }
  FeedbackResult r;
  r.admit.resize(total);
  r.sig_full.resize(total);
  r.sig_simple.resize(total);
  r.nnz.resize(total);
  check(hfz_feedback_batch_packed_host_v(ctx.get(), static_cast<std::uint32_t>(batches.size()), h3.data(), hoff.data(),
                                         d17.data(), doff.data(), n.data(), virgin, edge_counts, r.admit.data(),
                                         r.sig_full.data(), r.sig_simple.data(), r.nnz.data()),
        "hfz_feedback_batch_packed_host_v");
  return r;
}

}  // namespace b200

struct HostEdgeState {
  std::uint16_t prev_loc = 0;
};
inline void host_edge_update(HostEdgeState& st, std::uint16_t cur_loc, CoverageMap& map) {
  map.host_increment(static_cast<std::uint32_t>(st.prev_loc ^ cur_loc));
  st.prev_loc = static_cast<std::uint16_t>(cur_loc >> 1);
}
inline std::uint32_t device_edge_index(std::uint32_t prev_loc, std::uint32_t cur_loc) {
  return kDeviceIndexBase + ((prev_loc ^ cur_loc) % kHostSlots);
}

class DeviceEdgeState {
 public:
  std::uint32_t get(std::uint64_t tid) const {
    auto it = prev_.find(tid);
    return it == prev_.end() ? 0u : it->second;
  }
  void set(std::uint64_t tid, std::uint32_t v) { prev_[tid] = v; }
  void clear() { prev_.clear(); }
  std::size_t size() const { return prev_.size(); }

 private:
  std::unordered_map<std::uint64_t, std::uint32_t> prev_;
};

// Bucket ladders as data (rung lower bound -> one-hot class).  classify() on a single scalar is
// table lookup for callers that need it; the batch path classifies on the device.
class BucketLadder {
 public:
  struct Rung {
    std::uint64_t lower;
    std::uint8_t klass;
  };
  explicit BucketLadder(std::vector<Rung> rungs) : rungs_(std::move(rungs)) {}
  std::uint8_t classify(std::uint64_t count) const {
    std::uint8_t k = 0;
    for (const Rung& r : rungs_)
      if (count >= r.lower) k = r.klass;
    return k;
  }
  const std::vector<Rung>& rungs() const { return rungs_; }
  static const BucketLadder& host() {
    static const BucketLadder l({{1, 1}, {2, 2}, {3, 4}, {4, 8}, {8, 16}, {16, 32}, {32, 64}, {128, 128}});
    return l;
  }
  static const BucketLadder& device() {
    static const BucketLadder l({{1, 1}, {2, 2}, {3, 4}, {512, 8}, {4096, 16}, {16384, 32}, {65536, 64}});
    return l;
  }

 private:
  std::vector<Rung> rungs_;
};

struct ClassedTrace {
  std::vector<std::uint8_t> classed;   // kMapSize class bytes
  std::vector<std::uint32_t> nonzero;  // ascending logical indices
  ClassedTrace() : classed(kMapSize, 0) {}
};

class VirginMap {
 public:
  VirginMap() : bits_(kMapSize, 0) {}
  std::uint8_t at(std::uint32_t idx) const { return bits_[idx]; }
  bool edge_known(std::uint32_t idx) const { return bits_[idx] != 0; }
  std::uint64_t host_edges() const { return edges_[0]; }
  std::uint64_t device_edges() const { return edges_[1]; }
  void observe(std::uint32_t idx, std::uint8_t klass) {
    if (!bits_[idx]) ++edges_[idx < kHostSlots ? 0 : 1];
    bits_[idx] = static_cast<std::uint8_t>(bits_[idx] | klass);
  }
  // direct access for the batched device calls
  std::uint8_t* data() { return bits_.data(); }
  std::uint64_t* edge_counts() { return edges_; }

 private:
  std::vector<std::uint8_t> bits_;
  std::uint64_t edges_[2] = {0, 0};
};

enum class Admit : std::uint8_t { None = 0, NewCounts = 1, NewEdges = 2 };
enum class SignatureMode : std::uint8_t { Full, Simple };

namespace detail {
// The single-item calls below are batch-of-one device calls; their pinned list buffer is kept per thread
// (allocating and freeing page-locked memory per call cost more than the call: cudaHostAlloc + cudaFreeHost).
inline b200::SparseBatch& scratch_batch() {
  static thread_local b200::SparseBatch one;
  one.clear();
  return one;
}
// The touched-slot list of a map that classifies to exactly the given class bytes (lowest count of
// each rung): has_new_bits / trace_signature take a ClassedTrace, the device path takes counts.
// ~1,300 pairs (10 KB) cross PCIe per call instead of a dense 163,840-byte record.  A class byte
// that is not one rung of its half's ladder cannot come from classify_trace: refused, not guessed.
inline void pairs_from_classed(const ClassedTrace& t, b200::SparseBatch& out) {
  static const std::uint32_t host_lo[8] = {1, 2, 3, 4, 8, 16, 32, 128};
  static const std::uint32_t dev_lo[7] = {1, 2, 3, 512, 4096, 16384, 65536};
  static thread_local CoverageMap m;  // 160 KB: reused, back to all-zero in O(touched slots)
  m.reset();
  for (std::uint32_t idx : t.nonzero) {
    if (idx >= kMapSize) throw b200::Error("ClassedTrace: slot index out of range");
    const std::uint8_t k = t.classed[idx];
    int rung = 0;
    while (rung < 8 && !(k >> rung & 1)) ++rung;
    if (k == 0 || (k & (k - 1)) != 0 || (idx >= kHostSlots && rung > 6))
      throw b200::Error("ClassedTrace: class byte " + std::to_string(k) + " of slot " + std::to_string(idx) +
                        " is not a rung of the bucket ladder");
    if (idx < kHostSlots)
      m.host_assign(idx, static_cast<std::uint8_t>(host_lo[rung]));
    else
      m.device_store(idx, dev_lo[rung]);
  }
  out.append(m);
}
}  // namespace detail

namespace b200 {
// Everything Campaign::run_one needs from one execution's map (src/engine.cpp:471-478) in ONE device
// call: classes are implied, both signatures, the Admit code, virgin folded in place.  The
// reference-named functions below cost one call each; a host loop that adopts this library
// should call this (or, better, feedback_batch over many executions).
struct FeedbackOne {
  Admit admit;
  std::uint64_t sig_full, sig_simple;
  std::uint32_t nonzero_slots;
};
inline FeedbackOne feedback_one(const CoverageMap& map, VirginMap& virgin) {
  static thread_local SparseBatch one;  // pinned: kept per thread, not allocated per call
  one.clear();
  one.append(map);
  FeedbackResult r = feedback_batch(default_context(), one, virgin.data(), virgin.edge_counts());
  return FeedbackOne{static_cast<Admit>(r.admit[0]), r.sig_full[0], r.sig_simple[0], r.nnz[0]};
}
}  // namespace b200

inline ClassedTrace classify_trace(const CoverageMap& map) {
  b200::SparseBatch& one = detail::scratch_batch();
  one.append(map);
  std::vector<std::uint8_t> scratch_virgin(kMapSize, 0);
  std::uint64_t counts[2] = {0, 0};
  b200::FeedbackResult r =
      b200::feedback_batch(b200::default_context(), one, scratch_virgin.data(), counts, true);
  ClassedTrace out;
  out.classed = std::move(r.classed);
  out.nonzero.reserve(r.nnz[0]);
  // the touched list names every candidate slot: no scan of the 65,536 class bytes
  for (std::uint32_t s : map.touched())
    if (out.classed[s]) out.nonzero.push_back(s);
  std::sort(out.nonzero.begin(), out.nonzero.end());
  out.nonzero.erase(std::unique(out.nonzero.begin(), out.nonzero.end()), out.nonzero.end());  // a slot zeroed and hit again is listed twice
  return out;
}

inline Admit has_new_bits(const ClassedTrace& trace, VirginMap& virgin) {
  b200::SparseBatch& one = detail::scratch_batch();
  detail::pairs_from_classed(trace, one);
  b200::FeedbackResult r =
      b200::feedback_batch(b200::default_context(), one, virgin.data(), virgin.edge_counts());
  return static_cast<Admit>(r.admit[0]);
}

inline std::uint64_t trace_signature(const ClassedTrace& trace, SignatureMode mode) {
  b200::SparseBatch& one = detail::scratch_batch();
  detail::pairs_from_classed(trace, one);
  std::vector<std::uint8_t> scratch_virgin(kMapSize, 0);
  std::uint64_t counts[2] = {0, 0};
  b200::FeedbackResult r =
      b200::feedback_batch(b200::default_context(), one, scratch_virgin.data(), counts);
  return mode == SignatureMode::Full ? r.sig_full[0] : r.sig_simple[0];
}

inline void merge_device_into_map(const std::vector<std::uint32_t>& counters, CoverageMap& map) {
  for (std::size_t i = 0; i < counters.size(); ++i)
    if (counters[i]) map.device_store(kDeviceIndexBase + static_cast<std::uint32_t>(i), counters[i]);
}

// FNV-1a constants and helpers used by callers outside the hot path (dedup keys).
inline constexpr std::uint64_t kFnvOffset = 14695981039346656037ULL;
inline constexpr std::uint64_t kFnvPrime = 1099511628211ULL;
inline std::uint64_t fnv1a_step(std::uint64_t h, std::uint8_t byte) { return (h ^ byte) * kFnvPrime; }
inline std::uint64_t fnv1a_bytes(std::uint64_t h, const void* data, std::size_t len) {
  const auto* p = static_cast<const std::uint8_t*>(data);
  while (len--) h = fnv1a_step(h, *p++);
  return h;
}

}  // namespace hetfuzz
