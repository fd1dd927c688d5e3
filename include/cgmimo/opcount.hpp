// cgmimo/opcount.hpp -- drop-in subset of the reference's real-multiplication
// accounting (reference proj/include/cgmimo/opcount.hpp:21-79).  The GPU
// detect_cg cannot count inside the kernel; when a tally is active it
// records the count the reference's instrumented FP64 path would have
// recorded, stage by stage (tests/test_dropin.py checks it against the
// reference's own tallies).
#pragma once

#include <array>
#include <cstdint>

namespace cgmimo::opcount {

enum class Stage : int {
  kGram = 0,
  kMatchedFilter,
  kCgIteration,
  kTracker,
  kCholesky,
  kSubstitution,
  kNeumannTerm,
  kCglsIteration,
  kOther,
};
inline constexpr int kStageCount = 9;

class Tally {
 public:
  void add(Stage s, std::uint64_t n) { c_[static_cast<int>(s)] += n; }
  std::uint64_t get(Stage s) const { return c_[static_cast<int>(s)]; }
  std::uint64_t total() const {
    std::uint64_t t = 0;
    for (auto v : c_) t += v;
    return t;
  }
  void reset() { c_.fill(0); }

 private:
  std::array<std::uint64_t, kStageCount> c_{};
};

class ScopedTally {
 public:
  explicit ScopedTally(Tally& t);
  ~ScopedTally();
  ScopedTally(const ScopedTally&) = delete;
  ScopedTally& operator=(const ScopedTally&) = delete;

 private:
  Tally* prev_;
};

void record(Stage stage, std::uint64_t real_mults);
bool counting_active();

}  // namespace cgmimo::opcount
