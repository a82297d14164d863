// Duration distributions (point / continuous uniform / piecewise-linear CDF).
// Reference: /root/reference/proj/include/microslice/distribution.hpp:18-200.
// Sampling semantics that the decision log depends on:
//  * uniform: lo + u*(hi-lo), llround, clamp to [lo, hi]
//  * empirical: inverse CDF by binary search on the cumulative column, linear
//    interpolation inside the bracket, llround, clamp to the bracket
//  * mean(): exact (uniform = integer midpoint; empirical = trapezoid sum, llround)
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "microslice/common.hpp"

namespace microslice {

class DurationDist {
 public:
  enum class Kind { Point, Uniform, Empirical };

  struct CdfPoint {
    Ns value = 0;
    double cum = 0.0;
  };

  static DurationDist point(Ns v);
  static DurationDist uniform(Ns lo, Ns hi);
  static DurationDist empirical(std::vector<CdfPoint> pts);

  Kind kind() const { return kind_; }

  /// Inverse-transform sample for a uniform variate u in [0, 1).
  Ns sample(double u) const;
  Ns sample(RngStream& rng) const { return sample(rng.next_double()); }
  Ns sample_keyed(std::uint64_t key) const { return sample(u01_from_key(key)); }

  Ns mean() const;
  Ns min_value() const { return kind_ == Kind::Empirical ? cdf_.front().value : lo_; }
  Ns max_value() const { return kind_ == Kind::Empirical ? cdf_.back().value : hi_; }
  double cdf_at(Ns t) const;
  const std::vector<CdfPoint>& breakpoints() const { return cdf_; }

 private:
  void check() const;
  Ns sample_cdf(double u) const;

  Kind kind_ = Kind::Point;
  Ns lo_ = 1;
  Ns hi_ = 1;
  std::vector<CdfPoint> cdf_;
};

/// Shipped synthetic block-time CDF: 5/100/300/400/1000 us at cum 0/.9/.999/.999995/1
/// (distribution.hpp:180-188).
DurationDist default_block_time_cdf();

std::string kind_name(DurationDist::Kind k);

}  // namespace microslice
