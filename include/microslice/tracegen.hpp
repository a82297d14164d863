// Synthetic HP request arrivals: two-state Markov-modulated Poisson process.
// Reference: /root/reference/proj/include/microslice/tracegen.hpp:14-61.
// burstiness = 1 degenerates to plain Poisson; identical (params, seed) -> identical
// trace.  The configs' HP traces are produced here.
#pragma once

#include <cstdint>
#include <vector>

#include "microslice/common.hpp"

namespace microslice {

std::vector<Ns> generate_bursty_arrivals(double rate, double burstiness, Ns horizon,
                                         std::uint64_t seed, Ns dwell = seconds(2));

}  // namespace microslice
