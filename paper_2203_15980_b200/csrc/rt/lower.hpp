#pragma once
#include <cstdint>
#include <vector>

#include "delta/delta.h"
#include "deltasim/deltasim.hpp"

namespace delta_rt {

struct Program {
  deltasim::RunResult plan;
  std::vector<delta_action> actions;
  std::vector<std::uint64_t> inputs;  // arena offsets of COMPUTE/RECOMPUTE inputs
  std::uint64_t arena_bytes = 0;
  std::uint64_t pool_peak = 0;
  std::uint64_t host_bytes = 0;
  std::uint32_t n_events = 0;
};

// flags: DELTA_LOWER_DUPLEX_COPIES (delta.h) puts reloads on their own H2D
// stream; by default every copy runs on ONE copy stream in plan order, the
// reference's single copy stream (include/deltasim/device.hpp:45-74).
Program lower_plan(const deltasim::Trace& trace, const deltasim::EngineConfig& cfg,
                   std::uint64_t align, std::uint32_t flags = 0);

}  // namespace delta_rt
