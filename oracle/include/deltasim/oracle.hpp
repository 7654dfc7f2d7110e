// TEST INFRASTRUCTURE ONLY.  Declarations of the reference's independent
// verifier (ref include/deltasim/oracle.hpp:9-41), whose UNMODIFIED source
// (/root/reference/proj/src/oracle.cpp) oracle/Makefile compiles against the
// libdelta headers to certify libdelta timelines.  Not part of libdelta.
#pragma once
#include <string>
#include <vector>

#include "deltasim/deltasim.hpp"

namespace deltasim::oracle {

enum class ViolationCode {
  BudgetExceeded,
  UseWhileAbsent,
  BackwardRelease,
  PrefetchOverflow,
  NonmonotoneClock,
};
const char* to_string(ViolationCode c);

struct Violation {
  ViolationCode code;
  MicroTime ts = 0;
  NodeId node = 0;
  std::string detail;
};

std::vector<Violation> replay_check(const Timeline& timeline, const Trace& trace,
                                    const EngineConfig& cfg);
Bytes brute_force_min_peak(const Trace& trace, std::size_t max_nodes = 12);

}  // namespace deltasim::oracle
