// Internal definitions of the opaque kernel handles shared by the C-ABI
// launchers (runtime.cu) and the step executor (executor.cu).
#pragma once
#include <string>
#include "delta/delta_kernels.h"
#include "kernels/kernels.hpp"

struct delta_conv {
  delta_k::ConvPlan plan;
  const void* weight = nullptr;
};

struct delta_wgrad {
  delta_k::WgradPlan plan;
};

// thread-local last error of the C ABI (capi.cpp; also delta_rt::set_error)
void delta_set_error(const std::string& msg);
