// Shared device/host helpers for the hexdg_b200 kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/hexdg_b200.h"
#include "physics.cuh"

namespace hdg {

__device__ __forceinline__ Gas make_gas(const hdg_params& P) {
  Gas g;
  g.gamma = P.gamma;
  g.R = P.R;
  g.Pr = P.Pr;
  g.mu_ref = P.mu_ref;
  g.T_ref = P.T_ref;
  g.law = P.law;
  return g;
}

void set_error(const char* fmt, ...);
void count_launch();   // every kernel launch of the library (hdg_launch_count)

}  // namespace hdg
