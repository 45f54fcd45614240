// Bit-exact kernel set: compiled with -fmad=false so every float64 operation
// rounds exactly as in the reference's numba kernels (no FMA contraction).
#include "common.cuh"

namespace hdg_exact {
using namespace hdg;
// compile-time kernel-set flag: exact keeps the reference's operation order
constexpr bool kExact = true;
#include "kernels.cuh"
#include "elem.cuh"
#include "elem2.cuh"
#include "api_kernels.cuh"
#include "launch.cuh"
}  // namespace hdg_exact
