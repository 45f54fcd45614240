// Fast kernel set: the same source as kernels_exact.cu, compiled with FMA
// contraction (nvcc default). Agrees with the reference to <= 1e-12 normwise.
#include "common.cuh"

namespace hdg_fast {
using namespace hdg;
// compile-time kernel-set flag: exact keeps the reference's operation order
constexpr bool kExact = false;
#include "kernels.cuh"
#include "elem.cuh"
#include "elem2.cuh"
#include "api_kernels.cuh"
#include "launch.cuh"
}  // namespace hdg_fast
