// ptxas probe: compiles ONE element-kernel instantiation (registers / spills / SASS)
// without the whole library. nvcc -c tools/probe_elem2.cu -DPROBE_N=7 -DPROBE_VISC=1 ...
#include "../paper_2404_12703_b200/csrc/common.cuh"
#ifndef PROBE_EXACT
#define PROBE_EXACT 0
#endif
#ifndef PROBE_N
#define PROBE_N 7
#endif
#ifndef PROBE_VISC
#define PROBE_VISC 1
#endif
#ifndef PROBE_SHOCK
#define PROBE_SHOCK 0
#endif
#ifndef PROBE_LISTED
#define PROBE_LISTED 0
#endif
namespace hdg_probe {
using namespace hdg;
constexpr bool kExact = PROBE_EXACT;
#include "../paper_2404_12703_b200/csrc/kernels.cuh"
#include "../paper_2404_12703_b200/csrc/elem.cuh"
#include "../paper_2404_12703_b200/csrc/elem2.cuh"
template __global__ void elem2_kernel<PROBE_N, PROBE_VISC, PROBE_SHOCK, PROBE_LISTED, false>(
    hdg_domain, hdg_params, const double*, const int32_t*, int, Gate);
}
