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

__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// every thread fences its remote stores (system scope) before the block counts
// itself done; the block that completes the grid advances the phase epoch (a
// device counter, so the launch is graph-replayable) and releases it to every
// neighbour's flag word. The block counter wraps inside each launch (atomicInc
// with limit gridDim.x - 1 returns gridDim.x - 1 to the last block and stores 0),
// so it is back at 0 after every launch and never overflows.
__device__ __forceinline__ void publish_epoch(unsigned* counter, const unsigned long long* flag_ptrs,
                                              int n_nbr, unsigned long long* epoch_ctr) {
  __shared__ int s_last;
  __shared__ unsigned long long s_epoch;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    s_last = atomicInc(counter, gridDim.x - 1u) == gridDim.x - 1u;
    if (s_last) s_epoch = atomicAdd(epoch_ctr, 1ull) + 1ull;
  }
  __syncthreads();
  if (s_last && (int)threadIdx.x < n_nbr) {
    __threadfence_system();
    st_release_sys_u64(reinterpret_cast<unsigned long long*>(flag_ptrs[threadIdx.x]), s_epoch);
  }
}

// A kernel's wait for a neighbour exchange, fused into the consumer: work items
// at list position >= pos need the neighbours' payload of a phase, published
// with the epoch this rank's own send of that phase already wrote to *epoch
// (every rank sends each phase the same number of times). One thread spins
// (acquire, system scope, bounded ~10 s -> status[HDG_STATUS_PEER_TIMEOUT]),
// the block waits at a barrier. n == 0: no gate.
struct Gate {
  const unsigned long long* flags;
  const int32_t* idx;
  int n;
  int pos;
  const unsigned long long* epoch;
  int32_t* status;
};

__device__ __forceinline__ void gate_wait(const Gate& g) {
  if (threadIdx.x == 0) {
    const unsigned long long want = *reinterpret_cast<const volatile unsigned long long*>(g.epoch);
    for (int i = 0; i < g.n; ++i) {
      const unsigned long long* f = g.flags + g.idx[i];
      const long long t0 = clock64();
      while (ld_acquire_sys_u64(f) < want) {
        __nanosleep(64);
        if (clock64() - t0 > 20000000000LL) {
          atomicExch(&g.status[HDG_STATUS_PEER_TIMEOUT], 1);
          break;
        }
      }
    }
  }
  __syncthreads();
}

void set_error(const char* fmt, ...);
void count_launch();   // every kernel launch of the library (hdg_launch_count)

// SMs of the current device (host; one device per process), for grid caps
inline int sm_count() {
  static int n = 0;
  if (n <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace hdg
