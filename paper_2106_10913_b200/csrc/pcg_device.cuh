// Device-side PCG reductions shared by the PCG kernels (ops.cu) and the
// kernels that fuse a PCG dot into their epilogue (kernels.cu).
#pragma once

#include "awg_internal.cuh"

namespace awgb {
namespace pcgdev {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block partial -> fixed slot; the last block to arrive sums the slots in a
// fixed order (deterministic single-pass grid reduction) and runs `fin`.
// Every thread of every block must call it.
template <class Fin>
__device__ void grid_reduce(double v, double* part, unsigned* count, Fin fin) {
  __shared__ double sred[32];
  __shared__ int is_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += sred[w];
    part[blockIdx.x] = acc;
    __threadfence();
    const unsigned t = atomicAdd(count, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last && warp == 0) {
    __threadfence();
    double acc = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) acc += __ldcg(part + b);
    acc = warp_sum(acc);
    if (lane == 0) {
      fin(acc);
      *count = 0;
    }
  }
}

// rz = <r, z>: the initial check (krylov.cpp:51-53) or the beta step (:105-115)
__device__ inline void rz_finish(PcgState* st, double rz, int initial) {
  if (initial) {
    if (rz <= 0.0) {
      st->error = PCG_BAD_PRECOND;
      st->done = 1;
    }
    st->rz = rz;
    st->beta = 0.0;
    return;
  }
  if (rz <= 0.0) {
    if (!st->past_rtol) st->error = PCG_BAD_PRECOND;
    st->done = 1;
    return;
  }
  const double beta = rz / st->rz;
  st->beta = beta;
  st->rz = rz;
  st->beta_prev = beta;
  st->alpha_prev = st->alpha;
}

}  // namespace pcgdev
}  // namespace awgb
