// Fixed-order block reductions (deterministic: the association depends only
// on blockDim / gridDim, never on scheduling).
#pragma once
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;  // valid in lane 0
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Reduce NV values per thread over the block: ops[k] = 0 sum, 1 max, 2 min.
// Result valid in thread 0.  `sh` must hold NV * 32 doubles.  Requires
// blockDim.x a multiple of 32 and <= 1024.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], const int (&ops)[NV], double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        v[k] = ops[k] == 0 ? warp_sum(v[k]) : (ops[k] == 1 ? warp_max(v[k]) : warp_min(v[k]));
        if (lane == 0) sh[k * 32 + wid] = v[k];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double init = ops[k] == 0 ? 0.0 : (ops[k] == 1 ? -INFINITY : INFINITY);
            double t = lane < nw ? sh[k * 32 + lane] : init;
            v[k] = ops[k] == 0 ? warp_sum(t) : (ops[k] == 1 ? warp_max(t) : warp_min(t));
        }
    }
    __syncthreads();
}

// "Last block done" protocol: every block writes its NV partials to
// part[blockIdx.x * NV + k]; the block that finishes last reduces all
// partials in block-index-strided fixed order and returns true in every
// thread of that block with the totals in v (thread 0).  counter reset to 0.
template <int NV>
__device__ __forceinline__ bool grid_reduce_last(double (&v)[NV], const int (&ops)[NV], double *part,
                                                 unsigned *counter, double *sh) {
    __shared__ int s_last;
    block_reduce<NV>(v, ops, sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) part[(size_t)blockIdx.x * NV + k] = v[k];
        __threadfence();
        unsigned t = atomicAdd(counter, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = ops[k] == 0 ? 0.0 : (ops[k] == 1 ? -INFINITY : INFINITY);
    for (unsigned bI = threadIdx.x; bI < gridDim.x; bI += blockDim.x) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double t = __ldcg(part + (size_t)bI * NV + k);
            acc[k] = ops[k] == 0 ? acc[k] + t : (ops[k] == 1 ? fmax(acc[k], t) : fmin(acc[k], t));
        }
    }
    block_reduce<NV>(acc, ops, sh);
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = acc[k];
    if (threadIdx.x == 0) *counter = 0u;
    return true;
}
