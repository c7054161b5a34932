// prims.cuh -- warp/block building blocks shared by the CUDA kernels (not by the oracle).
#pragma once
#include "internal.cuh"

namespace gps {

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(kFull, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    return x;
}

// Exclusive scan across the block (blockDim.x multiple of 32, <= 1024).  Every
// thread must call it.  *total receives the block sum.  Ends with a barrier so
// it can be called repeatedly.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
    __shared__ T s_w[32];
    const uint32_t lane = lane_id(), wid = warp_id(), nwarps = blockDim.x >> 5;
    T x = warp_incl_scan(v);
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T y = lane < nwarps ? s_w[lane] : T(0);
        y = warp_incl_scan(y);
        s_w[lane] = y;
    }
    __syncthreads();
    T pre = wid ? s_w[wid - 1] : T(0);
    *total = s_w[nwarps - 1];
    __syncthreads();
    return pre + x - v;
}

// Two u64 exclusive scans sharing one set of barriers.
__device__ __forceinline__ ulonglong2 block_excl_scan2(ulonglong2 v, ulonglong2* total) {
    __shared__ unsigned long long s_w[2][32];
    const uint32_t lane = lane_id(), wid = warp_id(), nwarps = blockDim.x >> 5;
    unsigned long long x = warp_incl_scan(v.x), y = warp_incl_scan(v.y);
    if (lane == 31) {
        s_w[0][wid] = x;
        s_w[1][wid] = y;
    }
    __syncthreads();
    if (wid == 0) {
        unsigned long long a = lane < nwarps ? s_w[0][lane] : 0ull, b = lane < nwarps ? s_w[1][lane] : 0ull;
        a = warp_incl_scan(a);
        b = warp_incl_scan(b);
        s_w[0][lane] = a;
        s_w[1][lane] = b;
    }
    __syncthreads();
    const unsigned long long pa = wid ? s_w[0][wid - 1] : 0ull, pb = wid ? s_w[1][wid - 1] : 0ull;
    *total = make_ulonglong2(s_w[0][nwarps - 1], s_w[1][nwarps - 1]);
    __syncthreads();
    return make_ulonglong2(pa + x - v.x, pb + y - v.y);
}

template <typename T>
__device__ __forceinline__ T block_sum(T v) {
    T tot;
    block_excl_scan(v, &tot);
    return tot;
}

}  // namespace gps
