// scan.cuh — single-CTA exclusive prefix sums used by the format builders.
// The arrays scanned here are row pointers (<= n_rows+1) and part-tile flags (<= tiles), small
// enough that one 1024-thread CTA streaming contiguous per-thread chunks is latency-bound, not
// bandwidth-bound; it avoids a multi-pass device-wide scan.
#pragma once
#include "common.cuh"

namespace sf {

// out[0] = 0, out[i+1] = sum(in[0..i]) for i < count; out may alias nothing. Optional total.
__global__ void scan_exclusive_kernel(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                                      int64_t count, int32_t* total) {
    __shared__ int32_t warp_sums[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t per = (count + nt - 1) / nt;
    const int64_t b = per * tid, e = min(count, b + per);
    int32_t local = 0;
    for (int64_t i = b; i < e; ++i) local += in[i];
    // block exclusive scan of `local`
    const int lane = tid & 31, wid = tid >> 5;
    int32_t x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int32_t s = lane < (nt >> 5) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    int32_t run = x - local + (wid ? warp_sums[wid - 1] : 0);
    if (tid == 0) out[0] = 0;
    for (int64_t i = b; i < e; ++i) {
        run += in[i];
        out[i + 1] = run;
    }
    if (total && tid == nt - 1) *total = run;
    if (total && count == 0 && tid == 0) *total = 0;
}

// Three independent exclusive scans in one launch (blockIdx.y picks the array): the full / part /
// load row pointers of a BSR build.
__global__ void scan_exclusive3_kernel(const int32_t* in0, const int32_t* in1, const int32_t* in2, int32_t* out0,
                                       int32_t* out1, int32_t* out2, int64_t count, int32_t* totals) {
    __shared__ int32_t warp_sums[32];
    const int which = blockIdx.y;
    const int32_t* in = which == 0 ? in0 : (which == 1 ? in1 : in2);
    int32_t* out = which == 0 ? out0 : (which == 1 ? out1 : out2);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t per = (count + nt - 1) / nt;
    const int64_t b = per * tid, e = min(count, b + per);
    int32_t local = 0;
    for (int64_t i = b; i < e; ++i) local += in[i];
    const int lane = tid & 31, wid = tid >> 5;
    int32_t x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int32_t s = lane < (nt >> 5) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    int32_t run = x - local + (wid ? warp_sums[wid - 1] : 0);
    if (tid == 0) out[0] = 0;
    for (int64_t i = b; i < e; ++i) {
        run += in[i];
        out[i + 1] = run;
    }
    if (tid == nt - 1) totals[which] = run;
    if (count == 0 && tid == 0) totals[which] = 0;
}

inline sf_status scan_exclusive(const int32_t* in, int32_t* out, int64_t count, int32_t* total,
                                cudaStream_t st) {
    scan_exclusive_kernel<<<1, 1024, 0, st>>>(in, out, count, total);
    SF_LAUNCH_CHECK();
    return SF_OK;
}

}  // namespace sf
