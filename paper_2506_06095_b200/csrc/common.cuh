// common.cuh — shared host/device plumbing for the sm_100a library (status, errors, launch
// accounting, small device helpers). Everything here is internal; the public surface is
// include/sf_capi.h.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <utility>
#include <string>

#include "../../include/sf_capi.h"

namespace sf {

// Per-thread last error text (sf_last_error).
void set_error(const std::string& msg);
sf_status fail(sf_status st, const std::string& msg);
// Host-side launch counter (sf_launch_count): every kernel launch goes through note_launch().
void note_launch(int64_t n = 1);

// Programmatic dependent launch (PDL). The hot-path kernels are launched with programmatic stream
// serialization, so a kernel's grid is scheduled while its predecessor drains; each of them
// starts with pdl_enter(): wait for the predecessor grid (complete, memory visible) before
// touching any global data, then allow its own dependents to be scheduled. A kernel launched
// without the attribute passes both instantly. sf_set_pdl(0) turns the attribute off.
bool pdl_enabled();

// Stream-ordered allocation for the format builders' scratch and outputs. The device's default
// memory pool is set (once) to keep freed blocks instead of returning them to the driver at every
// synchronisation (release threshold 0 by default), so repeated builds reuse memory and a build's
// latency is its kernels and its one size read-back, not driver allocations.
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t st);
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// cudaLaunchKernelEx with the PDL attribute (plus up to one extra attribute, e.g. a cluster shape)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       const cudaLaunchAttribute* extra, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    int n = 1;
    if (extra) attr[n++] = *extra;
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define SF_CUDA_TRY(expr)                                                                    \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            return ::sf::fail(SF_CUDA_ERROR, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)

#define SF_LAUNCH_CHECK()                                                                    \
    do {                                                                                     \
        ::sf::note_launch();                                                                 \
        cudaError_t _e = cudaGetLastError();                                                 \
        if (_e != cudaSuccess)                                                               \
            return ::sf::fail(SF_CUDA_ERROR, std::string("launch: ") + cudaGetErrorString(_e)); \
    } while (0)

#define SF_TRY(expr)                                                                         \
    do {                                                                                     \
        sf_status _s = (expr);                                                               \
        if (_s != SF_OK) return _s;                                                          \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

// ---- device helpers -------------------------------------------------------------------------
template <typename T>
struct DT;
template <>
struct DT<__half> {
    static __device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
    static __device__ __forceinline__ __half from_f(float x) { return __float2half_rn(x); }
};
template <>
struct DT<__nv_bfloat16> {
    static __device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
    static __device__ __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// 64 bits of a bit-packed mask row starting at bit `start`; bits at or beyond `limit` are 0.
__device__ __forceinline__ uint64_t row_bits64(const uint32_t* row, int64_t start, int64_t limit) {
    if (start >= limit) return 0ull;
    const int64_t w0 = start >> 5;
    const int sh = static_cast<int>(start & 31);
    const int64_t wlim = (limit + 31) >> 5;
    uint64_t a = row[w0];
    uint64_t b = (w0 + 1 < wlim) ? row[w0 + 1] : 0u;
    uint64_t c = (w0 + 2 < wlim) ? row[w0 + 2] : 0u;
    uint64_t v = (a | (b << 32)) >> sh;
    if (sh) v |= c << (64 - sh);
    const int64_t avail = limit - start;
    if (avail < 64) v &= (1ull << avail) - 1ull;
    return v;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

}  // namespace sf
