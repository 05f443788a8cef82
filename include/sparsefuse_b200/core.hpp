// core.hpp — foundation of the C++ host API over the C ABI (include/sf_capi.h).
//
// Mirrors the reference's foundation (common.hpp:11-95): the same eight exception types (the
// error convention of the whole API), the seeded helpers (unit_real, mix_seed, fnv1a, pack_bits)
// and adds what a device-resident implementation needs: status -> exception translation and an
// owning device buffer. Header-only; link against libsf_b200.so and libcudart.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../sf_capi.h"

namespace sparsefuse {

// ---- error taxonomy (common.hpp:14-36): same names, same std bases ------------------------
struct invalid_parameter : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct shape_error : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct plan_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct degenerate_input : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct illegal_segment : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct internal_inconsistency : std::logic_error { using std::logic_error::logic_error; };
struct backend_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct io_error : std::runtime_error { using std::runtime_error::runtime_error; };
// device failures have no reference counterpart; they surface as backend_error so a tuning
// search skips the candidate exactly like an unexecutable one (search.hpp:336-341)
struct cuda_error : backend_error { using backend_error::backend_error; };

// Translate a C-ABI status into the matching exception.
inline void check(sf_status st) {
    if (st == SF_OK) return;
    const std::string msg = sf_last_error();
    switch (st) {
        case SF_INVALID_PARAMETER: throw invalid_parameter(msg);
        case SF_SHAPE_ERROR: throw shape_error(msg);
        case SF_PLAN_ERROR: throw plan_error(msg);
        case SF_DEGENERATE_INPUT: throw degenerate_input(msg);
        case SF_ILLEGAL_SEGMENT: throw illegal_segment(msg);
        case SF_INTERNAL_INCONSISTENCY: throw internal_inconsistency(msg);
        case SF_BACKEND_ERROR: throw backend_error(msg);
        case SF_IO_ERROR: throw io_error(msg);
        default: throw cuda_error(msg);
    }
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- seeded helpers (common.hpp:39-93) -------------------------------------------------------
// Floating draws use the raw 64-bit output (top 53 bits * 2^-53), never
// std::uniform_real_distribution, so values are reproducible everywhere.
inline double unit_real(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t tag) {  // splitmix64 finalizer
    std::uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

inline std::uint64_t fnv1a(std::string_view s, std::uint64_t h = 0xcbf29ce484222325ULL) {
    for (unsigned char c : s) h = (h ^ c) * 0x100000001b3ULL;
    return h;
}

inline std::string hex64(std::uint64_t v) {
    static const char* digits = "0123456789abcdef";
    std::string out(16, '0');
    for (int i = 15; i >= 0; --i, v >>= 4) out[static_cast<std::size_t>(i)] = digits[v & 0xf];
    return out;
}

inline std::vector<std::uint8_t> pack_bits(const std::vector<std::uint8_t>& bits) {
    std::vector<std::uint8_t> out((bits.size() + 7) / 8, 0);
    for (std::size_t i = 0; i < bits.size(); ++i)
        out[i >> 3] |= static_cast<std::uint8_t>((bits[i] ? 1u : 0u) << (i & 7));
    return out;
}

inline std::vector<std::uint8_t> unpack_bits(const std::vector<std::uint8_t>& bytes, std::size_t nbits) {
    if (bytes.size() < (nbits + 7) / 8) throw io_error("bit payload shorter than expected");
    std::vector<std::uint8_t> out(nbits);
    for (std::size_t i = 0; i < nbits; ++i) out[i] = (bytes[i >> 3] >> (i & 7)) & 1u;
    return out;
}

// ---- device memory -------------------------------------------------------------------------
template <typename T>
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t n) { resize(n); }
    ~DeviceBuffer() { reset(); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            reset();
            p_ = std::exchange(o.p_, nullptr);
            n_ = std::exchange(o.n_, 0);
        }
        return *this;
    }
    void resize(std::size_t n) {
        if (n == n_) return;
        reset();
        if (n) cuda_check(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)), "cudaMalloc");
        n_ = n;
    }
    void reset() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* data() { return p_; }
    const T* data() const { return p_; }
    std::size_t size() const { return n_; }
    void upload(const T* src, std::size_t n, cudaStream_t st = nullptr) {
        resize(n);
        if (n) cuda_check(cudaMemcpyAsync(p_, src, n * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
    }
    void download(T* dst, std::size_t n, cudaStream_t st = nullptr) const {
        if (n) cuda_check(cudaMemcpyAsync(dst, p_, n * sizeof(T), cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "sync");
    }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

}  // namespace sparsefuse
