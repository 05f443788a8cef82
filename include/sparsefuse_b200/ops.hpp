// ops.hpp — masks, storage formats, selector and masked MHA of the C++ host API.
//
// Same names / argument meaning / exception types as the reference's mask.hpp, bsr.hpp,
// planner.hpp, tensor.hpp and attention.hpp, but every computation runs on the B200 through the C
// ABI: masks are generated and kept bit-packed on the device (host bytes are materialised lazily
// when code reads them), formats are built by the device builders (bit-exact with build_bsr /
// build_rowwise), and the executors are the sm_100a kernels.
#pragma once

#include <algorithm>
#include <cmath>
#include <initializer_list>
#include <limits>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "core.hpp"

namespace sparsefuse {

// =============================================================================================
// DenseMask (mask.hpp:18-54): device-resident bit mask with a lazily synchronised host view.
class DenseMask {
public:
    explicit DenseMask(int seq_len, bool value = false) : n_(seq_len) {
        if (seq_len <= 0) throw invalid_parameter("seq_len must be positive");
        dev_.resize(words_total());
        if (value) {
            sf_mask_desc all{SF_PATTERN_GLOBAL, seq_len, 0, seq_len, 0, 16, 0.0, 0};
            check(sf_mask_generate(&all, 1, dev_.data(), nullptr));
        } else {
            cuda_check(cudaMemset(dev_.data(), 0, words_total() * 4), "cudaMemset");
        }
        dev_ok_ = true;
    }
    DenseMask(const DenseMask& o) : n_(o.n_), host_(o.host_), host_ok_(o.host_ok_), dev_ok_(o.dev_ok_) {
        if (o.dev_ok_) {
            dev_.resize(words_total());
            cuda_check(cudaMemcpy(dev_.data(), o.dev_.data(), words_total() * 4, cudaMemcpyDeviceToDevice), "D2D");
        }
    }
    DenseMask(DenseMask&&) noexcept = default;
    DenseMask& operator=(const DenseMask& o) {
        if (this != &o) *this = DenseMask(o);
        return *this;
    }
    DenseMask& operator=(DenseMask&&) noexcept = default;

    int seq_len() const { return n_; }
    bool get(int i, int j) const { return raw()[static_cast<std::size_t>(i) * n_ + static_cast<std::size_t>(j)] != 0; }
    void set(int i, int j, bool v) {
        sync_host();
        host_[static_cast<std::size_t>(i) * n_ + static_cast<std::size_t>(j)] = v ? 1 : 0;
        dev_ok_ = false;
    }
    std::int64_t true_count() const {
        std::int64_t c = 0;
        check(sf_mask_count(device_bits(), n_, &c, nullptr));
        return c;
    }
    const std::vector<std::uint8_t>& raw() const {
        sync_host();
        return host_;
    }
    bool operator==(const DenseMask& o) const { return n_ == o.n_ && raw() == o.raw(); }

    // Device view: n rows of sf_mask_words(n) uint32 (sf_capi.h layout).
    const std::uint32_t* device_bits() const {
        sync_device();
        return dev_.data();
    }
    std::uint32_t* mutable_device_bits() {
        sync_device();
        host_ok_ = false;
        return dev_.data();
    }
    std::size_t words_total() const { return static_cast<std::size_t>(n_) * sf_mask_words(n_); }

private:
    void sync_host() const {
        if (host_ok_) return;
        std::vector<std::uint32_t> w(words_total());
        dev_.download(w.data(), w.size());
        const int W = sf_mask_words(n_);
        host_.assign(static_cast<std::size_t>(n_) * n_, 0);
        for (int i = 0; i < n_; ++i)
            for (int j = 0; j < n_; ++j)
                host_[static_cast<std::size_t>(i) * n_ + j] = (w[static_cast<std::size_t>(i) * W + (j >> 5)] >> (j & 31)) & 1u;
        host_ok_ = true;
    }
    void sync_device() const {
        if (dev_ok_) return;
        DeviceBuffer<std::uint8_t> u8;
        u8.upload(host_.data(), host_.size());
        dev_.resize(words_total());
        check(sf_mask_pack_u8(u8.data(), n_, dev_.data(), nullptr));
        cuda_check(cudaDeviceSynchronize(), "pack");
        dev_ok_ = true;
    }

    int n_;
    mutable DeviceBuffer<std::uint32_t> dev_;
    mutable std::vector<std::uint8_t> host_;
    mutable bool host_ok_ = false, dev_ok_ = false;
};

inline double sparsity(const DenseMask& m) {  // mask.hpp:57-60
    const double total = static_cast<double>(m.seq_len()) * m.seq_len();
    return 1.0 - static_cast<double>(m.true_count()) / total;
}

struct PatternParams {  // mask.hpp:64-71
    int band_width = 0;
    int global_width = 0;
    int dilation_rate = 0;
    double filling_rate = 0.0;
    int block = 16;
    std::uint64_t seed = 0;
};

// io.hpp:158-162 (+ "causal", "causal_local", "strided", which the reference lacks)
struct MaskDescriptor {
    std::string pattern;
    int seq_len = 0;
    PatternParams params;
};

inline sf_pattern pattern_code(const std::string& p) {
    static const char* names[] = {"sliding", "dilated", "global", "random", "longformer",
                                  "bigbird", "causal", "causal_local", "strided"};
    for (int i = 0; i < 9; ++i)
        if (p == names[i]) return static_cast<sf_pattern>(i);
    throw invalid_parameter("unknown mask pattern: " + p);
}

inline sf_mask_desc to_c(const MaskDescriptor& d) {
    const auto& p = d.params;
    return sf_mask_desc{pattern_code(d.pattern), d.seq_len, p.band_width, p.global_width, p.dilation_rate,
                        p.block, p.filling_rate, p.seed};
}

// generate_mask (io.hpp:192-204): one descriptor, or the union of several (compose).
inline DenseMask generate_mask(const std::vector<MaskDescriptor>& terms) {
    std::vector<sf_mask_desc> c;
    for (const auto& t : terms) c.push_back(to_c(t));
    check(sf_mask_validate(c.data(), static_cast<int32_t>(c.size())));
    DenseMask m(c.front().seq_len);
    check(sf_mask_generate(c.data(), static_cast<int32_t>(c.size()), m.mutable_device_bits(), nullptr));
    return m;
}
inline DenseMask generate_mask(const MaskDescriptor& d) { return generate_mask(std::vector<MaskDescriptor>{d}); }

inline DenseMask gen_sliding_window(int n, int w) { return generate_mask({"sliding", n, {w, 0, 0, 0.0, 16, 0}}); }
inline DenseMask gen_dilated(int n, int w, int r) { return generate_mask({"dilated", n, {w, 0, r, 0.0, 16, 0}}); }
inline DenseMask gen_global(int n, int g) { return generate_mask({"global", n, {0, g, 0, 0.0, 16, 0}}); }
inline DenseMask gen_random_blocks(int n, int block, double fill, std::uint64_t seed) {
    return generate_mask({"random", n, {0, 0, 0, fill, block, seed}});
}
inline DenseMask gen_longformer(int n, int g, int w) { return generate_mask({"longformer", n, {w, g, 0, 0.0, 16, 0}}); }
inline DenseMask gen_bigbird(int n, int g, int w, double fill, std::uint64_t seed, int block = 16) {
    return generate_mask({"bigbird", n, {w, g, 0, fill, block, seed}});
}
inline DenseMask gen_causal(int n) { return generate_mask({"causal", n, {}}); }
inline DenseMask gen_strided(int n, int w) { return generate_mask({"strided", n, {w, 0, 0, 0.0, 16, 0}}); }

// compose (mask.hpp:146-166): element-wise union, on device.
inline DenseMask compose(std::span<const DenseMask> masks) {
    if (masks.empty()) throw invalid_parameter("compose needs at least one mask");
    const int n = masks.front().seq_len();
    for (const auto& m : masks)
        if (m.seq_len() != n) throw shape_error("compose: mismatched seq_len");
    DenseMask out(masks.front());
    for (std::size_t k = 1; k < masks.size(); ++k)
        check(sf_mask_or(masks[k].device_bits(), out.mutable_device_bits(), n, nullptr));
    return out;
}
inline DenseMask compose(std::initializer_list<DenseMask> masks) {
    std::vector<DenseMask> v(masks);
    return compose(std::span<const DenseMask>(v));
}

// =============================================================================================
// Storage formats (bsr.hpp:21-45): the reference's host arrays, plus the device copy the
// kernels read. build_bsr / build_rowwise run on the device and are bit-exact.
struct BsrDevice {
    sf_bsr_dev d{};
    ~BsrDevice() { sf_bsr_free(&d, nullptr); }
};

struct BsrMask {
    int seq_len = 0, block_m = 0, block_n = 0, n_rows = 0, n_cols = 0;
    std::vector<std::int32_t> full_row_ptr, full_col_idx, part_row_ptr, part_col_idx, part_tile_ids;
    std::vector<std::int32_t> load_row_ptr, load_col_idx;
    std::vector<std::vector<std::uint8_t>> part_mask_pool;  // block_m*block_n bytes each, row-major
    std::shared_ptr<BsrDevice> device;                      // null for host-constructed masks
};

struct RowwiseDevice {
    sf_csr_dev d{};
    ~RowwiseDevice() { sf_csr_free(&d, nullptr); }
};

struct RowwiseMask {
    int seq_len = 0;
    std::vector<std::int32_t> row_ptr, col_idx;
    std::shared_ptr<RowwiseDevice> device;
};

inline BsrMask build_bsr(const DenseMask& mask, int block_m, int block_n) {
    auto dev = std::make_shared<BsrDevice>();
    check(sf_bsr_build(mask.device_bits(), mask.seq_len(), block_m, block_n, &dev->d, nullptr));
    const sf_bsr_dev& d = dev->d;
    BsrMask b;
    b.seq_len = d.seq_len; b.block_m = d.block_m; b.block_n = d.block_n; b.n_rows = d.n_rows; b.n_cols = d.n_cols;
    b.full_row_ptr.resize(d.n_rows + 1); b.part_row_ptr.resize(d.n_rows + 1); b.load_row_ptr.resize(d.n_rows + 1);
    b.full_col_idx.resize(d.n_full); b.part_col_idx.resize(d.n_part); b.part_tile_ids.resize(d.n_part);
    b.load_col_idx.resize(d.n_load);
    std::vector<std::uint8_t> packed(static_cast<std::size_t>(d.n_pool) * d.tile_bytes);
    check(sf_bsr_to_host(&d, b.full_row_ptr.data(), b.full_col_idx.data(), b.part_row_ptr.data(),
                         b.part_col_idx.data(), b.part_tile_ids.data(), b.load_row_ptr.data(), b.load_col_idx.data(),
                         packed.data(), nullptr));
    const std::size_t nbits = static_cast<std::size_t>(block_m) * block_n;
    for (int t = 0; t < d.n_pool; ++t) {
        std::vector<std::uint8_t> bytes(packed.begin() + static_cast<std::ptrdiff_t>(t) * d.tile_bytes,
                                        packed.begin() + static_cast<std::ptrdiff_t>(t + 1) * d.tile_bytes);
        b.part_mask_pool.push_back(unpack_bits(bytes, nbits));
    }
    b.device = std::move(dev);
    return b;
}

inline RowwiseMask build_rowwise(const DenseMask& mask) {
    auto dev = std::make_shared<RowwiseDevice>();
    check(sf_rowwise_build(mask.device_bits(), mask.seq_len(), &dev->d, nullptr));
    RowwiseMask r;
    r.seq_len = mask.seq_len();
    r.row_ptr.resize(static_cast<std::size_t>(r.seq_len) + 1);
    r.col_idx.resize(static_cast<std::size_t>(dev->d.nnz));
    check(sf_csr_to_host(&dev->d, r.row_ptr.data(), r.col_idx.data(), nullptr));
    r.device = std::move(dev);
    return r;
}

// Device copy of a host-constructed BsrMask (e.g. read from an SFBR dump); shape checks that the
// packed device form cannot express are done here, with validate_bsr's messages.
inline std::shared_ptr<BsrDevice> upload_bsr(const BsrMask& b) {
    const std::size_t rp = static_cast<std::size_t>(b.n_rows) + 1;
    if (b.full_row_ptr.size() != rp) throw internal_inconsistency("full: bad row_ptr shape");
    if (b.part_row_ptr.size() != rp) throw internal_inconsistency("part: bad row_ptr shape");
    if (b.load_row_ptr.size() != rp) throw internal_inconsistency("load: bad row_ptr shape");
    if (b.part_tile_ids.size() != b.part_col_idx.size())
        throw internal_inconsistency("part_tile_ids not parallel to part_col_idx");
    const std::size_t nbits = static_cast<std::size_t>(b.block_m) * b.block_n, tb = (nbits + 7) / 8;
    std::vector<std::uint8_t> packed;
    packed.reserve(b.part_mask_pool.size() * tb);
    for (const auto& t : b.part_mask_pool) {
        if (t.size() != nbits) throw internal_inconsistency("pool tile has wrong size");
        const auto p = pack_bits(t);
        packed.insert(packed.end(), p.begin(), p.end());
    }
    auto dev = std::make_shared<BsrDevice>();
    check(sf_bsr_from_host(b.seq_len, b.block_m, b.block_n, static_cast<int32_t>(b.full_col_idx.size()),
                           static_cast<int32_t>(b.part_col_idx.size()), static_cast<int32_t>(b.load_col_idx.size()),
                           static_cast<int32_t>(b.part_mask_pool.size()), b.full_row_ptr.data(), b.full_col_idx.data(),
                           b.part_row_ptr.data(), b.part_col_idx.data(), b.part_tile_ids.data(), b.load_row_ptr.data(),
                           b.load_col_idx.data(), packed.data(), &dev->d, nullptr));
    return dev;
}

// validate_bsr (bsr.hpp:104-153): the structural checks run on the device copy; a mask whose host
// arrays were edited after the build is re-uploaded first.
inline void validate_bsr(const BsrMask& b, bool use_device_copy = false) {
    if (use_device_copy && b.device) {
        check(sf_bsr_validate(&b.device->d, nullptr));
        return;
    }
    const auto dev = upload_bsr(b);
    check(sf_bsr_validate(&dev->d, nullptr));
}

// to_dense (bsr.hpp:155-177): the exact inverse of build_bsr, expanded on the device.
inline DenseMask to_dense(const BsrMask& b) {
    const auto dev = upload_bsr(b);
    DenseMask m(b.seq_len);
    check(sf_bsr_to_dense(&dev->d, m.mutable_device_bits(), nullptr));
    cuda_check(cudaDeviceSynchronize(), "to_dense");
    return m;
}

struct BlockStats {  // bsr.hpp:179-196
    std::int64_t full_count = 0, part_count = 0, empty_count = 0;
    double valid_block_ratio = 0.0;
};

inline BlockStats block_stats(const BsrMask& b) {
    BlockStats s;
    s.full_count = b.full_row_ptr.back();
    s.part_count = b.part_row_ptr.back();
    const std::int64_t total = static_cast<std::int64_t>(b.n_rows) * b.n_cols;
    s.empty_count = total - s.full_count - s.part_count;
    s.valid_block_ratio = total > 0 ? static_cast<double>(s.full_count + s.part_count) / static_cast<double>(total) : 0.0;
    return s;
}

// SFBR bytes (io.hpp:97-122) of a device-built mask: the byte-exact parity currency.
inline std::string bsr_dump(const BsrMask& b) {
    if (!b.device) throw plan_error("BSR is not resident on the device (build it with build_bsr)");
    std::int64_t nb = 0;
    check(sf_bsr_serialize(&b.device->d, nullptr, 0, &nb, nullptr));
    std::string s(static_cast<std::size_t>(nb), '\0');
    check(sf_bsr_serialize(&b.device->d, reinterpret_cast<std::uint8_t*>(s.data()), nb, &nb, nullptr));
    return s;
}

// =============================================================================================
// Analytical selector (planner.hpp:20-161). Eq. 1 routes row-wise vs block-wise from the
// device-built 16x16 load count; Eq. 2 scans the setting grid on the host in exact doubles.
struct HardwareSpec {
    std::string name;
    int sm_num = 0;
    std::int64_t smem_size = 0;
    int max_warp = 0;
    int element_bytes = 2;
    void check() const {
        if (sm_num <= 0 || smem_size <= 0 || max_warp <= 0 || element_bytes <= 0)
            throw invalid_parameter("hardware spec fields must be positive");
    }
    sf_hw_spec to_c() const {
        sf_hw_spec h{};
        std::strncpy(h.name, name.c_str(), sizeof(h.name) - 1);
        h.sm_num = sm_num; h.smem_size = smem_size; h.max_warp = max_warp; h.element_bytes = element_bytes;
        return h;
    }
};

inline HardwareSpec hw_preset(const std::string& name) {
    sf_hw_spec h{};
    sparsefuse::check(sf_hw_preset(name.c_str(), &h));
    return {h.name, h.sm_num, h.smem_size, h.max_warp, h.element_bytes};
}

enum class KernelKind { RowWise, BlockWise };
inline const char* to_string(KernelKind k) { return k == KernelKind::RowWise ? "row_wise" : "block_wise"; }

struct KernelPlan {
    KernelKind kind = KernelKind::RowWise;
    int block_m = 0, block_n = 0, num_warps = 0;
    double score = 0.0;
    double threshold = std::numeric_limits<double>::quiet_NaN();
    bool fallback = false;
};

enum class PlanMode { Reference = SF_PLAN_REFERENCE, B200 = SF_PLAN_B200 };

constexpr int kMinBlock = 16;

inline double threshold(const DenseMask& mask, double tau = 1.2) {
    double t = 0.0;
    check(sf_threshold(mask.device_bits(), mask.seq_len(), tau, &t, nullptr));
    return t;
}

inline KernelPlan select_plan(const DenseMask& mask, const HardwareSpec& hw, std::int64_t seq_len, int h,
                              std::int64_t bs, int head_size, PlanMode mode = PlanMode::Reference) {
    hw.check();
    if (mask.seq_len() != seq_len) throw shape_error("mask seq_len differs from requested");
    const sf_hw_spec c = hw.to_c();
    sf_plan p{};
    check(sf_select_plan(mask.device_bits(), &c, seq_len, h, bs, head_size, static_cast<int32_t>(mode), &p, nullptr));
    KernelPlan k;
    k.kind = p.kind == SF_BLOCK_WISE ? KernelKind::BlockWise : KernelKind::RowWise;
    k.block_m = p.block_m; k.block_n = p.block_n; k.num_warps = p.num_warps;
    k.score = p.score; k.threshold = p.threshold; k.fallback = p.fallback != 0;
    return k;
}

// =============================================================================================
// Tensors (tensor.hpp:13-73) and the executors (attention.hpp:60-213, planner.hpp:165-172).
template <typename T>
struct Tensor4 {
    int bs = 0, h = 0, n = 0, d = 0;
    std::vector<T> v;
    Tensor4() = default;
    Tensor4(int bs_, int h_, int n_, int d_)
        : bs(bs_), h(h_), n(n_), d(d_), v(static_cast<std::size_t>(bs_) * h_ * n_ * d_, T(0)) {}
    T& at(int b, int hh, int i, int k) { return v[((static_cast<std::size_t>(b) * h + hh) * n + i) * d + k]; }
    const T& at(int b, int hh, int i, int k) const { return v[((static_cast<std::size_t>(b) * h + hh) * n + i) * d + k]; }
    template <typename U>
    Tensor4<U> cast() const {
        Tensor4<U> o(bs, h, n, d);
        for (std::size_t i = 0; i < v.size(); ++i) o.v[i] = static_cast<U>(v[i]);
        return o;
    }
};

template <typename T>
struct AttentionInput {
    Tensor4<T> q, k, v;
    int bs() const { return q.bs; }
    int h() const { return q.h; }
    int seq_len() const { return q.n; }
    int head_size() const { return q.d; }
    void check() const {
        auto same = [&](const Tensor4<T>& t) { return t.bs == q.bs && t.h == q.h && t.n == q.n && t.d == q.d; };
        if (!same(k) || !same(v)) throw shape_error("Q, K, V shapes differ");
        if (q.bs < 1 || q.h < 1 || q.n < 1 || q.d < 1) throw shape_error("empty attention input");
    }
};

template <typename T>
AttentionInput<T> random_attention_input(int bs, int h, int n, int d, std::uint64_t seed) {
    AttentionInput<T> in{Tensor4<T>(bs, h, n, d), Tensor4<T>(bs, h, n, d), Tensor4<T>(bs, h, n, d)};
    std::mt19937_64 rng(seed);
    for (Tensor4<T>* t : {&in.q, &in.k, &in.v})
        for (auto& x : t->v) x = static_cast<T>(2.0 * unit_real(rng) - 1.0);
    return in;
}

struct BlockExecStats {
    std::int64_t tiles_loaded = 0, full_tiles = 0, part_tiles = 0;
};

namespace detail {
// Host tensors -> device fp16 (bs, h, n, d) contiguous, run `launch`, device -> host.
template <typename TIn, typename TOut, typename F>
Tensor4<TOut> run_on_device(const AttentionInput<TIn>& in, F&& launch) {
    in.check();
    const std::size_t cnt = in.q.v.size();
    std::vector<__half> hq(cnt), hk(cnt), hv(cnt);
    for (std::size_t i = 0; i < cnt; ++i) {
        hq[i] = __float2half(static_cast<float>(in.q.v[i]));
        hk[i] = __float2half(static_cast<float>(in.k.v[i]));
        hv[i] = __float2half(static_cast<float>(in.v.v[i]));
    }
    DeviceBuffer<__half> q, k, v, o(cnt);
    q.upload(hq.data(), cnt); k.upload(hk.data(), cnt); v.upload(hv.data(), cnt);
    const int n = in.seq_len(), d = in.head_size();
    sf_attn_args a{in.bs(), in.h(), n, d, SF_F16, q.data(), k.data(), v.data(), o.data(),
                   static_cast<std::int64_t>(in.h()) * n * d, static_cast<std::int64_t>(n) * d, d,
                   static_cast<std::int64_t>(in.h()) * n * d, static_cast<std::int64_t>(n) * d, d, 0.f};
    launch(a);
    std::vector<__half> ho(cnt);
    o.download(ho.data(), cnt);
    Tensor4<TOut> out(in.bs(), in.h(), n, d);
    for (std::size_t i = 0; i < cnt; ++i) out.v[i] = static_cast<TOut>(__half2float(ho[i]));
    return out;
}
}  // namespace detail

// Device-resident entry points (sf_attn_args carries device pointers and strides).
inline void block_sparse_sdpa(const sf_attn_args& a, const BsrMask& bsr, const KernelPlan* plan = nullptr,
                              BlockExecStats* stats = nullptr, cudaStream_t st = nullptr) {
    if (!bsr.device) throw plan_error("BSR is not resident on the device (build it with build_bsr)");
    sf_plan p{};
    if (plan) {
        p.kind = plan->kind == KernelKind::BlockWise ? SF_BLOCK_WISE : SF_ROW_WISE;
        p.block_m = plan->block_m; p.block_n = plan->block_n; p.num_warps = plan->num_warps;
    }
    sf_attn_stats s{};
    check(sf_mha_blockwise(&a, &bsr.device->d, plan ? &p : nullptr, &s, st));
    if (stats) *stats = {s.tiles_loaded, s.full_tiles, s.part_tiles};
}
inline void rowwise_sdpa(const sf_attn_args& a, const RowwiseMask& rw, cudaStream_t st = nullptr) {
    if (!rw.device) throw plan_error("row-wise mask is not resident on the device (build it with build_rowwise)");
    check(sf_mha_rowwise(&a, &rw.device->d, st));
}

// Host-tensor entry points with the reference signatures (attention.hpp:71, :177; planner.hpp:165).
inline Tensor4<float> block_sparse_sdpa(const AttentionInput<float>& in, const BsrMask& bsr,
                                        BlockExecStats* stats = nullptr) {
    if (bsr.seq_len != in.seq_len()) throw shape_error("bsr seq_len differs from input");
    return detail::run_on_device<float, float>(in, [&](const sf_attn_args& a) { block_sparse_sdpa(a, bsr, nullptr, stats); });
}
inline Tensor4<float> block_sparse_sdpa(const AttentionInput<float>& in, const BsrMask& bsr, const KernelPlan& plan,
                                        BlockExecStats* stats = nullptr) {
    if (plan.kind != KernelKind::BlockWise) throw plan_error("plan does not select the block-wise kernel");
    if (plan.block_m != bsr.block_m || plan.block_n != bsr.block_n)
        throw plan_error("BSR block sizes do not match the active plan");
    return block_sparse_sdpa(in, bsr, stats);
}
inline Tensor4<double> rowwise_sdpa(const AttentionInput<double>& in, const RowwiseMask& rw) {
    if (rw.seq_len != in.seq_len()) throw shape_error("rowwise mask seq_len differs from input");
    return detail::run_on_device<double, double>(in, [&](const sf_attn_args& a) { rowwise_sdpa(a, rw); });
}

// dense_sdpa_oracle (attention.hpp:15-56): the dense masked SDPA on the device from the DENSE
// mask, fp64 accumulation and output. The inputs are rounded to fp16 on the way to the device,
// exactly as the sparse executors' inputs are, so the three legs of `attn verify` see the same
// values.
inline Tensor4<double> dense_sdpa_oracle(const AttentionInput<double>& in, const DenseMask& mask) {
    in.check();
    if (mask.seq_len() != in.seq_len()) throw shape_error("mask seq_len differs from input");
    const std::size_t cnt = in.q.v.size();
    std::vector<__half> hq(cnt), hk(cnt), hv(cnt);
    for (std::size_t i = 0; i < cnt; ++i) {
        hq[i] = __float2half(static_cast<float>(in.q.v[i]));
        hk[i] = __float2half(static_cast<float>(in.k.v[i]));
        hv[i] = __float2half(static_cast<float>(in.v.v[i]));
    }
    DeviceBuffer<__half> q, k, v;
    DeviceBuffer<double> o(cnt);
    q.upload(hq.data(), cnt); k.upload(hk.data(), cnt); v.upload(hv.data(), cnt);
    const int n = in.seq_len(), d = in.head_size();
    sf_attn_args a{in.bs(), in.h(), n, d, SF_F16, q.data(), k.data(), v.data(), nullptr,
                   static_cast<std::int64_t>(in.h()) * n * d, static_cast<std::int64_t>(n) * d, d,
                   static_cast<std::int64_t>(in.h()) * n * d, static_cast<std::int64_t>(n) * d, d, 0.f};
    a.o = o.data();  // not written (the fp64 output goes to o64); check_attn_args wants non-null
    check(sf_mha_dense_oracle(&a, mask.device_bits(), o.data(), nullptr));
    Tensor4<double> out(in.bs(), in.h(), n, d);
    o.download(out.v.data(), cnt);
    return out;
}

}  // namespace sparsefuse
