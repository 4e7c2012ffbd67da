// wrng_gpu/wallace.hpp — header-only C++ drop-in for the reference generator
// interface (/root/reference/proj/include/wrng/wallace.hpp), running on the
// B200 through the C ABI in wrng_gpu.h.
//
// A reference caller switches by putting include/wrng_gpu/compat first on its
// include path (so "wrng/wallace.hpp" resolves here) and linking
// libwrng_gpu.so instead of libwrng.a; no source changes.
// Names, argument meaning and exception types are the reference's:
//   Rotation2, PassParams, Pool{x, y, tracked_sumsq, withheld,
//     direct_sumsq(), max_abs()}, ScaleMode, WallaceConfig, Segment ... wallace.hpp:14-75
//   chi2_target, rotation_from_uniform, rotation_from_t,
//     select_pass_params, plan_segments, regenerate .................. wallace.hpp:77-111
//   WallaceState(const WallaceConfig&) ..... wallace.hpp:116-119 (validation
//                                            wallace.cpp:141-149 -> invalid_argument)
//   advance_pass, refill, fill(span), fill(count), drift_check, restart,
//   save_state, load_state, config, pool_size, pass_count,
//   numbers_emitted, avail, active_pool ............................... wallace.hpp:121-160
//   pool_stream_flawed, pool_stream_default ........................... wallace.hpp:176-191
//   errors ........................................ wrng_gpu/errors.hpp (errors.hpp)
//   UniformState .................................. wrng_gpu/uniform.hpp (uniform.hpp)
// Where the reference's semantics need the pool on the host, the drop-in
// keeps them with a host view of the device pool:
//   * active_pool() returns a reference to a host copy of the live pool,
//     taken on first use after the pool changed; edits made through it
//     (tests model a caller scribbling over the work area,
//     test_wallace_state.cpp:128-150) are written back to the device before
//     the next operation.  A reference held across a later operation keeps
//     the older contents (the reference's would alias the other buffer).
//   * uniform_state() is likewise a host view of the device generator;
//     draws made through it are written back before the next operation.
//   * WallaceState is copyable (a deep copy through save_state/load_state).
// Free functions on value-type pools run regenerate on the GPU
// (wrng_gpu_regenerate) and the scalar parts in libwrng_gpu.so, built with
// FMA contraction off so the bits match the reference's default build
// whatever flags the caller uses.
// The initial pool and restarts use the host glibc Box-Muller, exactly
// init_pool (wallace.cpp:158-167), unless WallaceConfig::device_init is set,
// so a default-constructed drop-in reproduces the reference bit for bit.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../wrng_gpu.h"
#include "errors.hpp"
#include "uniform.hpp"

namespace wrng {

/// GPU used by the free functions on value-type pools (regenerate); a
/// WallaceState uses WallaceConfig::device.
inline std::int32_t free_function_device = 0;

struct Rotation2 {
    double c;
    double s;
};

struct PassParams {
    std::uint32_t alpha;
    std::uint32_t beta;
    std::uint32_t gamma;
    std::uint32_t delta;
    Rotation2 rot;
    double scale;
    double target_sumsq;
    // n = 4 extension (docs/n4_spec.md): all strides/offsets and the variant
    std::array<std::uint32_t, 4> strides{};
    std::array<std::uint32_t, 4> offsets{};
    std::uint32_t variant = 0;
};

/// The pool: x, y as in the reference (wallace.hpp:36-50); `more` holds
/// arrays 2 and 3 of an n = 4 pool (empty for the reference's n = 2).
struct Pool {
    std::vector<double> x;
    std::vector<double> y;
    double tracked_sumsq = 0.0;
    double withheld = 0.0;
    std::vector<std::vector<double>> more;

    std::uint32_t n() const { return static_cast<std::uint32_t>(x.size()); }
    std::uint32_t n_arrays() const { return 2u + static_cast<std::uint32_t>(more.size()); }
    const std::vector<double>& array(std::uint32_t m) const {
        return m == 0 ? x : m == 1 ? y : more.at(m - 2);
    }
    std::vector<double>& array(std::uint32_t m) { return m == 0 ? x : m == 1 ? y : more.at(m - 2); }

    /// x then y (then arrays 2, 3), left to right (wallace.cpp:13-18).
    double direct_sumsq() const {
        double q = 0.0;
        for (std::uint32_t m = 0; m < n_arrays(); ++m)
            q = wrng_gpu_sumsq_continue(q, array(m).data(), array(m).size());
        return q;
    }
    /// Largest |value| over all arrays (wallace.cpp:20-25).
    double max_abs() const {
        double mx = 0.0;
        for (std::uint32_t m = 0; m < n_arrays(); ++m)
            for (double v : array(m)) mx = std::max(mx, std::abs(v));
        return mx;
    }
};

enum class ScaleMode : std::uint8_t { chisq = 0, fixed = 1 };

struct WallaceConfig {
    std::uint32_t pool_exponent = 10;
    std::uint32_t throwaway_f = 3;
    ScaleMode scale_mode = ScaleMode::chisq;
    std::uint64_t restart_interval_passes = 0;
    std::uint64_t drift_check_period = 64;
    std::uint64_t seed = 0;
    std::uint64_t stream_id = 0;
    // ---- B200 extensions (defaults = the reference's generator) ----
    std::uint32_t n_arrays = 2;    ///< 2 or 4
    bool fp32 = false;             ///< fp32 pools
    std::uint32_t pools = 1;       ///< independent pools, pool p = stream_id + p
    std::int32_t device = 0;
    bool device_init = false;      ///< Box-Muller on the device (a few ulp off glibc)
    bool force_hbm = false;        ///< HBM-resident engine
};

struct Segment {
    std::uint32_t low;
    std::uint32_t high;
    std::int64_t jx;
    std::int64_t jy;
};

namespace detail {
inline void check(wrng_gpu_status s, const wrng_gpu_t* g, const char* what) {
    if (s == WRNG_GPU_OK) return;
    std::string msg = std::string(what) + (g ? std::string(": ") + wrng_gpu_last_error(g) : "");
    switch (s) {
        case WRNG_GPU_EINVAL: throw std::invalid_argument(msg);
        case WRNG_GPU_ECORRUPT: throw corrupted_state_error(msg);
        case WRNG_GPU_EMALFORMED_BAD_MAGIC:
            throw malformed_state_error(state_error_kind::bad_magic, msg);
        case WRNG_GPU_EMALFORMED_VERSION:
            throw malformed_state_error(state_error_kind::unsupported_version, msg);
        case WRNG_GPU_EMALFORMED_TRUNCATED:
            throw malformed_state_error(state_error_kind::truncated, msg);
        case WRNG_GPU_EMALFORMED_FIELD_RANGE:
            throw malformed_state_error(state_error_kind::field_range, msg);
        default: throw device_error(msg + " (status " + std::to_string(int(s)) + ")");
    }
}

inline wrng_gpu_params to_c(const PassParams& p, std::uint32_t n_arrays) {
    wrng_gpu_params c{};
    if (n_arrays == 2) {
        c.stride[0] = p.alpha;
        c.stride[1] = p.beta;
        c.offset[0] = p.gamma;
        c.offset[1] = p.delta;
    } else {
        for (int m = 0; m < 4; ++m) {
            c.stride[m] = p.strides[m];
            c.offset[m] = p.offsets[m];
        }
        c.variant = p.variant;
    }
    c.c = p.rot.c;
    c.s = p.rot.s;
    c.scale = p.scale;
    c.target_sumsq = p.target_sumsq;
    return c;
}

inline PassParams from_c(const wrng_gpu_params& c) {
    PassParams p{c.stride[0], c.stride[1], c.offset[0], c.offset[1], {c.c, c.s}, c.scale,
                 c.target_sumsq};
    for (int m = 0; m < 4; ++m) {
        p.strides[m] = c.stride[m];
        p.offsets[m] = c.offset[m];
    }
    p.variant = c.variant;
    return p;
}

inline bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() &&
           (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0);
}
inline bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }
}  // namespace detail

// ---- free functions (wallace.hpp:77-111) ------------------------------------

/// S = (r + sqrt(2 nu - 1))^2 / 2 (wallace.cpp:27-31).
inline double chi2_target(double r, std::uint32_t nu) { return wrng_gpu_chi2_target(r, nu); }

/// (cos, sin) from t = tan(theta/2) and a sign region (wallace.cpp:33-42).
inline Rotation2 rotation_from_t(double t, std::uint32_t region) {
    Rotation2 r;
    wrng_gpu_rotation_from_t(t, region, &r.c, &r.s);
    return r;
}

/// One uniform, then next_int_below(3) (wallace.cpp:44-49).
inline Rotation2 rotation_from_uniform(UniformState& us) {
    Rotation2 r;
    wrng_gpu_rotation_from_uniform(us.c_state(), &r.c, &r.s);
    return r;
}

/// wallace.cpp:51-70 (n = 4 pools: docs/n4_spec.md §2).  Throws
/// corrupted_state_error after the draws when tracked_sumsq is not > 0.
inline PassParams select_pass_params(UniformState& us, const Pool& pool, ScaleMode mode) {
    wrng_gpu_params c{};
    const wrng_gpu_status s =
        wrng_gpu_select_pass_params(us.c_state(), pool.n_arrays(), pool.n(),
                                    static_cast<std::uint32_t>(mode), pool.tracked_sumsq,
                                    pool.withheld, &c);
    if (s == WRNG_GPU_ECORRUPT)
        throw corrupted_state_error("select_pass_params: tracked sum of squares is not positive");
    detail::check(s, nullptr, "select_pass_params");
    return detail::from_c(c);
}

/// wallace.cpp:72-111 (the GPU kernels index with (a*j + g) & (N-1) instead;
/// kept for callers of the reference's API).
inline std::vector<Segment> plan_segments(const PassParams& params, std::uint32_t n) {
    const wrng_gpu_params c = detail::to_c(params, 2);
    std::uint32_t count = 0;
    detail::check(wrng_gpu_plan_segments(&c, n, nullptr, 0, &count), nullptr, "plan_segments");
    std::vector<wrng_gpu_segment> raw(count);
    detail::check(wrng_gpu_plan_segments(&c, n, raw.data(), count, &count), nullptr,
                  "plan_segments");
    std::vector<Segment> out;
    out.reserve(count);
    for (const wrng_gpu_segment& s : raw) out.push_back({s.low, s.high, s.jx, s.jy});
    return out;
}

/// One pass src -> dst on the GPU (wallace.cpp:113-137): dst gets the new
/// arrays, tracked_sumsq = params.target_sumsq, withheld = its last value.
inline void regenerate(const Pool& src, Pool& dst, const PassParams& params) {
    const std::uint32_t n = src.n(), na = src.n_arrays();
    std::vector<double> in(std::size_t(na) * n), out(std::size_t(na) * n);
    for (std::uint32_t m = 0; m < na; ++m) {
        if (src.array(m).size() != n) throw std::invalid_argument("regenerate: ragged pool");
        std::copy(src.array(m).begin(), src.array(m).end(), in.begin() + std::size_t(m) * n);
    }
    const wrng_gpu_params c = detail::to_c(params, na);
    double withheld = 0.0;
    detail::check(wrng_gpu_regenerate(in.data(), out.data(), na, n, &c, &withheld,
                                      free_function_device),
                  nullptr, "regenerate");
    dst.more.resize(na - 2);
    for (std::uint32_t m = 0; m < na; ++m)
        dst.array(m).assign(out.begin() + std::size_t(m) * n, out.begin() + std::size_t(m + 1) * n);
    dst.tracked_sumsq = params.target_sumsq;
    dst.withheld = withheld;
}

// ---- the generator (wallace.hpp:113-174) -----------------------------------

class WallaceState {
public:
    explicit WallaceState(const WallaceConfig& config) : cfg_(config) {
        wrng_gpu_config c = to_c(config);
        detail::check(wrng_gpu_create(&c, &g_), nullptr, "WallaceState");
    }
    WallaceState(const WallaceState& o) : cfg_(o.cfg_) {
        const std::vector<std::uint8_t> b = o.save_state();
        detail::check(wrng_gpu_import_state(b.data(), b.size(), cfg_.device, flags(cfg_), &g_),
                      nullptr, "WallaceState(copy)");
    }
    WallaceState& operator=(const WallaceState& o) {
        if (this != &o) *this = WallaceState(o);
        return *this;
    }
    WallaceState(WallaceState&& o) noexcept
        : g_(o.g_), cfg_(o.cfg_), view_(std::move(o.view_)), shadow_(std::move(o.shadow_)),
          view_valid_(o.view_valid_), lent_(o.lent_), uview_(o.uview_), ushadow_(o.ushadow_),
          uview_valid_(o.uview_valid_), ulent_(o.ulent_) {
        o.g_ = nullptr;
        o.view_valid_ = o.lent_ = o.uview_valid_ = o.ulent_ = false;
    }
    WallaceState& operator=(WallaceState&& o) noexcept {
        if (this != &o) {
            wrng_gpu_destroy(g_);
            g_ = o.g_;
            cfg_ = o.cfg_;
            view_ = std::move(o.view_);
            shadow_ = std::move(o.shadow_);
            view_valid_ = o.view_valid_;
            lent_ = o.lent_;
            uview_ = o.uview_;
            ushadow_ = o.ushadow_;
            uview_valid_ = o.uview_valid_;
            ulent_ = o.ulent_;
            o.g_ = nullptr;
            o.view_valid_ = o.lent_ = o.uview_valid_ = o.ulent_ = false;
        }
        return *this;
    }
    ~WallaceState() { wrng_gpu_destroy(g_); }

    PassParams advance_pass() {
        begin_op();
        std::vector<wrng_gpu_params> p(cfg_.pools);
        detail::check(wrng_gpu_advance_pass(g_, p.data()), g_, "advance_pass");
        return detail::from_c(p[0]);
    }
    void refill() {
        begin_op();
        detail::check(wrng_gpu_refill(g_), g_, "refill");
    }
    void fill(std::span<double> out, double mu = 0.0, double sigma = 1.0) {
        begin_op();
        detail::check(wrng_gpu_fill_f64(g_, out.data(), out.size(), mu, sigma, 0, nullptr), g_,
                      "fill");
    }
    void fill(std::span<float> out, double mu = 0.0, double sigma = 1.0) {
        begin_op();
        detail::check(wrng_gpu_fill_f32(g_, out.data(), out.size(), mu, sigma, 0, nullptr), g_,
                      "fill");
    }
    std::vector<double> fill(std::size_t count, double mu = 0.0, double sigma = 1.0) {
        std::vector<double> v(count);
        fill(std::span<double>(v), mu, sigma);
        return v;
    }
    /// Device output, enqueued on a CUDA stream (cudaStream_t as void*).
    void fill_device(double* dev, std::size_t count, double mu, double sigma, void* stream) {
        begin_op();
        detail::check(wrng_gpu_fill_f64(g_, dev, count, mu, sigma, 1, stream), g_, "fill");
    }
    void fill_device(float* dev, std::size_t count, double mu, double sigma, void* stream) {
        begin_op();
        detail::check(wrng_gpu_fill_f32(g_, dev, count, mu, sigma, 1, stream), g_, "fill");
    }
    void drift_check() {
        begin_op();
        detail::check(wrng_gpu_drift_check(g_), g_, "drift_check");
    }
    void restart() {
        begin_op();
        detail::check(wrng_gpu_restart(g_), g_, "restart");
    }
    void synchronize() { detail::check(wrng_gpu_synchronize(g_), g_, "synchronize"); }
    /// GPU extension: generate `count` values (advancing like fill(count))
    /// and check them on the device (wrng_gpu_validate).
    wrng_gpu_validation validate(std::uint64_t count, std::uint32_t k = 1000,
                                 std::uint64_t lag = 1) {
        begin_op();
        wrng_gpu_validation v{};
        detail::check(wrng_gpu_validate(g_, count, k, lag, nullptr, nullptr, &v), g_,
                      "validate");
        return v;
    }

    std::vector<std::uint8_t> save_state() const {
        flush();
        std::size_t n = 0;
        detail::check(wrng_gpu_export_state(g_, nullptr, 0, &n), g_, "save_state");
        std::vector<std::uint8_t> b(n);
        detail::check(wrng_gpu_export_state(g_, b.data(), b.size(), &n), g_, "save_state");
        return b;
    }
    /// serialize.cpp:115-169.  `config` supplies the handle-only settings the
    /// bytes do not carry (device, device_init, force_hbm).
    static WallaceState load_state(std::span<const std::uint8_t> bytes,
                                   const WallaceConfig& config = WallaceConfig{}) {
        wrng_gpu_t* g = nullptr;
        detail::check(wrng_gpu_import_state(bytes.data(), bytes.size(), config.device,
                                            flags(config), &g),
                      nullptr, "load_state");
        wrng_gpu_config c;
        wrng_gpu_get_config(g, &c);
        WallaceConfig cfg = config;
        cfg.pool_exponent = c.pool_exponent;
        cfg.throwaway_f = c.throwaway_f;
        cfg.scale_mode = static_cast<ScaleMode>(c.scale_mode);
        cfg.restart_interval_passes = c.restart_interval_passes;
        cfg.drift_check_period = c.drift_check_period;
        cfg.seed = c.seed;
        cfg.stream_id = c.stream_id;
        cfg.n_arrays = c.n_arrays;
        cfg.fp32 = c.dtype == WRNG_GPU_F32;
        cfg.pools = c.pools;
        return WallaceState(g, cfg);
    }

    static WallaceState load_state(std::span<const std::uint8_t> bytes, std::int32_t device) {
        WallaceConfig c;
        c.device = device;
        return load_state(bytes, c);
    }

    const WallaceConfig& config() const { return cfg_; }
    std::uint32_t pool_size() const { return 1u << cfg_.pool_exponent; }
    std::uint64_t pass_count() const { return counters().pass_count; }
    std::uint64_t numbers_emitted() const { return counters().numbers_emitted; }
    std::uint64_t avail() const { return counters().avail; }

    /// The live pool (pool 0 of a bank) as a host view; edits are written
    /// back before the next operation (see the header comment).
    Pool& active_pool() {
        refresh_view();
        if (!lent_) {
            shadow_ = view_;
            lent_ = true;
        }
        return view_;
    }
    const Pool& active_pool() const {
        refresh_view();
        return view_;
    }
    /// Snapshot of pool `pool` of a bank.
    Pool active_pool(std::uint32_t pool) const {
        if (pool == 0) return active_pool();
        Pool p;
        read_pool(pool, p);
        return p;
    }
    /// Writes a pool back as the live pool of `pool`.
    void set_active_pool(const Pool& p, std::uint32_t pool = 0) {
        begin_op();
        const std::uint32_t n = pool_size(), na = cfg_.n_arrays;
        if (p.n_arrays() != na) throw std::invalid_argument("set_active_pool: wrong array count");
        std::vector<double> v(std::size_t(na) * n);
        for (std::uint32_t m = 0; m < na; ++m) {
            if (p.array(m).size() != n) throw std::invalid_argument("set_active_pool: wrong size");
            std::copy(p.array(m).begin(), p.array(m).end(), v.begin() + std::size_t(m) * n);
        }
        detail::check(wrng_gpu_write_pool(g_, pool, v.data(), p.tracked_sumsq, p.withheld), g_,
                      "set_active_pool");
    }
    /// The live uniform generator (of pool 0) as a host view, like
    /// active_pool(): draws made through it are written back to the device
    /// before the next operation (wallace.hpp:158).
    UniformState& uniform_state() {
        refresh_uview();
        if (!ulent_) {
            ushadow_ = uview_;
            ulent_ = true;
        }
        return uview_;
    }
    const UniformState& uniform_state() const {
        refresh_uview();
        return uview_;
    }
    /// Snapshot of pool `pool`'s uniform generator (banks).
    UniformState uniform_state(std::uint32_t pool) const {
        flush();
        UniformState u;
        read_uniform(pool, u);
        return u;
    }
    wrng_gpu_t* handle() const { return g_; }

private:
    WallaceState(wrng_gpu_t* g, const WallaceConfig& c) : g_(g), cfg_(c) {}

    static std::uint32_t flags(const WallaceConfig& c) {
        return (c.device_init ? 0u : (unsigned)WRNG_GPU_INIT_HOST) |
               (c.force_hbm ? (unsigned)WRNG_GPU_FORCE_HBM : 0u);
    }
    static wrng_gpu_config to_c(const WallaceConfig& config) {
        wrng_gpu_config c;
        wrng_gpu_config_default(&c);
        c.pool_exponent = config.pool_exponent;
        c.throwaway_f = config.throwaway_f;
        c.scale_mode = static_cast<std::uint32_t>(config.scale_mode);
        c.restart_interval_passes = config.restart_interval_passes;
        c.drift_check_period = config.drift_check_period;
        c.seed = config.seed;
        c.stream_id = config.stream_id;
        c.n_arrays = config.n_arrays;
        c.dtype = config.fp32 ? WRNG_GPU_F32 : WRNG_GPU_F64;
        c.pools = config.pools;
        c.device = config.device;
        c.flags = flags(config);
        return c;
    }
    wrng_gpu_counters counters() const {
        wrng_gpu_counters c;
        detail::check(wrng_gpu_get_counters(g_, 0, &c), g_, "counters");
        return c;
    }
    void read_pool(std::uint32_t pool, Pool& p) const {
        const std::uint32_t n = pool_size(), na = cfg_.n_arrays;
        std::vector<double> v(std::size_t(na) * n);
        detail::check(wrng_gpu_read_pool(g_, pool, v.data(), &p.tracked_sumsq, &p.withheld), g_,
                      "active_pool");
        p.more.resize(na - 2);
        for (std::uint32_t m = 0; m < na; ++m)
            p.array(m).assign(v.begin() + std::size_t(m) * n, v.begin() + std::size_t(m + 1) * n);
    }
    void read_uniform(std::uint32_t pool, UniformState& u) const {
        detail::check(wrng_gpu_read_uniform(g_, pool, u.lag_table.data(), &u.cursor_r,
                                            &u.cursor_s, &u.draws),
                      g_, "uniform_state");
        u.seed = cfg_.seed;
        u.stream_id = cfg_.stream_id + pool;
    }
    void refresh_uview() const {
        if (uview_valid_) return;
        read_uniform(0, uview_);
        uview_valid_ = true;
        ulent_ = false;
    }
    void refresh_view() const {
        if (view_valid_) return;
        read_pool(0, view_);
        view_valid_ = true;
        lent_ = false;
    }
    /// Writes back edits made through active_pool() / uniform_state()
    /// since they were read.
    void flush() const {
        if (ulent_) {
            ulent_ = false;
            if (std::memcmp(&uview_, &ushadow_, sizeof(UniformState)) != 0)
                detail::check(wrng_gpu_write_uniform(g_, 0, uview_.lag_table.data(),
                                                     uview_.cursor_r, uview_.cursor_s,
                                                     uview_.draws),
                              g_, "uniform_state (write back)");
        }
        if (!lent_) return;
        lent_ = false;
        bool same = view_.n_arrays() == shadow_.n_arrays() &&
                    detail::same_bits(view_.tracked_sumsq, shadow_.tracked_sumsq) &&
                    detail::same_bits(view_.withheld, shadow_.withheld);
        for (std::uint32_t m = 0; same && m < view_.n_arrays(); ++m)
            same = detail::same_bits(view_.array(m), shadow_.array(m));
        if (same) return;
        const std::uint32_t n = pool_size(), na = cfg_.n_arrays;
        if (view_.n_arrays() != na)
            throw std::invalid_argument("active_pool: array count changed");
        std::vector<double> v(std::size_t(na) * n);
        for (std::uint32_t m = 0; m < na; ++m) {
            if (view_.array(m).size() != n) throw std::invalid_argument("active_pool: resized");
            std::copy(view_.array(m).begin(), view_.array(m).end(),
                      v.begin() + std::size_t(m) * n);
        }
        detail::check(wrng_gpu_write_pool(g_, 0, v.data(), view_.tracked_sumsq, view_.withheld),
                      g_, "active_pool (write back)");
    }
    /// Before an operation that may change the pool: write back edits, then
    /// drop the view.
    void begin_op() {
        flush();
        view_valid_ = false;
        uview_valid_ = false;
    }

    wrng_gpu_t* g_ = nullptr;
    WallaceConfig cfg_;
    mutable Pool view_;
    mutable Pool shadow_;
    mutable bool view_valid_ = false;
    mutable bool lent_ = false;
    mutable UniformState uview_{};
    mutable UniformState ushadow_{};
    mutable bool uview_valid_ = false;
    mutable bool ulent_ = false;
};

// ---- diagnostic pool streams (wallace.hpp:176-191; wallace.cpp:238-291) ----

/// The discouraged unit-stride scheme: alpha = beta = 1, gamma = delta
/// fixed, rotation fixed at pi/6, scale 1; the pool contents x then y after
/// each pass, concatenated.
inline std::vector<double> pool_stream_flawed(std::uint64_t seed, std::uint64_t stream_id,
                                              std::uint32_t pool_exponent, std::uint32_t gamma,
                                              std::size_t count) {
    WallaceConfig cfg;
    cfg.pool_exponent = pool_exponent;
    cfg.throwaway_f = 1;
    cfg.scale_mode = ScaleMode::fixed;
    cfg.seed = seed;
    cfg.stream_id = stream_id;
    WallaceState st(cfg);
    const std::uint32_t n = st.pool_size();
    if (gamma >= n) throw std::invalid_argument("pool_stream_flawed: gamma must be in [0, N)");
    const double cos_pi6 = 0.86602540378443865, sin_pi6 = 0.5;
    std::vector<double> out;
    out.reserve(count + 2 * std::size_t(n));
    Pool cur = std::as_const(st).active_pool();
    Pool next = cur;
    while (out.size() < count) {
        const PassParams p{1, 1, gamma, gamma, {cos_pi6, sin_pi6}, 1.0, cur.tracked_sumsq};
        regenerate(cur, next, p);
        std::swap(cur, next);
        out.insert(out.end(), cur.x.begin(), cur.x.end());
        out.insert(out.end(), cur.y.begin(), cur.y.end());
    }
    out.resize(count);
    return out;
}

/// Recommended parameters redrawn every pass (chisq mode): the pool
/// contents x then y after each advance_pass, concatenated.
inline std::vector<double> pool_stream_default(std::uint64_t seed, std::uint64_t stream_id,
                                               std::uint32_t pool_exponent, std::size_t count) {
    WallaceConfig cfg;
    cfg.pool_exponent = pool_exponent;
    cfg.seed = seed;
    cfg.stream_id = stream_id;
    WallaceState st(cfg);
    std::vector<double> out;
    out.reserve(count + 2 * std::size_t(st.pool_size()));
    while (out.size() < count) {
        st.advance_pass();
        const Pool& pool = std::as_const(st).active_pool();
        out.insert(out.end(), pool.x.begin(), pool.x.end());
        out.insert(out.end(), pool.y.begin(), pool.y.end());
    }
    out.resize(count);
    return out;
}

}  // namespace wrng
