// wrng_gpu/wallace.hpp — header-only C++ drop-in for the reference generator
// interface (/root/reference/proj/include/wrng/wallace.hpp + errors.hpp),
// running on the B200 through the C ABI in wrng_gpu.h.
//
// A reference caller switches by including this header instead of
// "wrng/wallace.hpp" and linking libwrng_gpu.so instead of libwrng.a.  Names,
// argument meaning and exception types are the reference's:
//   WallaceConfig fields/defaults ........ wallace.hpp:57-65 (+ GPU extensions)
//   WallaceState(const WallaceConfig&) ... wallace.hpp:116-119 (validation
//                                          wallace.cpp:141-149 -> invalid_argument)
//   fill(span<double>, mu, sigma) ........ wallace.hpp:130-133
//   fill(count, mu, sigma) -> vector ..... wallace.hpp:134-135
//   advance_pass() -> PassParams ......... wallace.hpp:121-124
//   refill(), drift_check(), restart() ... wallace.hpp:126-145
//   save_state(), load_state(bytes) ...... wallace.hpp:147-148 ("WRNG" v1 bytes)
//   config(), pool_size(), pass_count(), numbers_emitted(), avail(),
//   active_pool(), uniform_state() ...... wallace.hpp:150-158
//   corrupted_state_error / malformed_state_error{kind} ... errors.hpp:10-32
// Differences, all forced by the pool living in device memory:
//   * active_pool() returns a snapshot (copy); write it back with
//     set_active_pool().  UniformState likewise is a snapshot.
//   * WallaceState is move-only (the reference's is copyable).
// The initial pool is filled on the host (glibc Box-Muller, exactly
// init_pool, wallace.cpp:158-167) unless WallaceConfig::device_init is set,
// so a default-constructed drop-in reproduces the reference bit for bit.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "wrng_gpu.h"

namespace wrng {

class corrupted_state_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

enum class state_error_kind { bad_magic, unsupported_version, truncated, field_range };

class malformed_state_error : public std::runtime_error {
public:
    malformed_state_error(state_error_kind kind, const std::string& what)
        : std::runtime_error(what), kind_(kind) {}
    state_error_kind kind() const noexcept { return kind_; }

private:
    state_error_kind kind_;
};

/// B200 device error (no reference analogue).
class device_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

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

/// Snapshot of the live pool.  x and y are arrays 0 and 1; `arrays` holds
/// all n arrays (n = 4 mode) in order.
struct Pool {
    std::vector<double> x;
    std::vector<double> y;
    std::vector<std::vector<double>> arrays;
    double tracked_sumsq = 0.0;
    double withheld = 0.0;

    std::uint32_t n() const { return static_cast<std::uint32_t>(x.size()); }
    double direct_sumsq() const {
        double q = 0.0;
        for (const auto& a : arrays)
            for (double v : a) q += v * v;
        return q;
    }
};

struct UniformState {
    std::array<std::uint64_t, 607> lag_table{};
    std::uint32_t cursor_r = 0;
    std::uint32_t cursor_s = 0;
    std::uint64_t draws = 0;
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
}  // namespace detail

class WallaceState {
public:
    explicit WallaceState(const WallaceConfig& config) : cfg_(config) {
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
        c.flags = (config.device_init ? 0u : (unsigned)WRNG_GPU_INIT_HOST) |
                  (config.force_hbm ? (unsigned)WRNG_GPU_FORCE_HBM : 0u);
        detail::check(wrng_gpu_create(&c, &g_), nullptr, "WallaceState");
    }
    WallaceState(WallaceState&& o) noexcept : g_(o.g_), cfg_(o.cfg_) { o.g_ = nullptr; }
    WallaceState& operator=(WallaceState&& o) noexcept {
        if (this != &o) {
            wrng_gpu_destroy(g_);
            g_ = o.g_;
            cfg_ = o.cfg_;
            o.g_ = nullptr;
        }
        return *this;
    }
    WallaceState(const WallaceState&) = delete;
    WallaceState& operator=(const WallaceState&) = delete;
    ~WallaceState() { wrng_gpu_destroy(g_); }

    PassParams advance_pass() {
        std::vector<wrng_gpu_params> p(cfg_.pools);
        detail::check(wrng_gpu_advance_pass(g_, p.data()), g_, "advance_pass");
        PassParams out{p[0].stride[0], p[0].stride[1], p[0].offset[0], p[0].offset[1],
                       {p[0].c, p[0].s}, p[0].scale, p[0].target_sumsq};
        for (int m = 0; m < 4; ++m) {
            out.strides[m] = p[0].stride[m];
            out.offsets[m] = p[0].offset[m];
        }
        out.variant = p[0].variant;
        return out;
    }
    void refill() { detail::check(wrng_gpu_refill(g_), g_, "refill"); }
    void fill(std::span<double> out, double mu = 0.0, double sigma = 1.0) {
        detail::check(wrng_gpu_fill_f64(g_, out.data(), out.size(), mu, sigma, 0, nullptr), g_,
                      "fill");
    }
    void fill(std::span<float> out, double mu = 0.0, double sigma = 1.0) {
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
        detail::check(wrng_gpu_fill_f64(g_, dev, count, mu, sigma, 1, stream), g_, "fill");
    }
    void fill_device(float* dev, std::size_t count, double mu, double sigma, void* stream) {
        detail::check(wrng_gpu_fill_f32(g_, dev, count, mu, sigma, 1, stream), g_, "fill");
    }
    void drift_check() { detail::check(wrng_gpu_drift_check(g_), g_, "drift_check"); }
    void restart() { detail::check(wrng_gpu_restart(g_), g_, "restart"); }
    void synchronize() { detail::check(wrng_gpu_synchronize(g_), g_, "synchronize"); }
    /// GPU extension: generate `count` values (advancing like fill(count))
    /// and check them on the device (wrng_gpu_validate).
    wrng_gpu_validation validate(std::uint64_t count, std::uint32_t k = 1000,
                                 std::uint64_t lag = 1) {
        wrng_gpu_validation v{};
        detail::check(wrng_gpu_validate(g_, count, k, lag, nullptr, nullptr, &v), g_,
                      "validate");
        return v;
    }

    std::vector<std::uint8_t> save_state() const {
        std::size_t n = 0;
        detail::check(wrng_gpu_export_state(g_, nullptr, 0, &n), g_, "save_state");
        std::vector<std::uint8_t> b(n);
        detail::check(wrng_gpu_export_state(g_, b.data(), b.size(), &n), g_, "save_state");
        return b;
    }
    static WallaceState load_state(std::span<const std::uint8_t> bytes, std::int32_t device = 0) {
        wrng_gpu_t* g = nullptr;
        detail::check(wrng_gpu_import_state(bytes.data(), bytes.size(), device, 0, &g), nullptr,
                      "load_state");
        wrng_gpu_config c;
        wrng_gpu_get_config(g, &c);
        WallaceConfig cfg;
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
        cfg.device = device;
        return WallaceState(g, cfg);
    }

    const WallaceConfig& config() const { return cfg_; }
    std::uint32_t pool_size() const { return 1u << cfg_.pool_exponent; }
    std::uint64_t pass_count() const { return counters().pass_count; }
    std::uint64_t numbers_emitted() const { return counters().numbers_emitted; }
    std::uint64_t avail() const { return counters().avail; }

    Pool active_pool(std::uint32_t pool = 0) const {
        const std::uint32_t n = pool_size(), na = cfg_.n_arrays;
        std::vector<double> v(std::size_t(na) * n);
        Pool p;
        detail::check(wrng_gpu_read_pool(g_, pool, v.data(), &p.tracked_sumsq, &p.withheld), g_,
                      "active_pool");
        for (std::uint32_t m = 0; m < na; ++m)
            p.arrays.emplace_back(v.begin() + std::size_t(m) * n,
                                  v.begin() + std::size_t(m + 1) * n);
        p.x = p.arrays[0];
        p.y = p.arrays[1];
        return p;
    }
    /// Writes a (modified) snapshot back as the live pool.  x and y win over
    /// arrays[0..1] when they were edited.
    void set_active_pool(const Pool& p, std::uint32_t pool = 0) {
        const std::uint32_t n = pool_size(), na = cfg_.n_arrays;
        std::vector<double> v(std::size_t(na) * n);
        for (std::uint32_t m = 0; m < na; ++m) {
            const std::vector<double>& src =
                m == 0 ? p.x : m == 1 ? p.y : p.arrays.at(m);
            std::copy(src.begin(), src.end(), v.begin() + std::size_t(m) * n);
        }
        detail::check(wrng_gpu_write_pool(g_, pool, v.data(), p.tracked_sumsq, p.withheld), g_,
                      "set_active_pool");
    }
    UniformState uniform_state(std::uint32_t pool = 0) const {
        UniformState u;
        detail::check(wrng_gpu_read_uniform(g_, pool, u.lag_table.data(), &u.cursor_r,
                                            &u.cursor_s, &u.draws),
                      g_, "uniform_state");
        return u;
    }
    wrng_gpu_t* handle() const { return g_; }

private:
    WallaceState(wrng_gpu_t* g, const WallaceConfig& c) : g_(g), cfg_(c) {}
    wrng_gpu_counters counters() const {
        wrng_gpu_counters c;
        detail::check(wrng_gpu_get_counters(g_, 0, &c), g_, "counters");
        return c;
    }
    wrng_gpu_t* g_ = nullptr;
    WallaceConfig cfg_;
};

}  // namespace wrng
