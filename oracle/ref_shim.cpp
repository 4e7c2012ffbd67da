// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (built from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libwrng_ref.so).  It lets the Python tests, the golden-vector
// dumper and bench.py's `--impl reference` arm drive the reference through its
// own public API (proj/include/wrng/*.hpp) without any C++ in Python.
//
// Exceptions never cross this boundary: every entry point maps them to the
// same status codes the product C ABI uses (include/wrng_gpu.h):
//   0 OK, 1 EINVAL (std::invalid_argument), 2 ECORRUPT
//   (wrng::corrupted_state_error), 3..6 EMALFORMED_{BAD_MAGIC, VERSION,
//   TRUNCATED, FIELD_RANGE} (wrng::malformed_state_error, errors.hpp:15-32).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "wrng/reference.hpp"
#include "wrng/stats.hpp"
#include "wrng/uniform.hpp"
#include "wrng/wallace.hpp"

using namespace wrng;

namespace {

int status_of(const std::exception_ptr& ep) {
    try {
        std::rethrow_exception(ep);
    } catch (const malformed_state_error& e) {
        switch (e.kind()) {
            case state_error_kind::bad_magic: return 3;
            case state_error_kind::unsupported_version: return 4;
            case state_error_kind::truncated: return 5;
            case state_error_kind::field_range: return 6;
        }
        return 6;
    } catch (const corrupted_state_error&) {
        return 2;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 99;
    }
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

}  // namespace

extern "C" {

// Mirrors PassParams (wallace.hpp:22-30) in a flat layout shared with the
// oracle / product params struct: stride[0..3], offset[0..3], variant, c, s,
// scale, target.  For n = 2: stride = {alpha, beta}, offset = {gamma, delta}.
struct ref_params {
    uint32_t stride[4];
    uint32_t offset[4];
    uint32_t variant;
    uint32_t pad_;
    double c;
    double s;
    double scale;
    double target;
};

static void to_flat(const PassParams& p, ref_params* o) {
    std::memset(o, 0, sizeof(*o));
    o->stride[0] = p.alpha;
    o->stride[1] = p.beta;
    o->offset[0] = p.gamma;
    o->offset[1] = p.delta;
    o->c = p.rot.c;
    o->s = p.rot.s;
    o->scale = p.scale;
    o->target = p.target_sumsq;
}

// ---- UniformState (uniform.hpp:16-40) -----------------------------------
void* ref_uniform_create(uint64_t seed, uint64_t stream) {
    return new UniformState(seed, stream);
}
void ref_uniform_destroy(void* u) { delete static_cast<UniformState*>(u); }
uint64_t ref_uniform_next_word(void* u) {
    return static_cast<UniformState*>(u)->next_word();
}
double ref_uniform_next_uniform(void* u) {
    return static_cast<UniformState*>(u)->next_uniform();
}
int ref_uniform_next_int_below(void* u, uint32_t m, uint32_t* out) {
    return guarded([&] { *out = static_cast<UniformState*>(u)->next_int_below(m); });
}
void ref_uniform_get(void* u, uint64_t* table, uint32_t* r, uint32_t* s,
                     uint64_t* draws) {
    auto* us = static_cast<UniformState*>(u);
    std::memcpy(table, us->lag_table.data(), sizeof(uint64_t) * 607);
    *r = us->cursor_r;
    *s = us->cursor_s;
    *draws = us->draws;
}
void ref_uniform_set(void* u, const uint64_t* table, uint32_t r, uint32_t s,
                     uint64_t draws) {
    auto* us = static_cast<UniformState*>(u);
    std::memcpy(us->lag_table.data(), table, sizeof(uint64_t) * 607);
    us->cursor_r = r;
    us->cursor_s = s;
    us->draws = draws;
}

// ---- free functions -----------------------------------------------------
double ref_chi2_target(double r, uint32_t nu) { return chi2_target(r, nu); }
void ref_rotation_from_t(double t, uint32_t region, double* c, double* s) {
    Rotation2 rot = rotation_from_t(t, region);
    *c = rot.c;
    *s = rot.s;
}
int ref_box_muller_pair(double u1, double u2, double* x, double* y) {
    return guarded([&] {
        NormalPair p = box_muller_pair(u1, u2);
        *x = p.x;
        *y = p.y;
    });
}
void ref_box_muller_fill(void* u, double* out, size_t n, double mu, double sigma) {
    box_muller_fill(*static_cast<UniformState*>(u), std::span<double>(out, n), mu,
                    sigma);
}
void ref_polar_fill(void* u, double* out, size_t n, double mu, double sigma) {
    polar_fill(*static_cast<UniformState*>(u), std::span<double>(out, n), mu, sigma);
}
// CPU timing of the reference's non-Wallace methods (main.cpp:287-312 loop):
// thread t fills per_thread values of UniformState(seed, t) in 64Ki calls.
double ref_bench_methods(int method, uint32_t threads, uint64_t per_thread, uint64_t seed) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (uint32_t t = 0; t < threads; ++t)
        th.emplace_back([=] {
            UniformState us(seed, t);
            std::vector<double> buf(1u << 16);
            double sink = 0.0;
            for (uint64_t done = 0; done < per_thread; done += buf.size()) {
                if (method == 0)
                    box_muller_fill(us, buf);
                else
                    polar_fill(us, buf);
                sink += buf[buf.size() / 2];
            }
            if (sink == 12345.678) std::abort();
        });
    for (auto& x : th) x.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
// select_pass_params on a caller-described pool (wallace.cpp:51-70).
int ref_select_pass_params(void* u, uint32_t n, double tracked, double withheld,
                           uint8_t mode, ref_params* out) {
    Pool pool;
    pool.x.assign(n, 0.0);
    pool.y.assign(n, 0.0);
    pool.tracked_sumsq = tracked;
    pool.withheld = withheld;
    return guarded([&] {
        PassParams p = select_pass_params(*static_cast<UniformState*>(u), pool,
                                          static_cast<ScaleMode>(mode));
        to_flat(p, out);
    });
}
// regenerate (wallace.cpp:113-137) on caller arrays.
int ref_regenerate(uint32_t n, const double* sx, const double* sy, double* dx,
                   double* dy, const ref_params* prm, double* dst_tracked,
                   double* dst_withheld) {
    return guarded([&] {
        Pool src, dst;
        src.x.assign(sx, sx + n);
        src.y.assign(sy, sy + n);
        dst.x.assign(n, 0.0);
        dst.y.assign(n, 0.0);
        PassParams p{prm->stride[0], prm->stride[1], prm->offset[0], prm->offset[1],
                     {prm->c, prm->s}, prm->scale, prm->target};
        regenerate(src, dst, p);
        std::memcpy(dx, dst.x.data(), n * sizeof(double));
        std::memcpy(dy, dst.y.data(), n * sizeof(double));
        *dst_tracked = dst.tracked_sumsq;
        *dst_withheld = dst.withheld;
    });
}
int ref_moments(const double* v, size_t n, double* out7) {
    return guarded([&] {
        MomentsReport m = moments(std::span<const double>(v, n));
        out7[0] = double(m.n);
        out7[1] = m.m1;
        out7[2] = m.m2;
        out7[3] = m.m4;
        out7[4] = m.z1;
        out7[5] = m.z2;
        out7[6] = m.z4;
    });
}

// ---- uniformity / serial-correlation checks (stats.cpp:10-38, 40-127) ----
// u/v chi-squared exactly as the CLI's uniformity test builds it
// (tools/main.cpp:160-193): pairs (v[2i], v[2i+1]), to_uv, chi2_bins.
int ref_uv_chi2(const double* v, size_t n, uint32_t k, double* out6) {
    return guarded([&] {
        constexpr double kPi2 = 1.5707963267948966;
        std::vector<double> us, vs;
        for (size_t i = 0; i + 1 < n; i += 2) {
            UvPair q = to_uv(v[i], v[i + 1]);
            if (q.skip) continue;
            us.push_back(q.u);
            vs.push_back(q.v);
        }
        Chi2Report a = chi2_bins(us, k, 0.0, 1.0);
        Chi2Report b = chi2_bins(vs, k, -kPi2, kPi2);
        out6[0] = a.statistic;
        out6[1] = a.p_value;
        out6[2] = b.statistic;
        out6[3] = b.p_value;
        out6[4] = double(a.sample_count);
        out6[5] = double(a.dof);
    });
}
int ref_chi2_sf(double statistic, uint32_t dof, double* out) {
    return guarded([&] { *out = chi2_sf(statistic, dof); });
}
int ref_autocorr(const double* v, size_t n, size_t lag, double* out) {
    return guarded([&] { *out = autocorr_at_lag(std::span<const double>(v, n), lag).r; });
}

// ---- WallaceState (wallace.hpp:113-174) --------------------------------
int ref_state_create(uint32_t pool_exponent, uint32_t f, uint8_t mode,
                     uint64_t restart, uint64_t drift, uint64_t seed,
                     uint64_t stream, void** out) {
    *out = nullptr;
    return guarded([&] {
        WallaceConfig cfg;
        cfg.pool_exponent = pool_exponent;
        cfg.throwaway_f = f;
        cfg.scale_mode = static_cast<ScaleMode>(mode);
        cfg.restart_interval_passes = restart;
        cfg.drift_check_period = drift;
        cfg.seed = seed;
        cfg.stream_id = stream;
        *out = new WallaceState(cfg);
    });
}
void ref_state_destroy(void* st) { delete static_cast<WallaceState*>(st); }
int ref_state_fill(void* st, double* out, size_t count, double mu, double sigma) {
    return guarded([&] {
        static_cast<WallaceState*>(st)->fill(std::span<double>(out, count), mu, sigma);
    });
}
int ref_state_advance_pass(void* st, ref_params* out) {
    return guarded([&] { to_flat(static_cast<WallaceState*>(st)->advance_pass(), out); });
}
int ref_state_refill(void* st) {
    return guarded([&] { static_cast<WallaceState*>(st)->refill(); });
}
int ref_state_drift_check(void* st) {
    return guarded([&] { static_cast<WallaceState*>(st)->drift_check(); });
}
void ref_state_restart(void* st) { static_cast<WallaceState*>(st)->restart(); }
// counters: pass_count, numbers_emitted, avail, pool_size
void ref_state_counters(void* st, uint64_t* out4) {
    auto* s = static_cast<WallaceState*>(st);
    out4[0] = s->pass_count();
    out4[1] = s->numbers_emitted();
    out4[2] = s->avail();
    out4[3] = s->pool_size();
}
// Active pool: x[N], y[N], {tracked, withheld}.
void ref_state_get_pool(void* st, double* x, double* y, double* tw) {
    const Pool& p = static_cast<WallaceState*>(st)->active_pool();
    std::memcpy(x, p.x.data(), p.x.size() * sizeof(double));
    std::memcpy(y, p.y.data(), p.y.size() * sizeof(double));
    tw[0] = p.tracked_sumsq;
    tw[1] = p.withheld;
}
void ref_state_set_pool(void* st, const double* x, const double* y,
                        const double* tw) {
    Pool& p = static_cast<WallaceState*>(st)->active_pool();
    std::memcpy(p.x.data(), x, p.x.size() * sizeof(double));
    std::memcpy(p.y.data(), y, p.y.size() * sizeof(double));
    p.tracked_sumsq = tw[0];
    p.withheld = tw[1];
}
void ref_state_uniform(void* st, uint64_t* table, uint32_t* r, uint32_t* s,
                       uint64_t* draws) {
    ref_uniform_get(&static_cast<WallaceState*>(st)->uniform_state(), table, r, s,
                    draws);
}
// save_state (serialize.cpp:82-113): returns the byte count; copies at most cap.
size_t ref_state_save(void* st, uint8_t* buf, size_t cap) {
    auto bytes = static_cast<WallaceState*>(st)->save_state();
    if (buf) std::memcpy(buf, bytes.data(), bytes.size() < cap ? bytes.size() : cap);
    return bytes.size();
}
int ref_state_load(const uint8_t* buf, size_t n, void** out) {
    *out = nullptr;
    return guarded([&] {
        *out = new WallaceState(
            WallaceState::load_state(std::span<const uint8_t>(buf, n)));
    });
}

// ---- CPU baseline: the reference's own bench loop (main.cpp:287-312) over
// `threads` host threads, thread t owning WallaceState{seed, stream0 + t}.
// Each thread fills `per_thread` values in chunks of `chunk` doubles.
// Returns wall seconds.
double ref_bench_threads(uint32_t pool_exponent, uint32_t f, uint8_t mode,
                         uint64_t seed, uint64_t stream0, uint32_t threads,
                         uint64_t per_thread, uint32_t chunk) {
    std::vector<WallaceState> states;
    states.reserve(threads);
    for (uint32_t t = 0; t < threads; ++t) {
        WallaceConfig cfg;
        cfg.pool_exponent = pool_exponent;
        cfg.throwaway_f = f;
        cfg.scale_mode = static_cast<ScaleMode>(mode);
        cfg.seed = seed;
        cfg.stream_id = stream0 + t;
        states.emplace_back(cfg);
    }
    std::vector<double> sinks(threads, 0.0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ws;
    for (uint32_t t = 0; t < threads; ++t) {
        ws.emplace_back([&, t] {
            std::vector<double> buf(chunk);
            uint64_t done = 0;
            double sink = 0.0;
            while (done < per_thread) {
                uint64_t take = per_thread - done < chunk ? per_thread - done : chunk;
                states[t].fill(std::span<double>(buf.data(), take), 0.0, 1.0);
                sink += buf[take / 2];
                done += take;
            }
            sinks[t] = sink;
        });
    }
    for (auto& w : ws) w.join();
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
}

// ---- the same threads filling one large host array: thread t fills its
// own contiguous segment out[t * per_thread, (t + 1) * per_thread) with one
// fill(span) call per `chunk` values, so every normal lands in memory (the
// shape of bench.py's workload and of its host-output e2e leg).
double ref_bench_array(uint32_t pool_exponent, uint32_t f, uint8_t mode, uint64_t seed,
                       uint64_t stream0, uint32_t threads, uint64_t per_thread,
                       uint64_t chunk, double* out) {
    std::vector<WallaceState> states;
    states.reserve(threads);
    for (uint32_t t = 0; t < threads; ++t) {
        WallaceConfig cfg;
        cfg.pool_exponent = pool_exponent;
        cfg.throwaway_f = f;
        cfg.scale_mode = static_cast<ScaleMode>(mode);
        cfg.seed = seed;
        cfg.stream_id = stream0 + t;
        states.emplace_back(cfg);
    }
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ws;
    for (uint32_t t = 0; t < threads; ++t) {
        ws.emplace_back([&, t] {
            double* seg = out + (uint64_t)t * per_thread;
            for (uint64_t done = 0; done < per_thread;) {
                const uint64_t take = per_thread - done < chunk ? per_thread - done : chunk;
                states[t].fill(std::span<double>(seg + done, take), 0.0, 1.0);
                done += take;
            }
        });
    }
    for (auto& w : ws) w.join();
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
