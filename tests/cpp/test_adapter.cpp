// C++ drop-in check: the reference's WallaceState test scenarios
// (proj/tests/test_wallace_state.cpp, test_serialize.cpp) written against
// include/wrng_gpu/wallace.hpp, i.e. the GPU path behind the C ABI.
// Built and run by tests/test_cpp_adapter.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "wrng_gpu/wallace.hpp"

using namespace wrng;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (cond) {                                                              \
            ++g_pass;                                                            \
        } else {                                                                 \
            ++g_fail;                                                            \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
    do {                                                                         \
        bool thrown_ = false;                                                    \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (const type&) {                                                  \
            thrown_ = true;                                                      \
        }                                                                        \
        CHECK(thrown_);                                                          \
    } while (0)

static WallaceConfig config_with(std::uint32_t f, ScaleMode mode, std::uint64_t seed = 1) {
    WallaceConfig cfg;
    cfg.throwaway_f = f;
    cfg.scale_mode = mode;
    cfg.seed = seed;
    return cfg;
}

int main() {
    // golden values of the reference library:
    // n=2, N=2^12, f=1, seed 12345
    {
        WallaceConfig cfg;
        cfg.pool_exponent = 12;
        cfg.throwaway_f = 1;
        cfg.seed = 12345;
        WallaceState st(cfg);
        CHECK(st.active_pool().tracked_sumsq == 8236.360304807602);
        WallaceState tw(cfg);
        PassParams p = tw.advance_pass();
        CHECK(p.alpha == 3 && p.beta == 11 && p.gamma == 3948 && p.delta == 1318);
        CHECK(p.rot.c == -0.62552007586993019 && p.rot.s == 0.78020807140382553);
        CHECK(p.scale == 0.98980443003586394 && p.target_sumsq == 8069.2676960779772);
        auto v = st.fill(3);
        CHECK(v[0] == -1.6696392613832525 && v[1] == -0.67003755728398262 &&
              v[2] == 1.2961430635378857);
    }
    // n=2, N=2^20, f=2, seed 7 (C2 analogue)
    {
        WallaceConfig cfg;
        cfg.pool_exponent = 20;
        cfg.throwaway_f = 2;
        cfg.seed = 7;
        WallaceState st(cfg);
        auto v = st.fill(3);
        CHECK(v[0] == 0.1899777484759049 && v[1] == 1.3612423129263154 &&
              v[2] == -1.2808974468989538);
    }
    // config validation (test_wallace_state.cpp:23-32)
    {
        WallaceConfig cfg;
        cfg.pool_exponent = 7;
        CHECK_THROWS_AS(WallaceState{cfg}, std::invalid_argument);
        cfg.pool_exponent = 21;
        CHECK_THROWS_AS(WallaceState{cfg}, std::invalid_argument);
        cfg.pool_exponent = 10;
        cfg.throwaway_f = 0;
        CHECK_THROWS_AS(WallaceState{cfg}, std::invalid_argument);
    }
    // init pool: exact tracked sum, determinism, chi-squared band (34-47)
    {
        WallaceState a(config_with(3, ScaleMode::chisq));
        Pool pa = a.active_pool();
        CHECK(pa.tracked_sumsq == pa.direct_sumsq());
        CHECK(a.avail() == 0);
        WallaceState b(config_with(3, ScaleMode::chisq));
        Pool pb = b.active_pool();
        CHECK(pa.x == pb.x && pa.y == pb.y && pa.withheld == pb.withheld);
        CHECK(pa.tracked_sumsq > 1728.0 && pa.tracked_sumsq < 2368.0);
    }
    // refill exposes 2N-1 values and advances pass_count by f (49-58)
    for (std::uint32_t f : {1u, 3u}) {
        WallaceState st(config_with(f, ScaleMode::chisq));
        st.refill();
        CHECK(st.avail() == 2047);
        CHECK(st.pass_count() == f);
        st.refill();
        CHECK(st.pass_count() == 2 * f);
    }
    // chisq: post-refill sum of squares equals the target (60-67)
    {
        WallaceState st(config_with(3, ScaleMode::chisq));
        for (int i = 0; i < 20; ++i) {
            st.refill();
            Pool p = st.active_pool();
            CHECK(std::abs(p.direct_sumsq() / p.tracked_sumsq - 1.0) < 1e-9);
        }
    }
    // fill: count 0, sigma 0, sigma < 0 (69-81)
    {
        WallaceState st(config_with(3, ScaleMode::chisq));
        CHECK(st.fill(std::size_t{0}, 0.0, 1.0).empty());
        CHECK(st.numbers_emitted() == 0 && st.pass_count() == 0);
        auto sevens = st.fill(std::size_t{5}, 7.0, 0.0);
        for (double v : sevens) CHECK(v == 7.0);
        std::vector<double> buf(1);
        CHECK_THROWS_AS(st.fill(std::span<double>(buf), 0.0, -1.0), std::invalid_argument);
    }
    // mu / sigma at CLT precision (83-95)
    {
        WallaceState st(config_with(3, ScaleMode::chisq, 2));
        const std::size_t n = 1000000;
        auto v = st.fill(n, 5.0, 2.0);
        double s1 = 0.0;
        for (double z : v) s1 += z;
        double mean = s1 / double(n), s2 = 0.0;
        for (double z : v) s2 += (z - mean) * (z - mean);
        CHECK(std::abs(mean - 5.0) < 0.008);
        CHECK(std::abs(s2 / double(n) - 4.0) < 0.023);
    }
    // emission accounting across calls (97-109)
    {
        const std::uint64_t cap = 2047;
        for (std::uint64_t total : {std::uint64_t{1}, cap, cap + 1, 3 * cap + 5}) {
            WallaceState st(config_with(3, ScaleMode::chisq));
            std::uint64_t first = total / 2;
            st.fill(std::size_t(first), 0.0, 1.0);
            st.fill(std::size_t(total - first), 0.0, 1.0);
            CHECK(st.numbers_emitted() == total);
            CHECK(st.pass_count() / 3 == (total + cap - 1) / cap);
        }
    }
    // drift guard (128-150)
    {
        WallaceState st(config_with(3, ScaleMode::chisq));
        st.refill();
        Pool p = st.active_pool();
        p.x[17] += 1000.0;
        st.set_active_pool(p);
        CHECK_THROWS_AS(st.drift_check(), corrupted_state_error);

        WallaceState s2(config_with(3, ScaleMode::chisq));
        s2.refill();
        Pool q = s2.active_pool();
        double actual = q.direct_sumsq();
        q.tracked_sumsq = actual * (1.0 + 1e-5);
        s2.set_active_pool(q);
        s2.drift_check();
        CHECK(s2.active_pool().tracked_sumsq == actual);

        WallaceConfig cfg = config_with(3, ScaleMode::chisq);
        cfg.drift_check_period = 6;
        WallaceState g(cfg);
        g.refill();
        Pool r = g.active_pool();
        r.x[0] += 1000.0;
        g.set_active_pool(r);
        CHECK_THROWS_AS(g.refill(), corrupted_state_error);
    }
    // restart determinism (152-173)
    {
        WallaceConfig cfg = config_with(3, ScaleMode::chisq);
        cfg.restart_interval_passes = 100;
        WallaceState a(cfg), b(cfg);
        auto va = a.fill(300000, 0.0, 1.0);
        auto vb = b.fill(300000, 0.0, 1.0);
        CHECK(va == vb);
        CHECK(a.pass_count() > 300);
    }
    // persistence (test_serialize.cpp:19-41)
    {
        WallaceConfig cfg;
        cfg.seed = 1;
        WallaceState st(cfg);
        st.fill(3500, 0.0, 1.0);
        auto bytes = st.save_state();
        WallaceState loaded = WallaceState::load_state(bytes);
        CHECK(loaded.pass_count() == st.pass_count());
        CHECK(loaded.numbers_emitted() == st.numbers_emitted());
        CHECK(loaded.avail() == st.avail());
        auto a = st.fill(10000, 0.0, 1.0);
        auto b = loaded.fill(10000, 0.0, 1.0);
        CHECK(std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0);
        auto again = WallaceState::load_state(bytes).save_state();
        CHECK(bytes == again);
        auto bad = bytes;
        bad[0] ^= 0xFF;
        try {
            WallaceState::load_state(bad);
            CHECK(false);
        } catch (const malformed_state_error& e) {
            CHECK(e.kind() == state_error_kind::bad_magic);
        }
        try {
            WallaceState::load_state(std::span<const std::uint8_t>(bytes.data(), 73));
            CHECK(false);
        } catch (const malformed_state_error& e) {
            CHECK(e.kind() == state_error_kind::truncated);
        }
    }
    // n = 4 fp32 bank through the same adapter
    {
        WallaceConfig cfg;
        cfg.n_arrays = 4;
        cfg.fp32 = true;
        cfg.pools = 8;
        cfg.throwaway_f = 1;
        cfg.seed = 2024;
        WallaceState st(cfg);
        std::vector<float> v(8 * 10000);
        st.fill(std::span<float>(v));
        double s2 = 0.0;
        for (float z : v) s2 += double(z) * z;
        CHECK(std::abs(s2 / v.size() - 1.0) < 0.03);
        PassParams p = st.advance_pass();
        CHECK(p.strides[2] == 13 || p.strides[2] == 17);
        CHECK(p.variant <= 1);
    }
    // the mutable uniform_state() (wallace.hpp:158): draws made through it
    // advance the generator, as in the reference; copies are deep
    {
        WallaceState a(config_with(1, ScaleMode::chisq, 3)), b(config_with(1, ScaleMode::chisq, 3)),
            c(config_with(1, ScaleMode::chisq, 3));
        a.fill(5000);
        b.fill(5000);
        c.fill(5000);
        for (int i = 0; i < 3; ++i) {
            a.uniform_state().next_word();
            b.uniform_state().next_word();
        }
        CHECK(a.uniform_state().draws == c.uniform_state().draws);  // next_word is not a draw
        PassParams pa = a.advance_pass(), pb = b.advance_pass(), pc = c.advance_pass();
        CHECK(pa.gamma == pb.gamma && pa.delta == pb.delta && pa.rot.c == pb.rot.c);
        CHECK(pa.gamma != pc.gamma || pa.delta != pc.delta || pa.rot.c != pc.rot.c);
        WallaceState d = a;  // copy
        auto va = a.fill(3000);
        auto vd = d.fill(3000);
        CHECK(va == vd);
    }
    std::printf("adapter checks: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
