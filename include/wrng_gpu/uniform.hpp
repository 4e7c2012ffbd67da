// wrng_gpu/uniform.hpp — the reference's uniform generator
// (/root/reference/proj/include/wrng/uniform.hpp:16-40): additive lagged
// Fibonacci, lags (607, 273), mod 2^64, splitmix64 seeding.
//
// A host value type for callers that draw their own parameters (the pools
// of WallaceState keep their generators in device memory, see
// WallaceState::uniform_state()).  Seeding runs in libwrng_gpu.so
// (wrng_gpu_uniform_seed); the per-word recurrence is integer-only and
// inline.  The layout equals the C struct wrng_gpu_uniform.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <stdexcept>

#include "../wrng_gpu.h"

namespace wrng {

struct UniformState {
    static constexpr std::uint32_t kTableSize = 607;
    static constexpr std::uint32_t kShortLag = 273;
    static constexpr std::uint32_t kMaxIntBound = 1u << 20;

    std::array<std::uint64_t, kTableSize> lag_table{};
    std::uint32_t cursor_r = 0;
    std::uint32_t cursor_s = kTableSize - kShortLag;
    std::uint64_t seed = 0;
    std::uint64_t stream_id = 0;
    std::uint64_t draws = 0;

    UniformState() : UniformState(0, 0) {}
    /// uniform.cpp:23-32: splitmix64(seed ^ rotl(stream_id, 32)), 6070
    /// warm-up words, draws = 0.
    UniformState(std::uint64_t seed_in, std::uint64_t stream_in) {
        wrng_gpu_uniform_seed(c_state(), seed_in, stream_in);
    }

    /// uniform.cpp:34-40
    std::uint64_t next_word() {
        const std::uint64_t w = lag_table[cursor_r] + lag_table[cursor_s];
        lag_table[cursor_r] = w;
        if (++cursor_r == kTableSize) cursor_r = 0;
        if (++cursor_s == kTableSize) cursor_s = 0;
        return w;
    }
    /// uniform.cpp:42-45: top 53 bits * 2^-53 (exact)
    double next_uniform() {
        ++draws;
        return static_cast<double>(next_word() >> 11) * 0x1.0p-53;
    }
    /// uniform.cpp:47-51
    std::uint32_t next_int_below(std::uint32_t m) {
        if (m < 1 || m > kMaxIntBound)
            throw std::invalid_argument("next_int_below: m must be in [1, 2^20]");
        return static_cast<std::uint32_t>(next_uniform() * m);
    }

    wrng_gpu_uniform* c_state() { return reinterpret_cast<wrng_gpu_uniform*>(this); }
};

static_assert(sizeof(UniformState) == sizeof(wrng_gpu_uniform), "layout of wrng_gpu_uniform");
static_assert(offsetof(UniformState, cursor_r) == offsetof(wrng_gpu_uniform, cursor_r), "layout");
static_assert(offsetof(UniformState, draws) == offsetof(wrng_gpu_uniform, draws), "layout");

}  // namespace wrng
