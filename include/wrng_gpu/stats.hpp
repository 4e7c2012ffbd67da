// wrng_gpu/stats.hpp — the reference's statistics on host spans
// (/root/reference/proj/include/wrng/stats.hpp:11-68), same sequential
// order and results, computed in libwrng_gpu.so.  MomentsReport adds m3
// (BASELINE's four moments) after the reference's fields.  For samples that
// live on the GPU see wrng_gpu_validate / wrng_gpu_moments_* (device
// reductions, including Anderson-Darling).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <utility>

#include "../wrng_gpu.h"
#include "wallace.hpp"

namespace wrng {

struct Chi2Report {
    double statistic;
    std::uint32_t dof;
    double p_value;
    std::uint32_t bin_count;
    std::size_t sample_count;
};

struct MomentsReport {
    std::size_t n;
    double m1;
    double m2;
    double m4;
    double z1;
    double z2;
    double z4;
    double m3 = 0.0;  ///< B200 extension: third moment
};

struct AutocorrReport {
    std::size_t lag;
    double r;
    std::size_t n;
};

struct UvPair {
    double u;
    double v;
    bool skip;
};

/// stats.cpp:10-16
inline UvPair to_uv(double x, double y) {
    UvPair p;
    std::int32_t skip = 0;
    wrng_gpu_to_uv(x, y, &p.u, &p.v, &skip);
    p.skip = skip != 0;
    return p;
}

/// stats.cpp:40-87
inline double chi2_sf(double statistic, std::uint32_t dof) {
    if (statistic < 0.0 || dof < 1)
        throw std::invalid_argument("chi2_sf: need statistic >= 0, dof >= 1");
    return wrng_gpu_chi2_sf(statistic, dof);
}

/// stats.cpp:18-38
inline Chi2Report chi2_bins(std::span<const double> values, std::uint32_t k, double lo,
                            double hi) {
    if (k < 2) throw std::invalid_argument("chi2_bins: need at least 2 bins");
    if (!(lo < hi)) throw std::invalid_argument("chi2_bins: lo must be < hi");
    double st = 0.0;
    if (wrng_gpu_chi2_bins(values.data(), values.size(), k, lo, hi, &st) != WRNG_GPU_OK)
        throw std::invalid_argument("chi2_bins: value out of [lo, hi]");
    return {st, k - 1, chi2_sf(st, k - 1), k, values.size()};
}

/// stats.cpp:89-108 (+ m3)
inline MomentsReport moments(std::span<const double> values) {
    if (values.empty()) throw std::invalid_argument("moments: empty input");
    double o[7];
    wrng_gpu_moments_host(values.data(), values.size(), o);
    MomentsReport r{values.size(), o[0], o[1], o[3], o[4], o[5], o[6]};
    r.m3 = o[2];
    return r;
}

/// stats.cpp:110-127
inline AutocorrReport autocorr_at_lag(std::span<const double> values, std::size_t lag) {
    if (values.size() < lag + 2)
        throw std::invalid_argument("autocorr_at_lag: need n > lag + 1");
    double r = 0.0;
    if (wrng_gpu_autocorr_host(values.data(), values.size(), lag, &r) != WRNG_GPU_OK)
        throw std::invalid_argument("autocorr_at_lag: zero-variance input");
    return {lag, r, values.size() - lag};
}

/// stats.cpp:129-146: advance `passes` passes recording each chi-squared
/// target; (sample mean, population variance).  Each pass runs on the GPU.
inline std::pair<double, double> sumsq_distribution_check(WallaceState& state,
                                                          std::uint64_t passes) {
    if (state.config().scale_mode != ScaleMode::chisq)
        throw std::invalid_argument("sumsq_distribution_check: state must be in chisq mode");
    if (passes == 0) throw std::invalid_argument("sumsq_distribution_check: passes >= 1");
    std::vector<double> s(passes);
    for (std::uint64_t i = 0; i < passes; ++i) s[i] = state.advance_pass().target_sumsq;
    double mv[2];
    wrng_gpu_target_stats(s.data(), passes, mv);
    return {mv[0], mv[1]};
}

}  // namespace wrng
