// wrng_gpu/reference.hpp — the reference's Box-Muller and polar generators
// (/root/reference/proj/include/wrng/reference.hpp:9-36) on a host
// UniformState, computed in libwrng_gpu.so (glibc libm, FMA contraction off:
// the reference's bits).  The GPU baselines over many streams are
// wrng_gpu_method_fill (include/wrng_gpu.h).
#pragma once

#include <span>
#include <stdexcept>

#include "../wrng_gpu.h"
#include "uniform.hpp"

namespace wrng {

struct NormalPair {
    double x;
    double y;
};

/// reference.cpp:9-15; u1 must be in (0, 1).
inline NormalPair box_muller_pair(double u1, double u2) {
    NormalPair p;
    if (wrng_gpu_box_muller_pair(u1, u2, &p.x, &p.y) != WRNG_GPU_OK)
        throw std::invalid_argument("box_muller_pair: u1 must be in (0, 1)");
    return p;
}

/// reference.cpp:17-22 (a raw u1 of 0 becomes 2^-53).
inline NormalPair box_muller_next(UniformState& us) {
    NormalPair p;
    wrng_gpu_box_muller_next(us.c_state(), &p.x, &p.y);
    return p;
}

/// reference.cpp:24-29
inline NormalPair polar_transform(double v1, double v2) {
    NormalPair p;
    wrng_gpu_polar_transform(v1, v2, &p.x, &p.y);
    return p;
}

/// reference.cpp:31-37
inline NormalPair polar_next(UniformState& us) {
    NormalPair p;
    wrng_gpu_polar_next(us.c_state(), &p.x, &p.y);
    return p;
}

/// reference.cpp:53-63 (pairs in order; an odd count drops the last partner)
inline void box_muller_fill(UniformState& us, std::span<double> out, double mu = 0.0,
                            double sigma = 1.0) {
    wrng_gpu_normal_fill(0, us.c_state(), out.data(), out.size(), mu, sigma);
}
inline void polar_fill(UniformState& us, std::span<double> out, double mu = 0.0,
                       double sigma = 1.0) {
    wrng_gpu_normal_fill(1, us.c_state(), out.data(), out.size(), mu, sigma);
}

}  // namespace wrng
