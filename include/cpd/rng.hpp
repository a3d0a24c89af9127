// SPDX-License-Identifier: Apache-2.0
// Drop-in for /root/reference/proj/include/cpd/rng.hpp (rng.hpp:15-70).
//
// Seeded generator whose draw order is part of every generator contract: the
// initial factors of cp_als_qr (solvers.hpp:116-122) must be bit-identical to
// the reference so trajectories can be compared sweep by sweep.  Algorithms
// (published, restated): splitmix64 state expansion, xoshiro256++ output,
// 53-bit uniforms, Marsaglia polar normals with the second variate cached.
// Host-only; the device generator (cpdb_tensor_synth) is counter-based.
#pragma once

#include <cmath>
#include <cstdint>

namespace cpd {

class Rng {
public:
    explicit Rng(std::uint64_t seed) {
        std::uint64_t x = seed;
        for (int i = 0; i < 4; ++i) s_[i] = splitmix(x);
    }

    std::uint64_t next_u64() {
        const std::uint64_t out = rot(s_[0] + s_[3], 23) + s_[0];
        const std::uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rot(s_[3], 45);
        return out;
    }

    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

    double normal() {
        if (cached_) {
            cached_ = false;
            return spare_;
        }
        for (;;) {
            const double u = 2.0 * uniform() - 1.0;
            const double v = 2.0 * uniform() - 1.0;
            const double s = u * u + v * v;
            if (s >= 1.0 || s == 0.0) continue;
            const double m = std::sqrt(-2.0 * std::log(s) / s);
            spare_ = v * m;
            cached_ = true;
            return u * m;
        }
    }

private:
    static std::uint64_t splitmix(std::uint64_t& x) {
        x += 0x9E3779B97F4A7C15ULL;
        std::uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    static std::uint64_t rot(std::uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

    std::uint64_t s_[4];
    double spare_ = 0.0;
    bool cached_ = false;
};

}  // namespace cpd
