// pyexact.hpp — IEEE-754 helpers that reproduce Python numeric semantics.
//
// The reference decision layer is Python; to be bit-exact the core must
// reproduce (1) int/int true division, which Python rounds correctly for
// arbitrarily large ints, and (2) int-vs-float comparison, which Python
// performs exactly (no int->double rounding). Everything else the reference
// does is plain double arithmetic, which C++ reproduces when compiled with
// -ffp-contract=off and without -ffast-math.
#pragma once

#include <cmath>
#include <cstdint>

namespace gmx {

using u128 = unsigned __int128;

inline int bit_length(u128 v) {
    const uint64_t hi = (uint64_t)(v >> 64), lo = (uint64_t)v;
    if (hi) return 128 - __builtin_clzll(hi);
    if (lo) return 64 - __builtin_clzll(lo);
    return 0;
}

// Correctly rounded (round-half-even) num/den for num >= 0, den > 0, both
// < 2^126. Equals CPython's long_true_divide for non-negative operands.
inline double true_div(u128 num, u128 den) {
    if (num == 0) return 0.0;
    const u128 exact = (u128)1 << 53;
    if (num < exact && den < exact) return (double)(uint64_t)num / (double)(uint64_t)den;
    // Long division producing at least 55 significant quotient bits + sticky.
    u128 q = num / den, r = num % den;
    int exp2 = 0;
    while (q < ((u128)1 << 55)) {
        r <<= 1;
        q <<= 1;
        if (r >= den) { r -= den; q |= 1; }
        --exp2;
    }
    const bool sticky = r != 0;
    const int drop = bit_length(q) - 53;
    u128 kept = q >> drop;
    const u128 rem = q & (((u128)1 << drop) - 1);
    const u128 half = (u128)1 << (drop - 1);
    if (rem > half || (rem == half && (sticky || (kept & 1)))) ++kept;
    return std::ldexp((double)(uint64_t)kept, exp2 + drop);
}

inline double true_div(int64_t a, int64_t b) { return true_div((u128)a, (u128)b); }

// Python `a >= x` for int a and float x (exact, no rounding of a).
inline bool int_ge_float(int64_t a, double x) {
    if (std::isnan(x)) return false;
    if (x >= 9223372036854775808.0) return false;
    if (x < -9223372036854775808.0) return true;
    return a >= (int64_t)std::ceil(x);
}

// Python math.ceil(float) -> int, and int(float) (truncation).
inline int64_t py_ceil(double x) { return (int64_t)std::ceil(x); }
inline int64_t py_trunc(double x) { return (int64_t)std::trunc(x); }

// SplitMix64 (gpumux/rng.py:19-42): same constants, 53-bit uniforms.
struct SplitMix64 {
    uint64_t state;
    uint64_t next() {
        state += 0x9E3779B97F4A7C15ull;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform(double lo, double hi) {
        const uint64_t u = next() >> 11;
        return lo + (hi - lo) * ((double)u * 0x1.0p-53);
    }
};

}  // namespace gmx
