// GF(2) jump-ahead of the xorshift64* stream (proj/include/hsaw/prng.hpp:41-48). The state update
// is linear over GF(2): the state after p steps is M^p * state for a 64x64 bit matrix M, so any
// stream position is reachable with a handful of matrix-vector products from precomputed powers
// of M. Host side: the algebra (powers, products); device side: byte-sliced tables, 8 lookups per
// product. Shared by the forward simulation (simulate.cu) and the R-MAT generator (rmat.cu).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace hsawgpu {

// ---- GF(2) algebra of the xorshift64* state step (host) -----------------------------------------
struct Mat64 {
    uint64_t col[64];  // col[j] = image of the unit vector e_j
};

inline uint64_t xs_step(uint64_t x) {  // prng.hpp:42-46 (state update only)
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return x;
}
inline uint64_t mat_apply(const Mat64& a, uint64_t s) {
    uint64_t y = 0;
    while (s) {
        y ^= a.col[__builtin_ctzll(s)];
        s &= s - 1;
    }
    return y;
}
inline Mat64 mat_mul(const Mat64& a, const Mat64& b) {  // a * b (apply b first)
    Mat64 r;
    for (int j = 0; j < 64; ++j) r.col[j] = mat_apply(a, b.col[j]);
    return r;
}
inline Mat64 mat_identity() {
    Mat64 r;
    for (int j = 0; j < 64; ++j) r.col[j] = 1ull << j;
    return r;
}

struct JumpAlgebra {
    Mat64 pow2[64];  // M^(2^j)
    JumpAlgebra() {
        for (int j = 0; j < 64; ++j) pow2[0].col[j] = xs_step(1ull << j);
        for (int j = 1; j < 64; ++j) pow2[j] = mat_mul(pow2[j - 1], pow2[j - 1]);
    }
    Mat64 power(uint64_t e) const {
        Mat64 r = mat_identity();
        for (int j = 0; e; ++j, e >>= 1)
            if (e & 1) r = mat_mul(pow2[j], r);
        return r;
    }
    uint64_t jump(uint64_t state, uint64_t steps) const {
        for (int j = 0; steps; ++j, steps >>= 1)
            if (steps & 1) state = mat_apply(pow2[j], state);
        return state;
    }
};
inline const JumpAlgebra& algebra() {
    static const JumpAlgebra a;
    return a;
}

// Byte-sliced form of a matrix: y = XOR_b tab[b][byte b of s]. 8 * 256 u64 = 16 KB per matrix.
constexpr int kTabWords = 8 * 256;
inline void slice_matrix(const Mat64& a, uint64_t* tab) {
    for (int b = 0; b < 8; ++b)
        for (int x = 0; x < 256; ++x) {
            uint64_t y = 0;
            for (int j = 0; j < 8; ++j)
                if (x >> j & 1) y ^= a.col[8 * b + j];
            tab[b * 256 + x] = y;
        }
}

__device__ __forceinline__ uint64_t tab_apply(const uint64_t* __restrict__ tab, uint64_t s) {
    uint64_t y = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) y ^= __ldg(tab + b * 256 + ((s >> (8 * b)) & 0xFF));
    return y;
}

}  // namespace hsawgpu
