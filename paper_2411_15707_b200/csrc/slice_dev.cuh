// slice_dev.cuh -- device code of K4 (X -> 8-bit planes in the swizzled tcgen05
// operand layout), the per-item body of k_slice_x (layout.cu).
#pragma once
#include "internal.h"

namespace nimbus {

__device__ __forceinline__ uint32_t swz_off(uint32_t r, uint32_t chunk) {
    return r * 128u + ((chunk ^ (r & 7u)) << 4);
}

// ---------------------------------------------------------------- K4 slice X
// X[alpha][beta] = sum_i x_i 2^(8i) (unsigned representative)
// Xt[mt][kb][i][RT rows][128 B] (RT = 128; 64 / 32 for the transposed ell = 32 /
// ell = 64 kernel), zero padded to whole tiles.  T = uint32_t, or uint64_t for
// ell > 32 (S_x = 8 slices).
template <int SX, int RT, typename T = uint32_t>
__device__ __forceinline__ void slice_item(const T* __restrict__ X, uint32_t k, uint32_t m, uint32_t KB,
                                           uint32_t ell, uint8_t* __restrict__ Xt, uint32_t idx, uint32_t* flag,
                                           int check) {
    const uint32_t alpha = idx / (KB * 8), ch = idx % (KB * 8);
    const uint32_t kb = ch >> 3, c16 = ch & 7;
    const uint32_t beta0 = kb * kBK + c16 * 16;
    T v[16];
    if (sizeof(T) == 4 && alpha < k && beta0 + 16 <= m && (m & 3) == 0) {
        const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)alpha * m + beta0);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint4 w = __ldg(src + q);
            v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
        }
    } else {
#pragma unroll
        for (int u = 0; u < 16; u++)
            v[u] = (alpha < k && beta0 + u < m) ? X[(size_t)alpha * m + beta0 + u] : (T)0;
    }
    if (check && ell < 8 * sizeof(T)) {
        T bad = 0;
#pragma unroll
        for (int u = 0; u < 16; u++) bad |= (v[u] >> ell);
        if (bad) atomicOr(flag, 1u);
    }
    const uint32_t mt = alpha / RT, r = alpha % RT;
#pragma unroll
    for (int i = 0; i < SX; i++) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; q++)
            w[q] = ((v[4 * q] >> (8 * i)) & 0xFF) | (((v[4 * q + 1] >> (8 * i)) & 0xFF) << 8) |
                   (((v[4 * q + 2] >> (8 * i)) & 0xFF) << 16) | (((v[4 * q + 3] >> (8 * i)) & 0xFF) << 24);
        uint8_t* dst = Xt + ((((size_t)mt * KB + kb) * SX + i) * RT) * kBK + swz_off(r, c16);
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

}  // namespace nimbus
