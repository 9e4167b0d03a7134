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
// Two phases, so that the kernel can read X and build the planes before its PDL wait (X is the
// caller's input, not written by the previous kernels of the chain) and only store them after it
// (Xt may still be read by the previous contraction in the stream).
template <int SX>
struct SlicePlanes {
    uint32_t w[SX][4];
    size_t dst;              // byte offset of plane 0's 16-byte chunk; plane i at + i RT 128
    bool bad;                // a value >= 2^ell
};

template <int SX, int RT, typename T = uint32_t>
__device__ __forceinline__ SlicePlanes<SX> slice_load(const T* __restrict__ X, uint32_t k, uint32_t m, uint32_t KB,
                                                      uint32_t ell, uint32_t idx, int check) {
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
    SlicePlanes<SX> sp;
    sp.bad = false;
    if (check && ell < 8 * sizeof(T)) {
        T bad = 0;
#pragma unroll
        for (int u = 0; u < 16; u++) bad |= (v[u] >> ell);
        sp.bad = bad != 0;
    }
    const uint32_t mt = alpha / RT, r = alpha % RT;
#pragma unroll
    for (int i = 0; i < SX; i++) {
#pragma unroll
        for (int q = 0; q < 4; q++)
            sp.w[i][q] = ((v[4 * q] >> (8 * i)) & 0xFF) | (((v[4 * q + 1] >> (8 * i)) & 0xFF) << 8) |
                         (((v[4 * q + 2] >> (8 * i)) & 0xFF) << 16) | (((v[4 * q + 3] >> (8 * i)) & 0xFF) << 24);
    }
    sp.dst = ((((size_t)mt * KB + kb) * SX) * RT) * kBK + swz_off(r, c16);
    return sp;
}

template <int SX, int RT>
__device__ __forceinline__ void slice_store(const SlicePlanes<SX>& sp, uint8_t* __restrict__ Xt, uint32_t* flag) {
    if (sp.bad) atomicOr(flag, 1u);
#pragma unroll
    for (int i = 0; i < SX; i++)
        *reinterpret_cast<uint4*>(Xt + sp.dst + (size_t)i * RT * kBK) =
            make_uint4(sp.w[i][0], sp.w[i][1], sp.w[i][2], sp.w[i][3]);
}

}  // namespace nimbus
