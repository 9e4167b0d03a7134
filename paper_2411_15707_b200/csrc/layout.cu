// layout.cu -- data-layout and epilogue kernels of the COP hot path:
//   K4  slice X into 8-bit planes in the tcgen05 operand layout (A3)
//   tile / untile Enc(W) between the canonical [beta][comp][limb][j] layout
//       and the resident byte-plane kernel layout (setup / export)
//   K7  RShift packing + mod-switch + mask (A5, A6; Alg. 1 steps 3-4)
//
// Kernel layout of a byte-plane tile: a 2-D block of
// R rows x 128 bytes, row r at offset r*128, the 16-byte chunk c of row r
// stored at chunk position c ^ (r & 7) -- the 128-byte swizzle that the
// tcgen05 shared-memory descriptor (SWIZZLE_128B, K-major) expects, applied
// once at rest so that one linear bulk copy lands a ready-to-use operand tile.
#include "internal.h"

namespace nimbus {

__device__ __forceinline__ uint32_t swz_off(uint32_t r, uint32_t chunk) {
    return r * 128u + ((chunk ^ (r & 7u)) << 4);
}

// ---------------------------------------------------------------- K4 slice X
// X[alpha][beta] = sum_i x_i 2^(8i) (unsigned representative)
// Xt[mt][kb][i][128 rows][128 B], zero padded to whole tiles.
template <int SX>
__global__ void k_slice_x(const uint32_t* __restrict__ X, uint32_t k, uint32_t m, uint32_t KB, uint32_t ell,
                          uint8_t* __restrict__ Xt, uint32_t total, uint32_t* flag, int check) {
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const uint32_t alpha = idx / (KB * 8), ch = idx % (KB * 8);
    const uint32_t kb = ch >> 3, c16 = ch & 7;
    const uint32_t beta0 = kb * kBK + c16 * 16;
    uint32_t v[16];
    if (alpha < k && beta0 + 16 <= m && (m & 3) == 0) {
        const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)alpha * m + beta0);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint4 w = __ldg(src + q);
            v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
        }
    } else {
#pragma unroll
        for (int u = 0; u < 16; u++)
            v[u] = (alpha < k && beta0 + u < m) ? X[(size_t)alpha * m + beta0 + u] : 0u;
    }
    if (check) {
        uint32_t bad = 0;
#pragma unroll
        for (int u = 0; u < 16; u++) bad |= (v[u] >> ell);
        if (bad) atomicOr(flag, 1u);
    }
    const uint32_t mt = alpha / kBM, r = alpha % kBM;
#pragma unroll
    for (int i = 0; i < SX; i++) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; q++)
            w[q] = ((v[4 * q] >> (8 * i)) & 0xFF) | (((v[4 * q + 1] >> (8 * i)) & 0xFF) << 8) |
                   (((v[4 * q + 2] >> (8 * i)) & 0xFF) << 16) | (((v[4 * q + 3] >> (8 * i)) & 0xFF) << 24);
        uint8_t* dst = Xt + ((((size_t)mt * KB + kb) * SX + i) * kBM) * kBK + swz_off(r, c16);
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ---------------------------------------------------------------- tile Enc(W)
// CTA (ct, kb): canonical E[beta][col] for beta in the k-block, col in the
// 64-column tile -> 4 byte planes Et[ct][kb][s][64][128 B swizzled].
__global__ void __launch_bounds__(256) k_tile_encw(const uint32_t* __restrict__ canon, uint32_t m,
                                                   uint32_t ncol, uint32_t KB, uint8_t* __restrict__ Et) {
    __shared__ uint32_t sE[kBK][kBNT + 1];
    const uint32_t ct = blockIdx.x, kb = blockIdx.y;
    for (uint32_t idx = threadIdx.x; idx < kBK * kBNT; idx += blockDim.x) {
        const uint32_t b = idx / kBNT, c = idx % kBNT, beta = kb * kBK + b;
        sE[b][c] = beta < m ? canon[(size_t)beta * ncol + (size_t)ct * kBNT + c] : 0u;
    }
    __syncthreads();
    uint8_t* base = Et + ((size_t)ct * KB + kb) * kSW * kBNT * kBK;
    for (uint32_t idx = threadIdx.x; idx < kSW * kBNT * 8; idx += blockDim.x) {
        const uint32_t s = idx / (kBNT * 8), r = (idx / 8) % kBNT, c16 = idx % 8;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint32_t acc = 0;
#pragma unroll
            for (int u = 0; u < 4; u++) acc |= ((sE[c16 * 16 + 4 * q + u][r] >> (8 * s)) & 0xFF) << (8 * u);
            w[q] = acc;
        }
        *reinterpret_cast<uint4*>(base + (size_t)s * kBNT * kBK + swz_off(r, c16)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

__global__ void __launch_bounds__(256) k_untile_encw(const uint8_t* __restrict__ Et, uint32_t m, uint32_t ncol,
                                                     uint32_t KB, uint32_t* __restrict__ canon) {
    __shared__ uint32_t sE[kBK][kBNT + 1];
    const uint32_t ct = blockIdx.x, kb = blockIdx.y;
    for (uint32_t idx = threadIdx.x; idx < kBK * kBNT; idx += blockDim.x) sE[idx / kBNT][idx % kBNT] = 0;
    __syncthreads();
    const uint8_t* base = Et + ((size_t)ct * KB + kb) * kSW * kBNT * kBK;
    for (uint32_t idx = threadIdx.x; idx < kSW * kBNT * kBK; idx += blockDim.x) {
        const uint32_t s = idx / (kBNT * kBK), r = (idx / kBK) % kBNT, b = idx % kBK;
        uint32_t byte = base[(size_t)s * kBNT * kBK + swz_off(r, b >> 4) + (b & 15)];
        atomicOr(&sE[b][r], byte << (8 * s));
    }
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < kBK * kBNT; idx += blockDim.x) {
        const uint32_t b = idx / kBNT, c = idx % kBNT, beta = kb * kBK + b;
        if (beta < m) canon[(size_t)beta * ncol + (size_t)ct * kBNT + c] = sE[b][c];
    }
}

// ---------------------------------------------------------------- K7 pack/moddown/mask
// Thread per output coefficient J of packed ciphertext tg = query*nct + theta.
//  step 3: s_i = sum_{r<rows} X^{r n} c[theta R + r] at J
//        = sum_r (J >= r n ? C_r[J - r n] : -C_r[J - r n + N])
//  mod-switch: drop p_{L-1}, ..., p_{L_out}:
//        c_i <- (c_i - rho) * p_l^-1 mod p_i, rho = centered c_l  ( = round(c / p_l) )
//  step 4: b_i -= Emb_{q'}(r_theta[J]) mod p_i; R rows = r at valid slots.
__global__ void __launch_bounds__(256) k_pack(Rns Rn, const uint32_t* __restrict__ C, uint32_t kq, uint32_t n,
                                              uint32_t nct, uint64_t key_mask, uint32_t* __restrict__ cts,
                                              uint32_t* __restrict__ Rout) {
    const uint32_t N = Rn.N, L = Rn.L, Lo = Rn.L_out;
    const uint32_t J = blockIdx.x * blockDim.x + threadIdx.x, tg = blockIdx.y;
    if (J >= N) return;
    const uint32_t query = tg / nct, theta = tg % nct, Rr = N / n;
    const uint32_t rows = min(Rr, kq - theta * Rr);
    const size_t ncol = (size_t)2 * L * N;
    const size_t row0 = (size_t)query * kq + (size_t)theta * Rr;
    const uint32_t rmask = samp_mod_t(prg_word(key_mask, (uint64_t)tg * N + J), Rn.ell);
#pragma unroll 1
    for (uint32_t comp = 0; comp < 2; comp++) {
        uint32_t res[NIMBUS_MAXL];
        for (uint32_t i = 0; i < L; i++) {
            const uint32_t p = Rn.p[i];
            uint64_t acc = 0;
            const uint32_t* base = C + row0 * ncol + ((size_t)comp * L + i) * N;
            for (uint32_t r = 0; r < rows; r++) {
                const uint32_t s = r * n;
                if (J >= s) acc += __ldg(base + r * ncol + (J - s));
                else        acc += p - __ldg(base + r * ncol + (J + N - s));
            }
            res[i] = mod64(acc, p, Rn.mu[i]);
        }
        for (uint32_t l = L - 1; l >= Lo; l--) {
            const uint32_t pl = Rn.p[l];
            const uint32_t cl = res[l];
            const bool neg = cl > (pl >> 1);                  // centered rho = cl - pl < 0
            const uint32_t mag = neg ? pl - cl : cl;          // |rho| < p_l / 2
            for (uint32_t i = 0; i < l; i++) {
                const uint32_t p = Rn.p[i];
                const uint32_t mm = mag >= p ? mag - p : mag;
                const uint32_t d = neg ? addmod(res[i], mm, p) : submod(res[i], mm, p);
                res[i] = mulmod(d, Rn.inv_p[l][i], p, Rn.mu[i]);
            }
            if (l == 0) break;
        }
        for (uint32_t i = 0; i < Lo; i++) {
            uint32_t v = res[i];
            if (comp == 0) {
                const uint32_t p = Rn.p[i];
                v = submod(v, emb_mod(rmask, Rn.qout_mod_t, Rn.ell, p, Rn.mu[i], Rn.t_inv[i]), p);
            }
            cts[(((size_t)tg * 2 + comp) * Lo + i) * N + J] = v;
        }
    }
    if (J < rows * n) Rout[row0 * n + J] = rmask;
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_slice_x(nimbus_ctx* c, const uint32_t* d_X, uint32_t k, uint32_t m, uint32_t KB,
                           uint8_t* d_Xt, cudaStream_t st) {
    const uint32_t Mt = (k + kBM - 1) / kBM;
    const uint32_t total = Mt * kBM * KB * 8;
    const uint32_t SX = sx_of(c->rns.ell);
    const int check = (c->prm.flags & NIMBUS_FLAG_CHECK_RANGE) && c->rns.ell < 32;
    dim3 g((total + 255) / 256);
    if (SX == 1) k_slice_x<1><<<g, 256, 0, st>>>(d_X, k, m, KB, c->rns.ell, d_Xt, total, c->d_flag, check);
    else if (SX == 2) k_slice_x<2><<<g, 256, 0, st>>>(d_X, k, m, KB, c->rns.ell, d_Xt, total, c->d_flag, check);
    else k_slice_x<4><<<g, 256, 0, st>>>(d_X, k, m, KB, c->rns.ell, d_Xt, total, c->d_flag, check);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_tile_encw(nimbus_ctx* c, const uint32_t* d_canon, uint32_t m, uint32_t KB, uint8_t* d_Et,
                             cudaStream_t st) {
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    k_tile_encw<<<dim3(ncol / kBNT, KB), 256, 0, st>>>(d_canon, m, ncol, KB, d_Et);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_untile_encw(nimbus_ctx* c, const uint8_t* d_Et, uint32_t m, uint32_t KB, uint32_t* d_canon,
                               cudaStream_t st) {
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    k_untile_encw<<<dim3(ncol / kBNT, KB), 256, 0, st>>>(d_Et, m, ncol, KB, d_canon);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_pack(nimbus_ctx* c, const uint32_t* d_C, uint32_t kq, uint32_t nq, uint32_t n,
                        uint64_t seed, uint32_t* d_cts, uint32_t* d_R, cudaStream_t st) {
    const uint32_t N = c->rns.N, Rr = N / n, nct = (kq + Rr - 1) / Rr;
    k_pack<<<dim3((N + 255) / 256, nq * nct), 256, 0, st>>>(c->rns, d_C, kq, n, nct, prg_key(seed, 6), d_cts, d_R);
    c->launches++;
    return cudaGetLastError();
}

}  // namespace nimbus
