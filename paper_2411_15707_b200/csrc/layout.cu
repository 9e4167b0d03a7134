// layout.cu -- data-layout kernels of the COP hot path:
//   K4  slice X into 8-bit planes in the tcgen05 operand layout (A3)
//   tile / untile Enc(W) between the canonical [beta][comp][limb][j] layout
//       and the resident byte-plane kernel layout (setup / export)
//   (K7, packing + mod-switch + mask, is in pack.cu)
//
// Kernel layout of a byte-plane tile: a 2-D block of
// R rows x 128 bytes, row r at offset r*128, the 16-byte chunk c of row r
// stored at chunk position c ^ (r & 7) -- the 128-byte swizzle that the
// tcgen05 shared-memory descriptor (SWIZZLE_128B, K-major) expects, applied
// once at rest so that one linear bulk copy lands a ready-to-use operand tile.
#include <cstdlib>
#include <mutex>
#include <vector>
#include "slice_dev.cuh"

namespace nimbus {

template <int SX, int RT, typename T = uint32_t>
__global__ void k_slice_x(const T* __restrict__ X, uint32_t k, uint32_t m, uint32_t KB, uint32_t ell,
                          uint8_t* __restrict__ Xt, uint32_t total, uint32_t* flag, int check, int late) {
    pdl_trigger();
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    // X (the caller's input) is read and sliced while the previous kernel of the stream may
    // still run; the planes are stored only after it is done (it may still read Xt).  late:
    // X is an output of that kernel (pdl_outputs_overlap), so it is read after the wait too.
    if (late) pdl_wait();
    SlicePlanes<SX> sp;
    if (idx < total) sp = slice_load<SX, RT, T>(X, k, m, KB, ell, idx, check);
    if (!late) pdl_wait();
    if (idx < total) slice_store<SX, RT>(sp, Xt, flag);
}

// ---------------------------------------------------------------- tile Enc(W)
// CTA (ct, kb): canonical E[beta][col] for beta in the k-block, col in the
// BN-column tile -> 4 byte planes Et[ct][kb][s][BN][128 B swizzled]; rows
// beta >= m and columns >= 2LN (padding tiles) are zero.
template <int BN>
__global__ void __launch_bounds__(256) k_tile_encw(const uint32_t* __restrict__ canon, uint32_t m,
                                                   uint32_t ncol, uint32_t KB, uint8_t* __restrict__ Et) {
    extern __shared__ uint32_t sE_raw[];
    uint32_t (*sE)[BN + 1] = reinterpret_cast<uint32_t (*)[BN + 1]>(sE_raw);
    const uint32_t ct = blockIdx.x, kb = blockIdx.y;
    for (uint32_t idx = threadIdx.x; idx < kBK * BN; idx += blockDim.x) {
        const uint32_t b = idx / BN, c = idx % BN, beta = kb * kBK + b;
        const size_t col = (size_t)ct * BN + c;
        sE[b][c] = (beta < m && col < ncol) ? canon[(size_t)beta * ncol + col] : 0u;
    }
    __syncthreads();
    uint8_t* base = Et + ((size_t)ct * KB + kb) * kSW * BN * kBK;
    for (uint32_t idx = threadIdx.x; idx < kSW * BN * 8; idx += blockDim.x) {
        const uint32_t s = idx / (BN * 8), r = (idx / 8) % BN, c16 = idx % 8;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint32_t acc = 0;
#pragma unroll
            for (int u = 0; u < 4; u++) acc |= ((sE[c16 * 16 + 4 * q + u][r] >> (8 * s)) & 0xFF) << (8 * u);
            w[q] = acc;
        }
        *reinterpret_cast<uint4*>(base + (size_t)s * BN * kBK + swz_off(r, c16)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <int BN>
__global__ void __launch_bounds__(256) k_untile_encw(const uint8_t* __restrict__ Et, uint32_t m, uint32_t ncol,
                                                     uint32_t KB, uint32_t* __restrict__ canon) {
    extern __shared__ uint32_t sE_raw[];
    uint32_t (*sE)[BN + 1] = reinterpret_cast<uint32_t (*)[BN + 1]>(sE_raw);
    const uint32_t ct = blockIdx.x, kb = blockIdx.y;
    for (uint32_t idx = threadIdx.x; idx < kBK * BN; idx += blockDim.x) sE[idx / BN][idx % BN] = 0;
    __syncthreads();
    const uint8_t* base = Et + ((size_t)ct * KB + kb) * kSW * BN * kBK;
    for (uint32_t idx = threadIdx.x; idx < kSW * BN * kBK; idx += blockDim.x) {
        const uint32_t s = idx / (BN * kBK), r = (idx / kBK) % BN, b = idx % kBK;
        uint32_t byte = base[(size_t)s * BN * kBK + swz_off(r, b >> 4) + (b & 15)];
        atomicOr(&sE[b][r], byte << (8 * s));
    }
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < kBK * BN; idx += blockDim.x) {
        const uint32_t b = idx / BN, c = idx % BN, beta = kb * kBK + b;
        const size_t col = (size_t)ct * BN + c;
        if (beta < m && col < ncol) canon[(size_t)beta * ncol + col] = sE[b][c];
    }
}

// ---------------------------------------------------------------- PDL output records
namespace {
struct PdlRecord {
    cudaStream_t st;
    std::vector<std::pair<uintptr_t, uintptr_t>> ranges;    // [lo, hi)
};
std::mutex g_pdl_mu;
std::vector<PdlRecord> g_pdl;                                // one record per stream (a few streams)
}  // namespace

void pdl_outputs_set(cudaStream_t st, const void* const* ptrs, const size_t* bytes, uint32_t n) {
    std::lock_guard<std::mutex> lk(g_pdl_mu);
    PdlRecord* r = nullptr;
    for (PdlRecord& x : g_pdl)
        if (x.st == st) r = &x;
    if (!r) {
        if (g_pdl.size() >= 64) g_pdl.erase(g_pdl.begin());
        g_pdl.push_back(PdlRecord{st, {}});
        r = &g_pdl.back();
    }
    r->ranges.clear();
    for (uint32_t i = 0; i < n; i++)
        if (ptrs[i] && bytes[i]) {
            const uintptr_t lo = reinterpret_cast<uintptr_t>(ptrs[i]);
            r->ranges.emplace_back(lo, lo + bytes[i]);
        }
}

bool pdl_outputs_overlap(cudaStream_t st, const void* p, size_t bytes) {
    static const bool off = getenv("NIMBUS_NO_PDL_GUARD") != nullptr;    // test switch: show the hazard
    if (off) return false;
    std::lock_guard<std::mutex> lk(g_pdl_mu);
    const uintptr_t lo = reinterpret_cast<uintptr_t>(p), hi = lo + bytes;
    for (const PdlRecord& x : g_pdl)
        if (x.st == st)
            for (const auto& r : x.ranges)
                if (lo < r.second && r.first < hi) return true;
    return false;
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_slice_x(nimbus_ctx* c, const void* d_Xv, uint32_t k, uint32_t m, uint32_t KB, uint32_t rt,
                           uint8_t* d_Xt, cudaStream_t st) {
    const uint32_t Mt = (k + rt - 1) / rt;
    const uint32_t total = Mt * rt * KB * 8;
    const uint32_t SX = sx_of(c->rns.ell);
    const int check = (c->prm.flags & NIMBUS_FLAG_CHECK_RANGE) && c->rns.ell < 32;
    dim3 g((total + 255) / 256);
    cudaError_t e;
    const uint32_t ell = c->rns.ell;
    const uint32_t* d_X = static_cast<const uint32_t*>(d_Xv);
    const int late = pdl_outputs_overlap(st, d_Xv, (size_t)k * m * elem_bytes(ell)) ? 1 : 0;
    if (SX == 8) {
        const int check64 = (c->prm.flags & NIMBUS_FLAG_CHECK_RANGE) && ell < 64;
        e = launch_pdl(k_slice_x<8, 32, uint64_t>, g, 256, 0, st, static_cast<const uint64_t*>(d_Xv), k, m, KB, ell,
                       d_Xt, total, c->d_flag, check64, late);
    } else if (rt == 64 && SX == 2) e = launch_pdl(k_slice_x<2, 64>, g, 256, 0, st, d_X, k, m, KB, ell, d_Xt, total, c->d_flag, check, late);
    else if (rt == 64) e = launch_pdl(k_slice_x<4, 64>, g, 256, 0, st, d_X, k, m, KB, ell, d_Xt, total, c->d_flag, check, late);
    else if (rt == 32) e = launch_pdl(k_slice_x<4, 32>, g, 256, 0, st, d_X, k, m, KB, ell, d_Xt, total, c->d_flag, check, late);
    else if (SX == 1) e = launch_pdl(k_slice_x<1, 128>, g, 256, 0, st, d_X, k, m, KB, ell, d_Xt, total, c->d_flag, check, late);
    else if (SX == 2) e = launch_pdl(k_slice_x<2, 128>, g, 256, 0, st, d_X, k, m, KB, ell, d_Xt, total, c->d_flag, check, late);
    else e = launch_pdl(k_slice_x<4, 128>, g, 256, 0, st, d_X, k, m, KB, ell, d_Xt, total, c->d_flag, check, late);
    c->launches++;
    return e;
}

cudaError_t launch_tile_encw(nimbus_ctx* c, const uint32_t* d_canon, uint32_t m, uint32_t KB, uint32_t bn,
                             uint8_t* d_Et, cudaStream_t st) {
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    const dim3 g(col_tiles(c, bn), KB);
    const size_t smem = (size_t)kBK * (bn + 1) * 4;
    cudaError_t e;
    if (bn == kBNR) {
        k_tile_encw<kBNR><<<g, 256, smem, st>>>(d_canon, m, ncol, KB, d_Et);
    } else if (bn == kBNW) {
        e = cudaFuncSetAttribute(k_tile_encw<kBNW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_tile_encw<kBNW><<<g, 256, smem, st>>>(d_canon, m, ncol, KB, d_Et);
    } else {
        k_tile_encw<kBNT><<<g, 256, smem, st>>>(d_canon, m, ncol, KB, d_Et);
    }
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_untile_encw(nimbus_ctx* c, const uint8_t* d_Et, uint32_t m, uint32_t KB, uint32_t bn,
                               uint32_t* d_canon, cudaStream_t st) {
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    const dim3 g(col_tiles(c, bn), KB);
    const size_t smem = (size_t)kBK * (bn + 1) * 4;
    cudaError_t e;
    if (bn == kBNR) {
        k_untile_encw<kBNR><<<g, 256, smem, st>>>(d_Et, m, ncol, KB, d_canon);
    } else if (bn == kBNW) {
        e = cudaFuncSetAttribute(k_untile_encw<kBNW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_untile_encw<kBNW><<<g, 256, smem, st>>>(d_Et, m, ncol, KB, d_canon);
    } else {
        k_untile_encw<kBNT><<<g, 256, smem, st>>>(d_Et, m, ncol, KB, d_canon);
    }
    c->launches++;
    return cudaGetLastError();
}

}  // namespace nimbus
