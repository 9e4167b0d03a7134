// pack.cu -- K7: RShift packing + mod-switch + mask (Alg. 1 steps 3-4,
// PAPER.md:672-680).  Memory-bound: reads the
// unpacked C (k x 2LN residues, L2-resident right after the contraction)
// once, writes the compact ciphertexts and the client share R.
//
// Thread = V consecutive output coefficients J of one component of packed
// ciphertext tg = query*nct + theta, all limbs (the mod-switch mixes limbs):
//   step 3:  s_i[J] = sum_{r < rows} (X^{r n} c[theta R + r])_i[J]
//                   = sum_r (J >= r n ? C_r[J - r n] : p_i - C_r[J - r n + N])  (RShift)
//            summed lazily in 64 bits, one reduction per coefficient;
//   switch:  for l = L-1 .. L_out:  c_i <- (c_i - rho) * p_l^-1 mod p_i,
//            rho = centered c_l  (= round(c / p_l));
//   step 4:  b_i -= Emb_{q'}(r_theta[J]),  r_theta[J] = word(seed, 6, tg*N + J) >> (64-ell)
//            (SURVEY.md §8(c) #13); R[alpha][j] = r_theta[(alpha mod R) n + j].
// V = 2 or 4 coefficients per thread (uint2 / uint4 loads and stores) when V
// divides n and the grid stays large; a group of V J never straddles a wrap
// point because J and r n are multiples of V.
#include <algorithm>
#include <cstdlib>
#include "pack_dev.cuh"

namespace nimbus {

#ifdef NIMBUS_TRACE
// Debug-only pack timeline (globaltimer ns): [0] first block start, [1] first block past the
// PDL wait, [2] last block past the wait, [3] last block end (tools/trace_tc.py).
__device__ unsigned long long* g_trace_pack = nullptr;
extern "C" int nimbus_trace_pack_set(void* p) { return (int)cudaMemcpyToSymbol(g_trace_pack, &p, sizeof(p)); }
__device__ __forceinline__ unsigned long long gtimer_pack() {
    unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}
#define PTRACE_MIN(i) do { if (g_trace_pack && threadIdx.x == 0) atomicMin(&g_trace_pack[i], gtimer_pack()); } while (0)
#define PTRACE_MAX(i) do { if (g_trace_pack) { __syncthreads(); if (threadIdx.x == 0) atomicMax(&g_trace_pack[i], gtimer_pack()); } } while (0)
#else
#define PTRACE_MIN(i) do { } while (0)
#define PTRACE_MAX(i) do { } while (0)
#endif

// blockIdx.z = comp + 2 * job: one launch packs the matmuls of a same-X group (PackJobs, all
// of one shape) whose contractions ran as one launch (k_cop_tc_res over a job list)
template <int V, int L, int RB, typename MT = uint32_t>
__global__ void __launch_bounds__(128) k_pack(Rns Rn, PackJobs P, uint32_t kq, uint32_t n, uint32_t Rr, uint32_t nct,
                                              const uint32_t* __restrict__ Z0) {
    pdl_trigger();
    PTRACE_MIN(0);
    const uint32_t J = (blockIdx.x * blockDim.x + threadIdx.x) * V;
#ifndef NIMBUS_TRACE
    if (J >= Rn.N) return;
#endif
    const uint32_t job = blockIdx.z >> 1, comp = blockIdx.z & 1;
    PackMask<V, L, MT> mk;
    if (comp == 0 && J < Rn.N) pack_mask<V, L, MT>(Rn, P.key[job], blockIdx.y, J, mk);
    pdl_wait();  // C is produced by the contraction kernel
    PTRACE_MIN(1);
    PTRACE_MAX(2);
    if (J < Rn.N)
        pack_item<V, L, RB, MT>(Rn, P.C[job], kq, n, Rr, nct, P.key[job], P.cts[job], static_cast<MT*>(P.R[job]), Z0,
                                blockIdx.y, comp, J, mk);
    PTRACE_MAX(3);
}

template <typename K, typename... Args>
static cudaError_t launch_maybe_pdl(bool pdl, K kernel, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    if (pdl) return launch_pdl(kernel, grid, block, 0, st, args...);
    kernel<<<grid, block, 0, st>>>(args...);
    return cudaGetLastError();
}

template <int V, int RB>
static cudaError_t launch_vr(nimbus_ctx* c, const PackJobs& P, uint32_t kq, uint32_t nq, uint32_t n, cudaStream_t st,
                             bool pdl, const uint32_t* Z0) {
    const uint32_t N = c->rns.N, Rr = N / n, nct = (kq + Rr - 1) / Rr;
    const uint32_t per_block = 128 * V;
    dim3 grid((N + per_block - 1) / per_block, nq * nct, 2 * P.nj);
    switch (c->rns.L) {
        case 1: return launch_maybe_pdl(pdl, k_pack<V, 1, RB>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
        case 2: return launch_maybe_pdl(pdl, k_pack<V, 2, RB>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
        case 3: return launch_maybe_pdl(pdl, k_pack<V, 3, RB>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
        case 4: return launch_maybe_pdl(pdl, k_pack<V, 4, RB>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
        case 5: return launch_maybe_pdl(pdl, k_pack<V, 5, RB>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
        default: return launch_maybe_pdl(pdl, k_pack<V, 6, RB>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
    }
}

// ell > 32: 64-bit masks and R, one coefficient per thread, L in {4, 5, 6}
template <int RB>
static cudaError_t launch_r64(nimbus_ctx* c, const PackJobs& P, uint32_t kq, uint32_t nq, uint32_t n, cudaStream_t st,
                              bool pdl, const uint32_t* Z0) {
    const uint32_t N = c->rns.N, Rr = N / n, nct = (kq + Rr - 1) / Rr;
    dim3 grid((N + 127) / 128, nq * nct, 2 * P.nj);
    switch (c->rns.L) {
        case 4: return launch_maybe_pdl(pdl, k_pack<1, 4, RB, uint64_t>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
        case 5: return launch_maybe_pdl(pdl, k_pack<1, 5, RB, uint64_t>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
        case 6: return launch_maybe_pdl(pdl, k_pack<1, 6, RB, uint64_t>, grid, dim3(128), st, c->rns, P, kq, n, Rr, nct, Z0);
        default: return cudaErrorInvalidValue;
    }
}

// rows per load batch: R itself when R is 1, 2, 4 or 5 (or a multiple of 5), else a power of two
static uint32_t rows_per_batch(uint32_t Rr, uint32_t kq) {
    const uint32_t r = Rr < kq ? Rr : kq;         // rows of the fullest packed ciphertext
    if (r <= 2) return r;
    if (r <= 4) return 4;
    if (r % 5 == 0) return 5;
    return 8;
}

static cudaError_t launch_64(nimbus_ctx* c, const PackJobs& P, uint32_t kq, uint32_t nq, uint32_t n, cudaStream_t st,
                             bool pdl, const uint32_t* Z0) {
    switch (rows_per_batch(c->rns.N / n, kq)) {
        case 1: return launch_r64<1>(c, P, kq, nq, n, st, pdl, Z0);
        case 2: return launch_r64<2>(c, P, kq, nq, n, st, pdl, Z0);
        case 4: return launch_r64<4>(c, P, kq, nq, n, st, pdl, Z0);
        case 5: return launch_r64<5>(c, P, kq, nq, n, st, pdl, Z0);
        default: return launch_r64<8>(c, P, kq, nq, n, st, pdl, Z0);
    }
}

template <int V>
static cudaError_t launch_v(nimbus_ctx* c, const PackJobs& P, uint32_t kq, uint32_t nq, uint32_t n, cudaStream_t st,
                            bool pdl, const uint32_t* Z0) {
    switch (rows_per_batch(c->rns.N / n, kq)) {
        case 1: return launch_vr<V, 1>(c, P, kq, nq, n, st, pdl, Z0);
        case 2: return launch_vr<V, 2>(c, P, kq, nq, n, st, pdl, Z0);
        case 4: return launch_vr<V, 4>(c, P, kq, nq, n, st, pdl, Z0);
        case 5: return launch_vr<V, 5>(c, P, kq, nq, n, st, pdl, Z0);
        default: return launch_vr<V, 8>(c, P, kq, nq, n, st, pdl, Z0);
    }
}

// R alone (the client's share Y_c = the mask at the valid slots):
// R[alpha][j] = r_theta[rho n + j], alpha = query kq + theta R + rho.  It depends only on
// the mask seed, so the host-buffer call computes and downloads it while the
// contraction runs (the pack then skips R).
template <typename MT>
__global__ void k_mask_R(uint32_t N, uint32_t ell, uint32_t kq, uint32_t nq, uint32_t n, uint32_t Rr, uint32_t nct,
                         uint64_t key, MT* __restrict__ R) {
    const uint64_t total = (uint64_t)kq * nq * n;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t alpha = (uint32_t)(i / n), j = (uint32_t)(i % n);
        const uint32_t query = alpha / kq, a = alpha % kq, theta = a / Rr, rho = a % Rr;
        const uint64_t w = prg_word(key, (uint64_t)(query * nct + theta) * N + rho * n + j);
        R[i] = (MT)(ell >= 64 ? w : w >> (64 - ell));
    }
}

cudaError_t launch_mask_R(nimbus_ctx* c, uint32_t kq, uint32_t nq, uint32_t n, uint64_t seed, void* d_R,
                          cudaStream_t st) {
    const uint32_t N = c->rns.N, Rr = N / n, nct = (kq + Rr - 1) / Rr;
    const uint64_t key = prg_key(seed, 6);
    const uint64_t total = (uint64_t)kq * nq * n;
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((total + 255) / 256, 4ull * c->num_sms);
    if (elem_bytes(c->rns.ell) == 8)
        k_mask_R<uint64_t><<<blocks, 256, 0, st>>>(N, c->rns.ell, kq, nq, n, Rr, nct, key, static_cast<uint64_t*>(d_R));
    else
        k_mask_R<uint32_t><<<blocks, 256, 0, st>>>(N, c->rns.ell, kq, nq, n, Rr, nct, key, static_cast<uint32_t*>(d_R));
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_pack(nimbus_ctx* c, const uint32_t* d_C, uint32_t kq, uint32_t nq, uint32_t n,
                        uint64_t seed, uint32_t* d_cts, void* d_R, cudaStream_t st, bool pdl, const uint32_t* Z0) {
    PackJobs P;
    P.nj = 1;
    P.C[0] = d_C; P.cts[0] = d_cts; P.R[0] = d_R; P.key[0] = prg_key(seed, 6);
    return launch_pack_jobs(c, P, kq, nq, n, st, pdl, Z0);
}

cudaError_t launch_pack_jobs(nimbus_ctx* c, const PackJobs& P, uint32_t kq, uint32_t nq, uint32_t n, cudaStream_t st,
                             bool pdl, const uint32_t* Z0) {
    {   // the pack writes the ciphertexts and R and triggers its dependents early
        const uint32_t Rr0 = c->rns.N / n, nct0 = (kq + Rr0 - 1) / Rr0;
        const void* op[2 * 4];
        size_t ob[2 * 4];
        uint32_t no = 0;
        for (uint32_t j = 0; j < P.nj && j < 4; j++) {
            op[no] = P.cts[j];
            ob[no++] = (size_t)nq * nct0 * 2 * c->rns.L_out * c->rns.N * 4;
            op[no] = P.R[j];
            ob[no++] = (size_t)kq * nq * n * elem_bytes(c->rns.ell);
        }
        pdl_outputs_set(st, op, ob, no);
    }
    if (elem_bytes(c->rns.ell) == 8) {
        cudaError_t e = launch_64(c, P, kq, nq, n, st, pdl, Z0);
        c->launches++;
        return e;
    }
    const uint32_t N = c->rns.N, Rr = N / n, nct = (kq + Rr - 1) / Rr;
    // V coefficients per thread (vector loads/stores; J and r n stay multiples of V): the
    // widest V whose grid (all jobs of the launch) still has >= 5 blocks of 128 per SM.  The
    // pack runs alone after the contraction in the PDL chain; since its masks are computed
    // before its PDL wait, what remains after it is the loads and the arithmetic, and fewer,
    // wider threads win until the grid drops under ~5 blocks per SM (B200, block timing, this
    // round: C2 V=2 20.05 us/step vs V=1 20.33 / V=4 20.57; C2-QKV V=2 40.3 vs V=1 42.2 /
    // V=4 42.0; round 1, masks after the wait, 16 blocks per SM was the threshold)
    const uint64_t threads_v1 = 2ull * nq * nct * N * P.nj;      // one thread per (job, comp, J)
    const uint64_t min_threads = 5ull * 128 * (uint64_t)c->num_sms;
    uint32_t V = (n % 4 == 0 && threads_v1 / 4 >= min_threads) ? 4
               : (n % 2 == 0 && threads_v1 / 2 >= min_threads) ? 2 : 1;
    if (const char* ev = getenv("NIMBUS_PACK_V")) {        // experiment switch: 1, 2 or 4
        const uint32_t v = (uint32_t)atoi(ev);
        if ((v == 1 || v == 2 || v == 4) && n % v == 0) V = v;
    }
    // vector stores need V * 4-byte aligned outputs: a caller's 4- or 8-byte aligned buffers get V = 1 / 2
    uintptr_t al = 0;
    for (uint32_t j = 0; j < P.nj; j++) al |= (uintptr_t)P.cts[j] | (uintptr_t)P.R[j];
    if (V == 4 && (al & 15)) V = 2;
    if (V == 2 && (al & 7)) V = 1;
    cudaError_t e = V == 4 ? launch_v<4>(c, P, kq, nq, n, st, pdl, Z0)
                  : V == 2 ? launch_v<2>(c, P, kq, nq, n, st, pdl, Z0)
                           : launch_v<1>(c, P, kq, nq, n, st, pdl, Z0);
    c->launches++;
    return e;
}

}  // namespace nimbus
