// ntt_dev.cuh -- device pieces shared by the NTT kernels (ntt.cu: KeyGen, decrypt,
// re-randomisation) and the fused Encrypt-rows kernel (encrypt.cu): the two butterflies
// with Shoup multiplication, and the distributed-shared-memory accessors of a cluster.
#pragma once
#include "internal.h"

namespace nimbus {

// Twiddle tables (ctx->d_tw, per limb: forward, its Shoup companions, inverse, companions):
// psi_rev[k] = psi^bitrev(k), k in [1, N), used by forward stage (m blocks, block i) as
// psi_rev[m + i]; the inverse stage with h blocks uses the inverse table at h + i.
// Cooley-Tukey butterfly (x, y) <- (x + S y, x - S y) and Gentleman-Sande (x, y) <- (x + y, (x - y) S).
__device__ __forceinline__ void ct_bfly(uint32_t& x, uint32_t& y, uint32_t S, uint32_t Ssh, uint32_t p) {
    const uint32_t V = mulmod_shoup(y, S, Ssh, p);
    y = submod(x, V, p);
    x = addmod(x, V, p);
}
__device__ __forceinline__ void gs_bfly(uint32_t& x, uint32_t& y, uint32_t S, uint32_t Ssh, uint32_t p) {
    const uint32_t U = x;
    x = addmod(U, y, p);
    y = mulmod_shoup(submod(U, y, p), S, Ssh, p);
}

__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(cta));
    return r;
}
__device__ __forceinline__ uint32_t ld_dsmem(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem(uint32_t a, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(a), "r"(v) : "memory");
}

}  // namespace nimbus
