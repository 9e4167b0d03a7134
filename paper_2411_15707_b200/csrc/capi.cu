// capi.cu -- the C ABI of libnimbus_cop.so (include/nimbus_cop.h): parameter
// validation, RNS constant / twiddle derivation, handle management, and the
// launch sequence of each entry point.  All arithmetic runs in the kernels.
#include <nvtx3/nvToolsExt.h>
#include <fcntl.h>
#include <unistd.h>
#include <cerrno>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "internal.h"

using namespace nimbus;

// ---------------------------------------------------------------- host number theory
static uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((u128)a * b % p); }
static uint64_t h_pow(uint64_t a, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    a %= p;
    while (e) { if (e & 1) r = h_mulmod(r, a, p); a = h_mulmod(a, a, p); e >>= 1; }
    return r;
}
static uint64_t h_inv(uint64_t a, uint64_t p) { return h_pow(a % p, p - 2, p); }

// deterministic Miller-Rabin for n < 2^32 (bases 2, 3, 5, 7)
static bool h_is_prime(uint64_t n) {
    if (n < 2) return false;
    for (uint64_t sp : {2ull, 3ull, 5ull, 7ull}) if (n % sp == 0) return n == sp;
    uint64_t d = n - 1; int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (uint64_t a : {2ull, 3ull, 5ull, 7ull}) {
        uint64_t x = h_pow(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; r++) { x = h_mulmod(x, x, n); if (x == n - 1) { comp = false; break; } }
        if (comp) return false;
    }
    return true;
}

static uint32_t bitrev(uint32_t x, uint32_t bits) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

static nimbus_status set_err(nimbus_ctx* c, nimbus_status st, const char* msg) {
    if (c) c->err = msg;
    return st;
}
static nimbus_status cuda_err(nimbus_ctx* c, cudaError_t e, const char* where) {
    if (e == cudaSuccess) return NIMBUS_OK;
    if (c) { c->err = std::string(where) + ": " + cudaGetErrorString(e); }
    return e == cudaErrorMemoryAllocation ? NIMBUS_ENOMEM : NIMBUS_ECUDA;
}
#define CK(call, where) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) return cuda_err(ctx, e_, where); } while (0)

static inline uint64_t ncols(const nimbus_ctx* c) { return 2ull * c->rns.L * c->rns.N; }

// Big (internal.h) arithmetic for q = prod p_i beyond 128 bits (ell = 64 needs q > 2^150)
// and the noise bound products.
static Big big_of(u128 x) { Big b; b.w[0] = (uint64_t)x; b.w[1] = (uint64_t)(x >> 64); return b; }
static void big_mul(Big& a, uint64_t m) {
    u128 c = 0;
    for (int i = 0; i < 6; i++) { c += (u128)a.w[i] * m; a.w[i] = (uint64_t)c; c >>= 64; }
}
static void big_add(Big& a, uint64_t v) {
    u128 c = v;
    for (int i = 0; i < 6 && c; i++) { c += a.w[i]; a.w[i] = (uint64_t)c; c >>= 64; }
}
static void big_shl(Big& a, uint32_t sh) {       // a <<= sh, sh <= 64
    if (sh == 64) { for (int i = 5; i > 0; i--) a.w[i] = a.w[i - 1]; a.w[0] = 0; return; }
    if (sh == 0) return;
    for (int i = 5; i > 0; i--) a.w[i] = (a.w[i] << sh) | (a.w[i - 1] >> (64 - sh));
    a.w[0] <<= sh;
}
static uint64_t big_divmod(Big& a, uint64_t d) {  // a /= d, returns a mod d
    u128 r = 0;
    for (int i = 5; i >= 0; i--) { r = (r << 64) | a.w[i]; a.w[i] = (uint64_t)(r / d); r %= d; }
    return (uint64_t)r;
}
static int big_cmp(const Big& a, const Big& b) {
    for (int i = 5; i >= 0; i--) if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

// Worst-case decryption bound (SURVEY.md §8(c) "Worst-case noise guarantee"),
// in integer upper bounds on 2|v|:  fresh+COP+packing 2v <= R m (t-1)(2 eta + 1);
// each limb drop v -> v/p + (1+N)/2; the mask adds 1/2.  Requires 2|v| t < q.
// extra2: a further bound on 2|v| added before the mod-switch (the public-key zero
// encryption of reading 26: 2 |v e_pk + e1 + f - e2 s| <= 4 eta N + 2 eta + 2^(F+1)).
static bool noise_ok(const nimbus_ctx* c, uint32_t m, uint32_t R_eff, uint64_t extra2 = 0, uint32_t flood2 = 0) {
    const uint32_t ell = c->rns.ell, N = c->rns.N;
    const uint64_t tm1 = ell >= 64 ? ~0ULL : (1ULL << ell) - 1;
    Big B = big_of((u128)R_eff * m * 43u);      // 2 eta + 1 = 43 for CBD(21)
    big_mul(B, tm1);
    big_add(B, extra2);
    if (flood2) {                               // + 2^flood2 (twice the flooding bound 2^F, F up to 126)
        Big F2;
        F2.w[flood2 / 64] = 1ull << (flood2 % 64);
        uint64_t carry = 0;
        for (int i = 0; i < 6; i++) {
            const u128 sum = (u128)B.w[i] + F2.w[i] + carry;
            B.w[i] = (uint64_t)sum;
            carry = (uint64_t)(sum >> 64);
        }
    }
    Big Bt = B;
    big_shl(Bt, ell);
    if (big_cmp(Bt, c->q) >= 0) return false;
    for (uint32_t l = c->rns.L; l > c->rns.L_out; l--) {
        const uint64_t p = c->rns.p[l - 1];
        const uint64_t r = big_divmod(B, p);      // ceil(B / p) + 1 + N
        big_add(B, (r ? 1 : 0) + 1 + N);
    }
    big_add(B, 1);
    big_shl(B, ell);
    return big_cmp(B, big_of(c->qout)) < 0;
}


// Every entry point that touches the GPU runs on its context's device and restores the
// caller's current device on return (a process may drive several devices).
// Every public call: run on the context's device (restoring the caller's), inside an
// NVTX range named after the call (visible to ncu --nvtx / Nsight Systems; a no-op
// without a tool attached).
struct DevGuard {
    int prev = -1;
    DevGuard(int dev, const char* name) {
        nvtxRangePushA(name);
        if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    DevGuard(const nimbus_ctx* c, const char* name) : DevGuard(c ? c->device : -1, name) {}
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
        nvtxRangePop();
    }
};

extern "C" {

nimbus_status nimbus_ctx_create(const nimbus_params* prm, int device, nimbus_ctx** out) {
    if (!prm || !out) return NIMBUS_EINVAL;
    *out = nullptr;
    const uint32_t N = prm->N, L = prm->L, ell = prm->ell, Lo = prm->L_out;
    if (N < 64 || N > 8192 || (N & (N - 1))) return NIMBUS_EINVAL;
    if (L < 1 || L > NIMBUS_MAXL || Lo < 1 || Lo > L || ell < 1 || ell > 64) return NIMBUS_EINVAL;
    if (ell > 32 && prm->impl != NIMBUS_IMPL_TCGEN05) return NIMBUS_EINVAL;   // CUDA-core ablation: ell <= 32
    if (prm->impl > 1) return NIMBUS_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return NIMBUS_ECUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return NIMBUS_ECUDA;
    if (prop.major != 10 || prop.minor != 0) return NIMBUS_EARCH;

    nimbus_ctx* ctx = new (std::nothrow) nimbus_ctx();
    if (!ctx) return NIMBUS_ENOMEM;
    ctx->prm = *prm;
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    if (const char* cl = getenv("NIMBUS_CLUSTER")) ctx->cluster = atoi(cl) == 2 ? 2 : 1;
    if (const char* rr = getenv("NIMBUS_RES")) ctx->res_ring = atoi(rr) == 2 ? 2 : 1;
    if (const char* nf = getenv("NIMBUS_NO_FUSE")) ctx->fuse_r1 = atoi(nf) == 0;
    Rns& R = ctx->rns;
    R.N = N; R.L = L; R.L_out = Lo; R.ell = ell;
    R.logN = 0; while ((1u << R.logN) < N) R.logN++;
    // primes: the L largest p < 2^31 with p = 1 mod 2N, descending
    {
        const uint64_t step = 2ull * N;
        uint64_t cnd = ((((1ull << 31) - 2)) / step) * step + 1;
        uint32_t f = 0;
        while (f < L && cnd > (1ull << 30)) { if (h_is_prime(cnd)) R.p[f++] = (uint32_t)cnd; cnd -= step; }
        if (f < L) { delete ctx; return NIMBUS_EINVAL; }
    }
    ctx->q = Big();
    ctx->q.w[0] = 1;
    for (uint32_t i = 0; i < L; i++) big_mul(ctx->q, R.p[i]);
    ctx->qout = 1;
    for (uint32_t i = 0; i < Lo; i++) ctx->qout *= R.p[i];
    // decrypt arithmetic: the remainder of the long division by 2q' is shifted 32 bits
    // at a time in 128 bits, so q' < 2^95 (at most 3 limbs)
    {
        int qb = 0; u128 x = ctx->qout; while (x) { qb++; x >>= 1; }
        if (Lo > 3 || qb > 95) { delete ctx; return NIMBUS_EINVAL; }
    }
    const uint64_t tmask = ell >= 64 ? ~0ULL : (1ULL << ell) - 1;
    R.q_mod_t = ctx->q.w[0] & tmask;                 // q mod 2^ell = low bits
    R.qout_mod_t = (uint64_t)ctx->qout & tmask;
    for (uint32_t i = 0; i < L; i++) {
        const uint64_t p = R.p[i];
        R.mu[i] = (uint64_t)((((u128)1) << 64) / p);
        R.t_inv[i] = (uint32_t)h_inv(h_pow(2, ell, p), p);
        for (uint32_t s = 0; s < 12; s++) R.pow8[i][s] = (uint32_t)h_pow(2, 8 * s, p);
        R.c32[i] = (uint32_t)(((u128)1 << 32) % p);
        if (R.c32[i] >= (1u << 21)) { delete ctx; return NIMBUS_EINVAL; }   // reduce64_pm precondition
        R.t_inv_sh[i] = (uint32_t)(((uint64_t)R.t_inv[i] << 32) / p);
        for (uint32_t l = 0; l < L; l++) {
            R.inv_p[l][i] = (l == i) ? 0 : (uint32_t)h_inv(R.p[l], p);
            R.inv_p_sh[l][i] = (uint32_t)(((uint64_t)R.inv_p[l][i] << 32) / p);
        }
        R.ninv[i] = (uint32_t)h_inv(N, p);
        R.ninv_sh[i] = (uint32_t)(((uint64_t)R.ninv[i] << 32) / p);
    }
    // twiddles: psi a primitive 2N-th root (psi^N = -1), bit-reversed powers
    std::vector<uint32_t> tw((size_t)L * 4 * N);
    for (uint32_t i = 0; i < L; i++) {
        const uint64_t p = R.p[i];
        uint64_t psi = 0;
        for (uint64_t x = 3; x < p; x++) {
            uint64_t c = h_pow(x, (p - 1) / (2ull * N), p);
            if (h_pow(c, N, p) == p - 1) { psi = c; break; }
        }
        const uint64_t ipsi = h_inv(psi, p);
        uint32_t* b = tw.data() + (size_t)i * 4 * N;
        for (uint32_t kk = 0; kk < N; kk++) {
            const uint32_t e = bitrev(kk, R.logN);
            const uint32_t w = (uint32_t)h_pow(psi, e, p), iw = (uint32_t)h_pow(ipsi, e, p);
            b[kk] = w;
            b[N + kk] = (uint32_t)(((uint64_t)w << 32) / p);
            b[2 * N + kk] = iw;
            b[3 * N + kk] = (uint32_t)(((uint64_t)iw << 32) / p);
        }
    }
    DevGuard dg_(device, __func__);
    cudaError_t e = cudaMalloc(&ctx->d_tw, tw.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(ctx->d_tw, tw.data(), tw.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_flag, 16);
    if (e == cudaSuccess) e = cudaMemset(ctx->d_flag, 0, 16);
    if (e != cudaSuccess) { nimbus_ctx_destroy(ctx); return e == cudaErrorMemoryAllocation ? NIMBUS_ENOMEM : NIMBUS_ECUDA; }
    *out = ctx;
    return NIMBUS_OK;
}

static void ctx_retain(nimbus_ctx* ctx) { ctx->refs.fetch_add(1, std::memory_order_relaxed); }

static void ctx_free(nimbus_ctx* ctx);
static void ctx_release(nimbus_ctx* ctx) {
    if (ctx && ctx->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) ctx_free(ctx);
}

void nimbus_ctx_destroy(nimbus_ctx* ctx) { ctx_release(ctx); }

static void ctx_free(nimbus_ctx* ctx) {
    DevGuard dg_(ctx, "nimbus_ctx_destroy");
    if (ctx->d_tw) cudaFree(ctx->d_tw);
    if (ctx->d_scratch) cudaFree(ctx->d_scratch);
    if (ctx->d_flag) cudaFree(ctx->d_flag);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->ev_pending) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->sync_ev) cudaEventDestroy(e);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    for (cudaEvent_t e : ctx->stream_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->host_ev) cudaEventDestroy(e);
    for (uint8_t* h : ctx->h_read) if (h) cudaFreeHost(h);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    delete ctx;
}

nimbus_status nimbus_ctx_primes(const nimbus_ctx* ctx, uint32_t* out) {
    if (!ctx || !out) return NIMBUS_EINVAL;
    for (uint32_t i = 0; i < ctx->rns.L; i++) out[i] = ctx->rns.p[i];
    return NIMBUS_OK;
}

const char* nimbus_last_error(const nimbus_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

uint64_t nimbus_launch_count(const nimbus_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* nimbus_last_contraction(const nimbus_ctx* ctx) { return ctx ? ctx->last_contraction : ""; }

nimbus_status nimbus_cop_prefetch_next(nimbus_ctx* ctx, const nimbus_encw* next) {
    if (!ctx || (next && next->ctx != ctx)) return NIMBUS_EINVAL;
    ctx->pf_next = next;
    return NIMBUS_OK;
}

nimbus_status nimbus_sync(nimbus_ctx* ctx, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (!ctx) return NIMBUS_EINVAL;
    CK(cudaStreamSynchronize((cudaStream_t)stream), "sync");
    if (ctx->io_error.exchange(0)) return set_err(ctx, NIMBUS_EIO, "reading a file-backed Enc(W) failed");
    uint32_t flag = 0;
    CK(cudaMemcpy(&flag, ctx->d_flag, 4, cudaMemcpyDeviceToHost), "sync flag");
    if (flag) {
        CK(cudaMemset(ctx->d_flag, 0, 4), "sync flag reset");
        return set_err(ctx, NIMBUS_ERANGE, "an input entry was >= t");
    }
    return NIMBUS_OK;
}

// ---------------------------------------------------------------- keys
nimbus_status nimbus_keygen(nimbus_ctx* ctx, uint64_t seed, void* stream, nimbus_sk** out) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !out) return NIMBUS_EINVAL;
    *out = nullptr;
    nimbus_sk* sk = new (std::nothrow) nimbus_sk();
    if (!sk) return NIMBUS_ENOMEM;
    sk->ctx = ctx;
    ctx_retain(ctx);
    const uint32_t N = ctx->rns.N, L = ctx->rns.L;
    cudaError_t e = cudaMalloc(&sk->d_s, N);
    if (e == cudaSuccess) e = cudaMalloc(&sk->d_s_ntt, (size_t)L * N * 4);
    if (e == cudaSuccess) e = launch_keygen(ctx, seed, sk->d_s, sk->d_s_ntt, (cudaStream_t)stream);
    if (e == cudaSuccess && (N == 4096 || N == 8192)) {
        // s_hat in the fused encrypt kernel's thread order, with Shoup companions (encrypt.cu)
        e = cudaMalloc(&sk->d_s_enc, (size_t)2 * L * N * 4);
        if (e == cudaSuccess) e = launch_perm_s(ctx, sk->d_s_ntt, sk->d_s_enc, (cudaStream_t)stream);
    }
    if (e != cudaSuccess) { nimbus_sk_destroy(sk); return cuda_err(ctx, e, "keygen"); }
    *out = sk;
    return NIMBUS_OK;
}

void nimbus_sk_destroy(nimbus_sk* sk) {
    DevGuard dg_(sk ? sk->ctx : nullptr, __func__);
    if (!sk) return;
    if (sk->d_s) cudaFree(sk->d_s);
    if (sk->d_s_ntt) cudaFree(sk->d_s_ntt);
    if (sk->d_s_enc) cudaFree(sk->d_s_enc);
    nimbus_ctx* ctx = sk->ctx;
    delete sk;
    ctx_release(ctx);
}

nimbus_status nimbus_sk_export(const nimbus_sk* sk, int8_t* d_s, void* stream) {
    DevGuard dg_(sk ? sk->ctx : nullptr, __func__);
    if (!sk || !d_s) return NIMBUS_EINVAL;
    nimbus_ctx* ctx = sk->ctx;
    CK(cudaMemcpyAsync(d_s, sk->d_s, ctx->rns.N, cudaMemcpyDeviceToDevice, (cudaStream_t)stream), "sk export");
    return NIMBUS_OK;
}

// ---------------------------------------------------------------- public key (reading 25)
nimbus_status nimbus_keygen_pk(nimbus_ctx* ctx, const nimbus_sk* sk, uint64_t seed, void* stream, nimbus_pk** out) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !sk || !out || sk->ctx != ctx) return set_err(ctx, NIMBUS_EINVAL, "null argument");
    *out = nullptr;
    nimbus_pk* pk = new (std::nothrow) nimbus_pk();
    if (!pk) return NIMBUS_ENOMEM;
    pk->ctx = ctx;
    ctx_retain(ctx);
    const size_t words = 2ull * ctx->rns.L * ctx->rns.N;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMalloc(&pk->d_pk, words * 4);
    if (e == cudaSuccess) e = cudaMalloc(&pk->d_pk_ntt, words * 4);
    if (e == cudaSuccess) e = launch_keygen_pk(ctx, sk->d_s_ntt, seed, pk->d_pk, st);
    if (e == cudaSuccess) e = launch_ntt_rows(ctx, pk->d_pk, 2, pk->d_pk_ntt, st);
    if (e != cudaSuccess) { nimbus_pk_destroy(pk); return cuda_err(ctx, e, "keygen_pk"); }
    *out = pk;
    return NIMBUS_OK;
}

void nimbus_pk_destroy(nimbus_pk* pk) {
    DevGuard dg_(pk ? pk->ctx : nullptr, __func__);
    if (!pk) return;
    if (pk->d_pk) cudaFree(pk->d_pk);
    if (pk->d_pk_ntt) cudaFree(pk->d_pk_ntt);
    nimbus_ctx* ctx = pk->ctx;
    delete pk;
    ctx_release(ctx);
}

nimbus_status nimbus_pk_export(const nimbus_pk* pk, uint32_t* d_out, void* stream) {
    DevGuard dg_(pk ? pk->ctx : nullptr, __func__);
    if (!pk || !d_out) return NIMBUS_EINVAL;
    nimbus_ctx* ctx = pk->ctx;
    CK(cudaMemcpyAsync(d_out, pk->d_pk, 2ull * ctx->rns.L * ctx->rns.N * 4, cudaMemcpyDeviceToDevice,
                       (cudaStream_t)stream), "pk export");
    return NIMBUS_OK;
}

nimbus_status nimbus_pk_import(nimbus_ctx* ctx, const uint32_t* d_in, void* stream, nimbus_pk** out) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !d_in || !out) return set_err(ctx, NIMBUS_EINVAL, "null argument");
    *out = nullptr;
    nimbus_pk* pk = new (std::nothrow) nimbus_pk();
    if (!pk) return NIMBUS_ENOMEM;
    pk->ctx = ctx;
    ctx_retain(ctx);
    const size_t words = 2ull * ctx->rns.L * ctx->rns.N;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMalloc(&pk->d_pk, words * 4);
    if (e == cudaSuccess) e = cudaMalloc(&pk->d_pk_ntt, words * 4);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pk->d_pk, d_in, words * 4, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = launch_ntt_rows(ctx, pk->d_pk, 2, pk->d_pk_ntt, st);
    if (e != cudaSuccess) { nimbus_pk_destroy(pk); return cuda_err(ctx, e, "pk import"); }
    *out = pk;
    return NIMBUS_OK;
}

// ---------------------------------------------------------------- Enc(W)
static nimbus_status new_encw(nimbus_ctx* ctx, uint32_t m, uint32_t n, nimbus_encw** out, bool alloc = true) {
    if (m == 0 || n == 0) return set_err(ctx, NIMBUS_EINVAL, "m and n must be positive");
    if (n > ctx->rns.N) return set_err(ctx, NIMBUS_ESHAPE, "n > N (PAPER.md:232 needs n < N)");
    if (m > 8192) return set_err(ctx, NIMBUS_ESHAPE, "m > 8192 exceeds the int32 slice-accumulator bound");
    // ell > 32: the 11 shifted accumulators, 7 of them scaled by 2^(8s) mod p, must sum below 2^64
    if (ctx->rns.ell > 32 && m > 4096) return set_err(ctx, NIMBUS_ESHAPE, "m > 4096 at ell > 32 (64-bit recombination)");
    if (!noise_ok(ctx, m, 1)) return set_err(ctx, NIMBUS_ENOISE, "parameters fail the decryption noise bound");
    nimbus_encw* w = new (std::nothrow) nimbus_encw();
    if (!w) return NIMBUS_ENOMEM;
    w->ctx = ctx; w->m = m; w->n = n; w->KB = (m + kBK - 1) / kBK;
    // resident-X kernel (tcgen05, ell <= 16, m <= 768) uses 32-column tiles, the streaming kernel 48.
    // The transposed ell = 32 kernel (128-column tiles) is chosen by NIMBUS_FLAG_LARGE_K (or
    // NIMBUS_TRANSPOSED=1): 2.7% faster at C5 (k = 2048) but 7% slower at C4 (k = 128: 768 work
    // units = 5.19 waves on 148 SMs), and the layout is fixed before k is known.  At ell <= 16 the
    // same hint selects it too (ahead of the resident-X layout): there it feeds the packed
    // contraction at S_x = 2 (the C5@l16 pass) and k_cop_tc_t<2, 64> otherwise.
    w->bn = kBNT;
    if (ctx->prm.impl == NIMBUS_IMPL_TCGEN05) {
        const char* tr = getenv("NIMBUS_TRANSPOSED");
        const bool large_k = (ctx->prm.flags & NIMBUS_FLAG_LARGE_K) || (tr && atoi(tr) == 1);
        const uint32_t sx = sx_of(ctx->rns.ell);
        if ((sx == 4 || sx == 2) && ctx->rns.N >= kBNW && large_k) w->bn = kBNW;
        else if (sx == 2 && w->KB <= kResMaxKB && !getenv("NIMBUS_NO_RESIDENT")) w->bn = kBNR;
        else if (sx_of(ctx->rns.ell) == 8) w->bn = kBNW;      // 8 X slices: transposed kernel only
    }
    w->bytes = (size_t)w->KB * kBK * col_tiles(ctx, w->bn) * w->bn * 4;
    if (alloc) {
        cudaError_t e = cudaMalloc(&w->d_Et, w->bytes);
        if (e != cudaSuccess) { delete w; return cuda_err(ctx, e, "encw alloc"); }
    }
    if (packed_layout_ok(ctx, w)) {
        // the packed contraction's complement correction (cop_pk.cu): corr + ColSum, 2 x 2LN residues
        cudaError_t e = cudaMalloc(&w->d_corr, 2 * ncols(ctx) * 4);
        if (e != cudaSuccess) { if (w->d_Et) cudaFree(w->d_Et); delete w; return cuda_err(ctx, e, "encw corr alloc"); }
    }
    ctx_retain(ctx);
    *out = w;
    return NIMBUS_OK;
}

// the element width at the boundary follows ell: uint32 up to 32 bits, uint64 beyond
static nimbus_status want_width(nimbus_ctx* ctx, uint32_t bytes) {
    if (!ctx) return NIMBUS_EINVAL;
    if (elem_bytes(ctx->rns.ell) != bytes)
        return set_err(ctx, NIMBUS_EINVAL, bytes == 4 ? "ell > 32: use the _u64 entry point"
                                                      : "ell <= 32: use the 32-bit entry point");
    return NIMBUS_OK;
}

// encrypt straight into w's resident planes (encrypt.cu, N = 4096 / 8192); other ring degrees:
// canonical rows (stream-ordered temporary) then tile (the canonical rows go to the context's
// grow-only scratch: a fresh 50-600 MB allocation per call costs more than the kernels; calls on
// a context are serialised)
static cudaError_t encrypt_into(nimbus_ctx* ctx, const nimbus_sk* sk, const void* d_W, uint64_t seed,
                                cudaStream_t s, nimbus_encw* w) {
    if (sk->d_s_enc && encrypt_planes_ok(ctx)) {
        cudaError_t e = launch_encrypt_planes(ctx, sk->d_s_enc, d_W, w->m, w->n, seed, w->KB, w->bn, w->d_Et, s);
        if (e == cudaSuccess) e = launch_pk_corr(ctx, w, s);
        return e;
    }
    const size_t need = (size_t)w->m * ncols(ctx) * 4;
    if (ctx->scratch_bytes < need) {
        cudaError_t e = cudaStreamSynchronize(s);         // earlier work may still use the old scratch
        if (e != cudaSuccess) return e;
        if (ctx->d_scratch) cudaFree(ctx->d_scratch);
        ctx->d_scratch = nullptr;
        ctx->scratch_bytes = 0;
        e = cudaMalloc(&ctx->d_scratch, need);
        if (e != cudaSuccess) return e;
        ctx->scratch_bytes = need;
    }
    uint32_t* canon = static_cast<uint32_t*>(ctx->d_scratch);
    cudaError_t e = launch_encrypt(ctx, sk->d_s_ntt, d_W, w->m, w->n, seed, canon, s);
    if (e == cudaSuccess) e = launch_tile_encw(ctx, canon, w->m, w->KB, w->bn, w->d_Et, s);
    if (e == cudaSuccess) e = launch_pk_corr(ctx, w, s);
    return e;
}

static nimbus_status encrypt_weights(nimbus_ctx* ctx, const nimbus_sk* sk, const void* d_W, uint32_t m,
                                     uint32_t n, uint64_t seed, void* stream, nimbus_encw** out) {
    if (!ctx || !sk || !d_W || !out || sk->ctx != ctx) return set_err(ctx, NIMBUS_EINVAL, "null argument");
    *out = nullptr;
    nimbus_encw* w = nullptr;
    nimbus_status st = new_encw(ctx, m, n, &w);
    if (st != NIMBUS_OK) return st;
    cudaError_t e = encrypt_into(ctx, sk, d_W, seed, (cudaStream_t)stream, w);
    if (e != cudaSuccess) { nimbus_encw_destroy(w); return cuda_err(ctx, e, "encrypt_weights"); }
    *out = w;
    return NIMBUS_OK;
}

static nimbus_status reencrypt_weights(nimbus_ctx* ctx, const nimbus_sk* sk, const void* d_W, uint64_t seed,
                                       void* stream, nimbus_encw* w) {
    if (!ctx || !sk || !d_W || !w || sk->ctx != ctx || w->ctx != ctx) return set_err(ctx, NIMBUS_EINVAL, "null argument");
    if (!w->d_Et) return set_err(ctx, NIMBUS_EINVAL, "Enc(W) is host-resident: nimbus_encw_reload first");
    CK(encrypt_into(ctx, sk, d_W, seed, (cudaStream_t)stream, w), "encrypt_weights_into");
    return NIMBUS_OK;
}

nimbus_status nimbus_encrypt_weights_into(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_W, uint64_t seed,
                                          void* stream, nimbus_encw* encw) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st : reencrypt_weights(ctx, sk, d_W, seed, stream, encw);
}

nimbus_status nimbus_encrypt_weights_into_u64(nimbus_ctx* ctx, const nimbus_sk* sk, const uint64_t* d_W,
                                              uint64_t seed, void* stream, nimbus_encw* encw) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 8);
    return st != NIMBUS_OK ? st : reencrypt_weights(ctx, sk, d_W, seed, stream, encw);
}


nimbus_status nimbus_encrypt_weights(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_W, uint32_t m,
                                     uint32_t n, uint64_t seed, void* stream, nimbus_encw** out) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st : encrypt_weights(ctx, sk, d_W, m, n, seed, stream, out);
}

nimbus_status nimbus_encrypt_weights_u64(nimbus_ctx* ctx, const nimbus_sk* sk, const uint64_t* d_W, uint32_t m,
                                         uint32_t n, uint64_t seed, void* stream, nimbus_encw** out) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 8);
    return st != NIMBUS_OK ? st : encrypt_weights(ctx, sk, d_W, m, n, seed, stream, out);
}

void nimbus_encw_destroy(nimbus_encw* w) {
    DevGuard dg_(w ? w->ctx : nullptr, __func__);
    if (!w) return;
    if (w->d_Et) cudaFree(w->d_Et);
    if (w->d_corr) cudaFree(w->d_corr);
    if (w->h_Et) cudaFreeHost(w->h_Et);
    nimbus_ctx* ctx = w->ctx;
    if (ctx && ctx->pf_next == w) ctx->pf_next = nullptr;     // a pending prefetch hint must not outlive its Enc(W)
    delete w;
    ctx_release(ctx);
}

static bool read_at(const char* path, uint64_t off, uint8_t* dst, uint64_t bytes);
static nimbus_status payload_to_device(nimbus_ctx* ctx, nimbus_encw* w, const uint8_t* host, uint64_t nbytes);

nimbus_status nimbus_encw_offload(nimbus_encw* w, void* stream) {
    DevGuard dg_(w ? w->ctx : nullptr, __func__);
    if (!w) return NIMBUS_EINVAL;
    nimbus_ctx* ctx = w->ctx;
    if (!w->d_Et) return NIMBUS_OK;                       // already host-resident
    cudaStream_t s = (cudaStream_t)stream;
    if (!w->h_Et) CK(cudaMallocHost(&w->h_Et, w->bytes), "pinned host alloc");
    CK(cudaMemcpyAsync(w->h_Et, w->d_Et, w->bytes, cudaMemcpyDeviceToHost, s), "offload copy");
    CK(cudaStreamSynchronize(s), "offload sync");
    CK(cudaFree(w->d_Et), "offload free");
    w->d_Et = nullptr;
    return NIMBUS_OK;
}

nimbus_status nimbus_encw_reload(nimbus_encw* w, void* stream) {
    DevGuard dg_(w ? w->ctx : nullptr, __func__);
    if (!w) return NIMBUS_EINVAL;
    nimbus_ctx* ctx = w->ctx;
    if (w->d_Et) return NIMBUS_OK;
    if (!w->h_Et && !w->file.empty()) {                   // file-backed: read, upload, tile
        std::vector<uint8_t> host(w->canon_bytes);
        if (!read_at(w->file.c_str(), w->file_off, host.data(), w->canon_bytes))
            return set_err(ctx, NIMBUS_EIO, "cannot read the store file");
        return payload_to_device(ctx, w, host.data(), w->canon_bytes);
    }
    CK(cudaMalloc(&w->d_Et, w->bytes), "reload alloc");
    CK(cudaMemcpyAsync(w->d_Et, w->h_Et, w->bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream), "reload copy");
    return NIMBUS_OK;
}

int nimbus_encw_is_resident(const nimbus_encw* w) { return w && w->d_Et ? 1 : 0; }

size_t nimbus_encw_bytes(const nimbus_encw* w) { return w ? w->bytes : 0; }

nimbus_status nimbus_encw_export(const nimbus_encw* w, uint32_t* d_out, void* stream) {
    DevGuard dg_(w ? w->ctx : nullptr, __func__);
    if (!w || !d_out) return NIMBUS_EINVAL;
    nimbus_ctx* ctx = w->ctx;
    if (!w->d_Et) return set_err(ctx, NIMBUS_EINVAL, "Enc(W) is host-resident (nimbus_encw_reload first)");
    CK(launch_untile_encw(ctx, w->d_Et, w->m, w->KB, w->bn, d_out, (cudaStream_t)stream), "encw export");
    return NIMBUS_OK;
}

nimbus_status nimbus_encw_import(nimbus_ctx* ctx, const uint32_t* d_in, uint32_t m, uint32_t n, void* stream,
                                 nimbus_encw** out) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !d_in || !out) return set_err(ctx, NIMBUS_EINVAL, "null argument");
    *out = nullptr;
    nimbus_encw* w = nullptr;
    nimbus_status st = new_encw(ctx, m, n, &w);
    if (st != NIMBUS_OK) return st;
    cudaError_t e = launch_tile_encw(ctx, d_in, m, w->KB, w->bn, w->d_Et, (cudaStream_t)stream);
    if (e == cudaSuccess) e = launch_pk_corr(ctx, w, (cudaStream_t)stream);
    if (e != cudaSuccess) { nimbus_encw_destroy(w); return cuda_err(ctx, e, "encw import"); }
    *out = w;
    return NIMBUS_OK;
}

// ---------------------------------------------------------------- store file
static uint64_t fnv1a(const uint8_t* p, size_t n, uint64_t h = 0xcbf29ce484222325ULL) {
    for (size_t i = 0; i < n; i++) { h ^= p[i]; h *= 0x100000001b3ULL; }
    return h;
}

nimbus_status nimbus_encw_save(const nimbus_encw* w, const char* path) {
    if (!w || !path) return NIMBUS_EINVAL;
    nimbus_ctx* ctx = w->ctx;
    DevGuard dg_(ctx, __func__);
    if (!w->d_Et) return set_err(ctx, NIMBUS_EINVAL, "Enc(W) is host-resident (nimbus_encw_reload first)");
    const size_t bytes = (size_t)w->m * ncols(ctx) * 4;
    uint32_t* d_canon = nullptr;
    CK(cudaMalloc(&d_canon, bytes), "save alloc");
    std::vector<uint8_t> host(bytes);
    cudaError_t e = launch_untile_encw(ctx, w->d_Et, w->m, w->KB, w->bn, d_canon, 0);
    if (e == cudaSuccess) e = cudaMemcpy(host.data(), d_canon, bytes, cudaMemcpyDeviceToHost);
    cudaFree(d_canon);
    CK(e, "save export");
    FILE* f = fopen(path, "wb");
    if (!f) return set_err(ctx, NIMBUS_EIO, "cannot open store file for writing");
    const uint32_t hdr[6] = {1u, ctx->rns.N, ctx->rns.L, ctx->rns.ell, w->m, w->n};
    const uint64_t nbytes = bytes, sum = fnv1a(host.data(), bytes);
    bool ok = fwrite("NIMBUSEW", 1, 8, f) == 8 && fwrite(hdr, 4, 6, f) == 6 &&
              fwrite(ctx->rns.p, 4, ctx->rns.L, f) == ctx->rns.L && fwrite(&nbytes, 8, 1, f) == 1 &&
              fwrite(host.data(), 1, bytes, f) == bytes && fwrite(&sum, 8, 1, f) == 1;
    ok = (fclose(f) == 0) && ok;
    return ok ? NIMBUS_OK : set_err(ctx, NIMBUS_EIO, "store file write failed");
}

// Store-file header (written by nimbus_encw_save): checks magic, version and that the file
// was made for this context's N, L, ell and primes; returns m, n, payload offset and bytes.
static bool read_store_header(const nimbus_ctx* ctx, FILE* f, uint32_t* m, uint32_t* n, uint64_t* off,
                              uint64_t* nbytes) {
    char magic[8];
    uint32_t hdr[6], pr[NIMBUS_MAXL];
    const bool ok = fread(magic, 1, 8, f) == 8 && memcmp(magic, "NIMBUSEW", 8) == 0 && fread(hdr, 4, 6, f) == 6 &&
                    hdr[0] == 1u && hdr[1] == ctx->rns.N && hdr[2] == ctx->rns.L && hdr[3] == ctx->rns.ell &&
                    fread(pr, 4, ctx->rns.L, f) == ctx->rns.L && memcmp(pr, ctx->rns.p, 4 * ctx->rns.L) == 0 &&
                    fread(nbytes, 8, 1, f) == 1 && hdr[4] > 0 && hdr[5] > 0 &&
                    *nbytes == (uint64_t)hdr[4] * ncols(ctx) * 4;
    *m = hdr[4];
    *n = hdr[5];
    *off = 8 + 24 + 4ull * ctx->rns.L + 8;
    return ok;
}

// read exactly `bytes` at `off` of `path` into `dst` (large reads, EINTR-safe); payloads over
// 64 MB are split over up to 8 threads (one pread stream per thread: from the page cache a
// single thread copies at ~6 GB/s)
static bool read_range(int fd, uint64_t off, uint8_t* dst, uint64_t bytes) {
    uint64_t done = 0;
    while (done < bytes) {
        const size_t chunk = (size_t)std::min<uint64_t>(bytes - done, 1ull << 30);
        const ssize_t r = pread(fd, dst + done, chunk, (off_t)(off + done));
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) return false;
        done += (uint64_t)r;
    }
    return true;
}

static bool read_at(const char* path, uint64_t off, uint8_t* dst, uint64_t bytes) {
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return false;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = bytes > (64ull << 20) ? std::min(8u, hw) : 1u;
    bool ok = true;
    if (nt == 1) {
        ok = read_range(fd, off, dst, bytes);
    } else {
        const uint64_t per = ((bytes + nt - 1) / nt + 4095) & ~uint64_t(4095);
        std::vector<std::thread> th;
        std::vector<char> res(nt, 1);
        for (unsigned t = 0; t < nt; t++) {
            const uint64_t b0 = std::min<uint64_t>(bytes, t * per), b1 = std::min<uint64_t>(bytes, b0 + per);
            if (b1 > b0) th.emplace_back([&, t, b0, b1] { res[t] = read_range(fd, off + b0, dst + b0, b1 - b0); });
        }
        for (auto& x : th) x.join();
        for (char r : res) ok = ok && r;
    }
    close(fd);
    return ok;
}

// canonical payload (host) -> a fresh tiled device copy in w->d_Et
static nimbus_status payload_to_device(nimbus_ctx* ctx, nimbus_encw* w, const uint8_t* host, uint64_t nbytes) {
    uint32_t* d_canon = nullptr;
    CK(cudaMalloc(&d_canon, nbytes), "load alloc");
    cudaError_t e = w->d_Et ? cudaSuccess : cudaMalloc(&w->d_Et, w->bytes);
    if (e == cudaSuccess) e = cudaMemcpy(d_canon, host, nbytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_tile_encw(ctx, d_canon, w->m, w->KB, w->bn, w->d_Et, nullptr);
    if (e == cudaSuccess) e = launch_pk_corr(ctx, w, nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(d_canon);
    return e == cudaSuccess ? NIMBUS_OK : cuda_err(ctx, e, "load import");
}

nimbus_status nimbus_encw_load(nimbus_ctx* ctx, const char* path, nimbus_encw** out) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !path || !out) return set_err(ctx, NIMBUS_EINVAL, "null argument");
    *out = nullptr;
    FILE* f = fopen(path, "rb");
    if (!f) return set_err(ctx, NIMBUS_EIO, "cannot open store file");
    uint32_t m = 0, n = 0;
    uint64_t off = 0, nbytes = 0, sum = 0;
    bool ok = read_store_header(ctx, f, &m, &n, &off, &nbytes);
    std::vector<uint8_t> host;
    if (ok) {
        host.resize(nbytes);
        ok = fread(host.data(), 1, nbytes, f) == nbytes && fread(&sum, 8, 1, f) == 1 &&
             sum == fnv1a(host.data(), nbytes);
    }
    fclose(f);
    if (!ok) return set_err(ctx, NIMBUS_EIO, "store file corrupt or made for other parameters");
    nimbus_encw* w = nullptr;
    nimbus_status st = new_encw(ctx, m, n, &w);
    if (st != NIMBUS_OK) return st;
    st = payload_to_device(ctx, w, host.data(), nbytes);
    if (st != NIMBUS_OK) { nimbus_encw_destroy(w); return st; }
    *out = w;
    return NIMBUS_OK;
}

nimbus_status nimbus_encw_open(nimbus_ctx* ctx, const char* path, int verify, nimbus_encw** out) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !path || !out) return set_err(ctx, NIMBUS_EINVAL, "null argument");
    *out = nullptr;
    FILE* f = fopen(path, "rb");
    if (!f) return set_err(ctx, NIMBUS_EIO, "cannot open store file");
    uint32_t m = 0, n = 0;
    uint64_t off = 0, nbytes = 0, sum = 0;
    bool ok = read_store_header(ctx, f, &m, &n, &off, &nbytes);
    // whole file present: payload + trailing checksum
    ok = ok && fseeko(f, 0, SEEK_END) == 0 && (uint64_t)ftello(f) == off + nbytes + 8;
    if (ok && verify) {                  // one streaming pass over the payload
        ok = fseeko(f, (off_t)off, SEEK_SET) == 0;
        std::vector<uint8_t> buf(64u << 20);
        uint64_t h = 0xcbf29ce484222325ULL, left = nbytes;
        while (ok && left) {
            const size_t c = (size_t)std::min<uint64_t>(left, buf.size());
            ok = fread(buf.data(), 1, c, f) == c;
            h = fnv1a(buf.data(), c, h);
            left -= c;
        }
        ok = ok && fread(&sum, 8, 1, f) == 1 && sum == h;
    }
    fclose(f);
    if (!ok) return set_err(ctx, NIMBUS_EIO, "store file corrupt, truncated or made for other parameters");
    nimbus_encw* w = nullptr;
    nimbus_status st = new_encw(ctx, m, n, &w, /*alloc=*/false);
    if (st != NIMBUS_OK) return st;
    w->file = path;
    w->file_off = off;
    w->canon_bytes = nbytes;
    *out = w;
    return NIMBUS_OK;
}

// ---------------------------------------------------------------- online path
// packed ciphertexts per query: ceil(k_q / floor(N/n))
static uint32_t cts_per_query(const nimbus_ctx* ctx, uint32_t kq, uint32_t n) {
    const uint32_t R = ctx->rns.N / n;
    return (kq + R - 1) / R;
}

nimbus_status nimbus_cop_out_count(const nimbus_ctx* ctx, uint32_t kq, uint32_t n, uint32_t nq, uint32_t* n_cts) {
    if (!ctx || !n_cts || kq == 0 || n == 0 || nq == 0) return NIMBUS_EINVAL;
    if (n > ctx->rns.N) return NIMBUS_ESHAPE;
    *n_cts = nq * cts_per_query(ctx, kq, n);
    return NIMBUS_OK;
}

struct WsLayout {
    size_t xt = 0, c = 0, stage_x = 0, stage_cts = 0, stage_r = 0, total = 0;
};
static WsLayout ws_layout(const nimbus_ctx* ctx, const nimbus_encw* w, uint32_t k) {
    auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
    WsLayout L;
    const size_t Mt = (k + kBM - 1) / kBM;
    const size_t xt_bytes = sx_of(ctx->rns.ell) * Mt * kBM * (size_t)w->KB * kBK;
    const size_t c_bytes = (size_t)k * ncols(ctx) * 4;
    L.xt = 0;
    L.c = al(xt_bytes);
    L.stage_x = L.c + al(c_bytes);
    const size_t es = elem_bytes(ctx->rns.ell);
    L.stage_cts = L.stage_x + al((size_t)k * w->m * es);
    L.stage_r = L.stage_cts + al((size_t)k * 2 * ctx->rns.L_out * ctx->rns.N * 4);
    L.total = L.stage_r + al((size_t)k * w->n * es);
    if (packed_layout_ok(ctx, w)) {
        // packed X slices (cop_pk.cu) at offset 0: room for ceil(k / R) packed ciphertexts plus one
        // per query boundary for up to 64 queries; cop_matmul falls back when a call needs more
        const uint64_t Rr = ctx->rns.N / w->n;
        size_t pk = 0;
        const uint32_t* cand;
        uint32_t ncand;
        packed_rt_candidates(ctx, &cand, &ncand);
        for (uint32_t i = 0; i < ncand; i++)
            pk = std::max(pk, 1024 + packed_xp_bytes(ctx, w, (k + Rr - 1) / Rr + 64, cand[i]));
        L.total = std::max(L.total, al(pk));
    }
    return L;
}

nimbus_status nimbus_cop_workspace_size(const nimbus_ctx* ctx, const nimbus_encw* w, uint32_t k, size_t* bytes) {
    if (!ctx || !w || !bytes || k == 0) return NIMBUS_EINVAL;
    *bytes = ws_layout(ctx, w, k).total;
    return NIMBUS_OK;
}

static nimbus_status check_shape(nimbus_ctx* ctx, const nimbus_encw* w, uint32_t kq, uint32_t nq) {
    if (!ctx || !w || w->ctx != ctx) return set_err(ctx, NIMBUS_EINVAL, "bad context / encw");
    if (kq == 0 || nq == 0) return set_err(ctx, NIMBUS_EINVAL, "k must be positive");
    if ((uint64_t)kq * nq > (1u << 24)) return set_err(ctx, NIMBUS_ESHAPE, "k too large");
    const uint32_t R = ctx->rns.N / w->n;
    if (!noise_ok(ctx, w->m, kq < R ? kq : R)) return set_err(ctx, NIMBUS_ENOISE, "noise bound violated");
    return NIMBUS_OK;
}
static nimbus_status check_online(nimbus_ctx* ctx, const nimbus_encw* w, uint32_t kq, uint32_t nq) {
    nimbus_status st = check_shape(ctx, w, kq, nq);
    if (st != NIMBUS_OK) return st;
    if (!w->d_Et) return set_err(ctx, NIMBUS_EINVAL, "Enc(W) is host-resident: use nimbus_cop_matmul_streamed");
    return NIMBUS_OK;
}

// stage events: ev[0] before slice, ev[1] after slice, ev[2] after contraction, ev[3] after pack
static cudaEvent_t prof_event(nimbus_ctx* ctx) {
    cudaEvent_t e;
    if (!ctx->ev_pool.empty()) { e = ctx->ev_pool.back(); ctx->ev_pool.pop_back(); }
    else cudaEventCreate(&e);
    ctx->ev_pending.push_back(e);
    return e;
}
static void prof_mark(nimbus_ctx* ctx, cudaStream_t s) {
    if (ctx->profile) cudaEventRecord(prof_event(ctx), s);
}

static nimbus_status run_accumulate(nimbus_ctx* ctx, const nimbus_encw* w, const void* d_X, uint32_t k,
                                    uint32_t* d_C, uint8_t* ws, cudaStream_t s) {
    if (ctx->prm.impl == NIMBUS_IMPL_TCGEN05) {
        uint8_t* xt = ws + ws_layout(ctx, w, k).xt;
        // X rows per tile: 128, or 256 / S_x in the transposed orientation
        const uint32_t rt = w->bn == kBNW ? transposed_rows(ctx) : kBM;
        CK(launch_slice_x(ctx, d_X, k, w->m, w->KB, rt, xt, s), "slice X");
        prof_mark(ctx, s);
        CK(launch_cop_tcgen05(ctx, w, xt, k, d_C, s), "cop tcgen05");
    } else {
        prof_mark(ctx, s);
        CK(launch_cop_cudacore(ctx, w, static_cast<const uint32_t*>(d_X), k, d_C, s), "cop cudacore");
    }
    return NIMBUS_OK;
}

nimbus_status nimbus_cop_accumulate(nimbus_ctx* ctx, const nimbus_encw* w, const uint32_t* d_X, uint32_t k,
                                    uint32_t* d_C, void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    if (st != NIMBUS_OK) return st;
    st = check_online(ctx, w, k, 1);
    if (st != NIMBUS_OK && st != NIMBUS_ENOISE) return st;
    if (!d_X || !d_C || !d_ws) return set_err(ctx, NIMBUS_EINVAL, "null buffer");
    if (ws_bytes < ws_layout(ctx, w, k).total) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    const bool pf = ctx->profile;
    ctx->profile = false;
    st = run_accumulate(ctx, w, d_X, k, d_C, (uint8_t*)d_ws, (cudaStream_t)stream);
    ctx->profile = pf;
    return st;
}

nimbus_status nimbus_cop_pack(nimbus_ctx* ctx, const uint32_t* d_C, uint32_t kq, uint32_t nq, uint32_t n,
                              uint64_t seed, uint32_t* d_cts, uint32_t* d_R, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (want_width(ctx, 4) != NIMBUS_OK) return NIMBUS_EINVAL;
    if (!ctx || !d_C || !d_cts || !d_R || kq == 0 || nq == 0 || n == 0) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    if (n > ctx->rns.N) return set_err(ctx, NIMBUS_ESHAPE, "n > N");
    CK(launch_pack(ctx, d_C, kq, nq, n, seed, d_cts, d_R, (cudaStream_t)stream, true), "pack");
    return NIMBUS_OK;
}

// allow_no_R: d_R may be null (the host-buffer call produces R separately)
static nimbus_status cop_matmul(nimbus_ctx* ctx, const nimbus_encw* w, const void* d_X, uint32_t kq,
                                uint32_t nq, uint64_t seed, uint32_t* d_cts, void* d_R, void* d_ws,
                                size_t ws_bytes, void* stream, bool allow_no_R = false,
                                const uint32_t* d_zero = nullptr) {
    nimbus_status st = check_online(ctx, w, kq, nq);
    if (st != NIMBUS_OK) return st;
    if (!d_X || !d_cts || (!d_R && !allow_no_R) || !d_ws) return set_err(ctx, NIMBUS_EINVAL, "null buffer");
    const uint32_t k = kq * nq;
    const WsLayout L = ws_layout(ctx, w, k);
    if (ws_bytes < L.total) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t* C = reinterpret_cast<uint32_t*>((uint8_t*)d_ws + L.c);
    prof_mark(ctx, s);
    // the fused epilogue stores cts and R with 16-byte vector stores: 16-byte aligned buffers only
    const bool aligned16 = (((uintptr_t)d_cts | (uintptr_t)d_R) & 15) == 0;
    if (!d_zero && packed_ok(ctx, w, kq, nq)) {
        // packed contraction: slice into the packed layout, then one kernel that writes the compact
        // output ciphertexts (mod-switch + mask in its epilogue) -- no C round trip, no pack launch
        PkHostJob J;
        J.w = w; J.d_X = static_cast<const uint32_t*>(d_X); J.kq = kq; J.nq = nq; J.seed = seed;
        J.d_cts = d_cts; J.d_R = static_cast<uint32_t*>(d_R); J.d_Xp = (const uint8_t*)d_ws + 1024;
        const uint32_t rt = packed_rt(ctx, &J, 1);
        if (1024 + packed_job_bytes(ctx, J, rt) <= ws_bytes) {
            // workspace: [dispatch counter | packed X slices | dropped-limb residues | flags]
            CK(launch_cop_packed(ctx, &J, 1, rt, static_cast<uint32_t*>(d_ws), s, prof_mark), "cop packed");
            prof_mark(ctx, s);      // after the contraction; the (empty) pack stage: two more marks
            prof_mark(ctx, s);
            prof_mark(ctx, s);
            return NIMBUS_OK;
        }
    }
    if (!d_zero && aligned16 && ctx->prm.impl == NIMBUS_IMPL_TCGEN05 && fused_r1_ok(ctx, w, k)) {
        // R = 1 (n > N/2): packing is the identity, the contraction's epilogue does the
        // mod-switch and the mask; no C round trip, no pack launch (the pack stage times 0)
        CK(launch_slice_x(ctx, d_X, k, w->m, w->KB, kBM, (uint8_t*)d_ws + L.xt, s), "slice X");
        prof_mark(ctx, s);
        CK(launch_cop_fused_r1(ctx, w, (uint8_t*)d_ws + L.xt, k, seed, d_cts, static_cast<uint32_t*>(d_R), s),
           "cop fused");
        prof_mark(ctx, s);
        prof_mark(ctx, s);
        prof_mark(ctx, s);
        return NIMBUS_OK;
    }
    st = run_accumulate(ctx, w, d_X, k, C, (uint8_t*)d_ws, s);
    if (st != NIMBUS_OK) return st;
    prof_mark(ctx, s);
    prof_mark(ctx, s);
    CK(launch_pack(ctx, C, kq, nq, w->n, seed, d_cts, d_R, s, true, d_zero), "pack");
    prof_mark(ctx, s);
    return NIMBUS_OK;
}

nimbus_status nimbus_cop_matmul(nimbus_ctx* ctx, const nimbus_encw* w, const uint32_t* d_X, uint32_t kq,
                                uint32_t nq, uint64_t seed, uint32_t* d_cts, uint32_t* d_R, void* d_ws,
                                size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st : cop_matmul(ctx, w, d_X, kq, nq, seed, d_cts, d_R, d_ws, ws_bytes, stream);
}

nimbus_status nimbus_cop_matmul_u64(nimbus_ctx* ctx, const nimbus_encw* w, const uint64_t* d_X, uint32_t kq,
                                    uint32_t nq, uint64_t seed, uint32_t* d_cts, uint64_t* d_R, void* d_ws,
                                    size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 8);
    return st != NIMBUS_OK ? st : cop_matmul(ctx, w, d_X, kq, nq, seed, d_cts, d_R, d_ws, ws_bytes, stream);
}

// ---------------------------------------------------------------- circuit privacy (reading 26)
static constexpr uint32_t kMaxFlood = 126;      // flooding noise in [-2^F, 2^F), F <= 126 (two PRG words)
// the zero encryption's noise bound, doubled: 2 |v e_pk + e1 + f - e2 s| <= 4 eta N + 2 eta + 2^(F+1)
static uint64_t rerand_extra2(const nimbus_ctx* ctx) { return 84ull * ctx->rns.N + 42; }
static uint32_t rerand_flood2(uint32_t F) { return F ? F + 1 : 0; }

nimbus_status nimbus_rerand_flood_max(const nimbus_ctx* ctx, const nimbus_encw* w, uint32_t kq, uint32_t* bits) {
    if (!ctx || !w || !bits || w->ctx != ctx || kq == 0) return NIMBUS_EINVAL;
    const uint32_t R = ctx->rns.N / w->n, Reff = kq < R ? kq : R;
    for (uint32_t F = kMaxFlood; F >= 1; F--)
        if (noise_ok(ctx, w->m, Reff, rerand_extra2(ctx), rerand_flood2(F))) { *bits = F; return NIMBUS_OK; }
    if (noise_ok(ctx, w->m, Reff, rerand_extra2(ctx), 0)) { *bits = 0; return NIMBUS_OK; }
    return NIMBUS_ENOISE;
}

nimbus_status nimbus_rerand_prepare(nimbus_ctx* ctx, const nimbus_pk* pk, const nimbus_encw* w, uint32_t kq,
                                    uint32_t nq, uint64_t seed, uint32_t flood_bits, uint32_t* d_zero,
                                    void* stream) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !pk || !w || !d_zero || pk->ctx != ctx) return set_err(ctx, NIMBUS_EINVAL, "null argument");
    nimbus_status st = check_shape(ctx, w, kq, nq);
    if (st != NIMBUS_OK) return st;
    if (flood_bits > kMaxFlood) return set_err(ctx, NIMBUS_EINVAL, "flood_bits > 126");
    const uint32_t R = ctx->rns.N / w->n, Reff = kq < R ? kq : R;
    if (!noise_ok(ctx, w->m, Reff, rerand_extra2(ctx), rerand_flood2(flood_bits)))
        return set_err(ctx, NIMBUS_ENOISE, "flooding noise exceeds the decryption bound (see nimbus_rerand_flood_max)");
    const uint32_t n_cts = nq * cts_per_query(ctx, kq, w->n);
    CK(launch_rerand(ctx, pk->d_pk_ntt, seed, n_cts, flood_bits, d_zero, (cudaStream_t)stream), "rerand");
    return NIMBUS_OK;
}

nimbus_status nimbus_cop_matmul_rr(nimbus_ctx* ctx, const nimbus_encw* w, const uint32_t* d_X, uint32_t kq,
                                   uint32_t nq, uint64_t seed, const uint32_t* d_zero, uint32_t* d_cts,
                                   uint32_t* d_R, void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (!d_zero) return set_err(ctx, NIMBUS_EINVAL, "null zero encryptions");
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st
                           : cop_matmul(ctx, w, d_X, kq, nq, seed, d_cts, d_R, d_ws, ws_bytes, stream, false, d_zero);
}

nimbus_status nimbus_cop_matmul_rr_u64(nimbus_ctx* ctx, const nimbus_encw* w, const uint64_t* d_X, uint32_t kq,
                                       uint32_t nq, uint64_t seed, const uint32_t* d_zero, uint32_t* d_cts,
                                       uint64_t* d_R, void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (!d_zero) return set_err(ctx, NIMBUS_EINVAL, "null zero encryptions");
    nimbus_status st = want_width(ctx, 8);
    return st != NIMBUS_OK ? st
                           : cop_matmul(ctx, w, d_X, kq, nq, seed, d_cts, d_R, d_ws, ws_bytes, stream, false, d_zero);
}

// ---------------------------------------------------------------- batched online path
static size_t al1k(size_t x) { return (x + 1023) & ~size_t(1023); }

// the batch as one packed job list (cop_pk.cu) when every job qualifies: the packed X slices of
// all jobs side by side in the workspace, one slice launch and one contraction launch in total
static bool batch_packed(const nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count,
                         std::vector<PkHostJob>* out, uint32_t* rt, size_t* bytes) {
    std::vector<PkHostJob> v(count);
    for (uint32_t i = 0; i < count; i++) {
        const nimbus_cop_job& J = jobs[i];
        if (!J.encw || !packed_ok(ctx, J.encw, J.k_per_query, J.n_queries)) return false;
        v[i].w = J.encw; v[i].d_X = J.d_X; v[i].kq = J.k_per_query; v[i].nq = J.n_queries;
        v[i].seed = J.mask_seed; v[i].d_cts = J.d_cts; v[i].d_R = J.d_R;
    }
    *rt = packed_rt(ctx, v.data(), count);
    size_t off = 1024;                                              // [0, 1024): dispatch counter
    for (uint32_t i = 0; i < count; i++) {
        v[i].d_Xp = reinterpret_cast<const uint8_t*>(off);          // offset; rebased by the caller
        off += al1k(packed_job_bytes(ctx, v[i], *rt));
    }
    *bytes = off;
    if (out) out->swap(v);
    return true;
}

// Same-X groups (Q, K, V of a layer share their input): consecutive jobs with the
// same X pointer and shape whose contraction is the resident-X kernel run as ONE contraction
// launch over their Enc(W)s and one pack launch.  Returns the group length at job i (1 = alone).
static bool groupable(const nimbus_ctx* ctx, const nimbus_encw* w, uint32_t k) {
    return w && w->d_Et && ctx->prm.impl == NIMBUS_IMPL_TCGEN05 && ctx->res_ring == 1 && resident_ok(ctx, w, k) &&
           !fused_r1_ok(ctx, w, k) && !getenv("NIMBUS_NO_GROUP");
}

// the group length at job i: consecutive jobs with the same X pointer (device X here, host X in
// same_hx_group) and shape, at most 4
static uint32_t same_x_group(const nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count, uint32_t i) {
    const nimbus_cop_job& A = jobs[i];
    const uint32_t k = A.k_per_query * A.n_queries;
    if (!groupable(ctx, A.encw, k)) return 1;
    uint32_t g = 1;
    while (g < 4 && i + g < count) {
        const nimbus_cop_job& B = jobs[i + g];
        if (B.d_X != A.d_X || B.k_per_query != A.k_per_query || B.n_queries != A.n_queries || !B.encw ||
            B.encw->m != A.encw->m || B.encw->n != A.encw->n || !groupable(ctx, B.encw, k))
            break;
        g++;
    }
    return g;
}

static uint32_t same_hx_group(const nimbus_ctx* ctx, const nimbus_cop_host_job* jobs, uint32_t count, uint32_t i) {
    const nimbus_cop_host_job& A = jobs[i];
    const uint32_t k = A.k_per_query * A.n_queries;
    if (!groupable(ctx, A.encw, k)) return 1;
    uint32_t g = 1;
    while (g < 4 && i + g < count) {
        const nimbus_cop_host_job& B = jobs[i + g];
        if (B.h_X != A.h_X || B.k_per_query != A.k_per_query || B.n_queries != A.n_queries || !B.encw ||
            B.encw->m != A.encw->m || B.encw->n != A.encw->n || !groupable(ctx, B.encw, k))
            break;
        g++;
    }
    return g;
}

// one slice of the group's shared X, ONE resident-X contraction over their Enc(W)s into C buffers
// 0..g-1, ONE pack launch, PDL-chained on stream a (ws: the X planes, then g C buffers of cbytes)
static cudaError_t run_x_group(nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t g, uint8_t* ws, size_t xt,
                               size_t cbytes, cudaStream_t a) {
    const nimbus_cop_job& J = jobs[0];
    const uint32_t k = J.k_per_query * J.n_queries;
    prof_mark(ctx, a);
    cudaError_t e = launch_slice_x(ctx, J.d_X, k, J.encw->m, J.encw->KB, kBM, ws, a);
    if (e != cudaSuccess) return e;
    prof_mark(ctx, a);
    ResJobs RJ;
    PackJobs PJ;
    RJ.nj = PJ.nj = g;
    for (uint32_t q = 0; q < g; q++) {
        uint32_t* C = reinterpret_cast<uint32_t*>(ws + xt + q * cbytes);
        RJ.Et[q] = jobs[q].encw->d_Et;
        RJ.C[q] = C;
        PJ.C[q] = C;
        PJ.cts[q] = jobs[q].d_cts;
        PJ.R[q] = jobs[q].d_R;
        PJ.key[q] = prg_key(jobs[q].mask_seed, 6);
    }
    e = launch_res_jobs(ctx, RJ, J.encw->KB, ws, k, a);
    if (e != cudaSuccess) return e;
    prof_mark(ctx, a);
    prof_mark(ctx, a);
    e = launch_pack_jobs(ctx, PJ, J.k_per_query, J.n_queries, J.encw->n, a, true);
    prof_mark(ctx, a);
    return e;
}

nimbus_status nimbus_cop_workspace_size_batch(const nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count,
                                              size_t* bytes) {
    if (!ctx || !jobs || !bytes || count == 0) return NIMBUS_EINVAL;
    size_t xt = 0, c = 0;
    for (uint32_t i = 0; i < count; i++) {
        if (!jobs[i].encw) return NIMBUS_EINVAL;
        const uint32_t k = jobs[i].k_per_query * jobs[i].n_queries;
        const WsLayout L = ws_layout(ctx, jobs[i].encw, k);
        xt = xt > L.c ? xt : L.c;                                   // X planes (1 KB aligned)
        const size_t cb = al1k((size_t)k * ncols(ctx) * 4);
        c = c > cb ? c : cb;
    }
    uint32_t nbuf = 2;                                              // C buffers: 2, or the largest group
    for (uint32_t i = 0; i < count;) {
        const uint32_t g = same_x_group(ctx, jobs, count, i);
        nbuf = std::max(nbuf, g);
        i += g;
    }
    *bytes = xt + nbuf * c;
    uint32_t rt = 0;
    size_t pk = 0;
    if (batch_packed(ctx, jobs, count, nullptr, &rt, &pk)) *bytes = std::max(*bytes, pk);
    return NIMBUS_OK;
}

// element-width-agnostic: d_X / d_R are passed through untouched (uint64 when ell > 32)
static nimbus_status cop_matmul_batch(nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count, void* d_ws,
                                      size_t ws_bytes, void* stream) {
    if (!ctx || !jobs || count == 0 || !d_ws) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    for (uint32_t i = 0; i < count; i++) {
        nimbus_status st = check_online(ctx, jobs[i].encw, jobs[i].k_per_query, jobs[i].n_queries);
        if (st != NIMBUS_OK) return st;
        if (!jobs[i].d_X || !jobs[i].d_cts || !jobs[i].d_R) return set_err(ctx, NIMBUS_EINVAL, "null buffer");
    }
    size_t need = 0;
    nimbus_cop_workspace_size_batch(ctx, jobs, count, &need);
    if (ws_bytes < need) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    {
        std::vector<PkHostJob> pj;
        uint32_t rt = 0;
        size_t pk = 0;
        if (batch_packed(ctx, jobs, count, &pj, &rt, &pk)) {
            cudaStream_t a = (cudaStream_t)stream;
            for (auto& j : pj) j.d_Xp = (const uint8_t*)d_ws + reinterpret_cast<uintptr_t>(j.d_Xp);
            prof_mark(ctx, a);
            CK(launch_cop_packed(ctx, pj.data(), count, rt, static_cast<uint32_t*>(d_ws), a,
                                 count <= 128 ? prof_mark : nullptr), "cop packed batch");
            if (count > 128) prof_mark(ctx, a);
            prof_mark(ctx, a);
            prof_mark(ctx, a);
            prof_mark(ctx, a);
            return NIMBUS_OK;
        }
    }
    size_t xt = 0;
    for (uint32_t i = 0; i < count; i++) {
        const WsLayout L = ws_layout(ctx, jobs[i].encw, jobs[i].k_per_query * jobs[i].n_queries);
        xt = xt > L.c ? xt : L.c;
    }
    size_t cbytes = 0;
    for (uint32_t i = 0; i < count; i++)
        cbytes = std::max(cbytes, al1k((size_t)jobs[i].k_per_query * jobs[i].n_queries * ncols(ctx) * 4));
    uint8_t* ws = (uint8_t*)d_ws;
    uint32_t* Cbuf[4];
    for (uint32_t b = 0; b < 4; b++) Cbuf[b] = reinterpret_cast<uint32_t*>(ws + xt + b * cbytes);
    cudaStream_t a = (cudaStream_t)stream;
    if (!ctx->side) CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "side stream");
    cudaStream_t b = ctx->side;
    while (ctx->sync_ev.size() < 2 * (size_t)count + 2) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        ctx->sync_ev.push_back(e);
    }
    cudaEvent_t* done_c = ctx->sync_ev.data();             // contraction i finished (stream a)
    cudaEvent_t* done_p = ctx->sync_ev.data() + count;     // pack i finished (stream b)
    cudaEvent_t start = ctx->sync_ev[2 * count];
    // the side stream must not start before earlier work on `stream`
    CK(cudaEventRecord(start, a), "record");
    CK(cudaStreamWaitEvent(b, start, 0), "wait");
    const nimbus_encw* after = ctx->pf_next;               // the caller's hint: what follows the list
    for (uint32_t i = 0; i < count; i++) {
        const nimbus_cop_job& J = jobs[i];
        const uint32_t k = J.k_per_query * J.n_queries;
        const uint32_t g = same_x_group(ctx, jobs, count, i);
        ctx->pf_next = i + g < count ? jobs[i + g].encw : after;   // the list names each unit's successor
        if (g > 1) {
            // one slice of the shared X, one contraction over the group's Enc(W)s into C buffers
            // 0..g-1, one pack launch, all on `stream` (PDL-chained); earlier packs on the side
            // stream may still read buffers 0 / 1
            if (i >= 1) CK(cudaStreamWaitEvent(a, done_p[i - 1], 0), "wait pack");
            if (i >= 2) CK(cudaStreamWaitEvent(a, done_p[i - 2], 0), "wait pack");
            CK(run_x_group(ctx, jobs + i, g, ws, xt, cbytes, a), "cop group");
            for (uint32_t q = 0; q < g; q++) {
                CK(cudaEventRecord(done_c[i + q], a), "record");
                CK(cudaEventRecord(done_p[i + q], a), "record");
            }
            i += g - 1;
            continue;
        }
        uint32_t* C = Cbuf[i & 1];
        // C[i%2] is free once the pack of job i-2 has read it
        if (i >= 2) CK(cudaStreamWaitEvent(a, done_p[i - 2], 0), "wait pack");
        prof_mark(ctx, a);
        nimbus_status st = run_accumulate(ctx, J.encw, J.d_X, k, C, ws, a);
        if (st != NIMBUS_OK) return st;
        prof_mark(ctx, a);
        CK(cudaEventRecord(done_c[i], a), "record");
        // pack of job i overlaps the contraction of job i+1 (memory- vs tensor-bound)
        CK(cudaStreamWaitEvent(b, done_c[i], 0), "wait contraction");
        prof_mark(ctx, b);
        CK(launch_pack(ctx, C, J.k_per_query, J.n_queries, J.encw->n, J.mask_seed, J.d_cts, J.d_R, b, false),
           "pack");
        prof_mark(ctx, b);
        CK(cudaEventRecord(done_p[i], b), "record");
    }
    CK(cudaStreamWaitEvent(a, done_p[count - 1], 0), "join");   // everything complete in `stream` order
    return NIMBUS_OK;
}

// the _u64 job list viewed as the 32-bit one (same layout; the pointers are passed through)
static std::vector<nimbus_cop_job> jobs_of(const nimbus_cop_job_u64* jobs, uint32_t count) {
    std::vector<nimbus_cop_job> v(count);
    for (uint32_t i = 0; i < count; i++)
        v[i] = {jobs[i].encw, reinterpret_cast<const uint32_t*>(jobs[i].d_X), jobs[i].k_per_query,
                jobs[i].n_queries, jobs[i].mask_seed, jobs[i].d_cts, reinterpret_cast<uint32_t*>(jobs[i].d_R)};
    return v;
}

nimbus_status nimbus_cop_matmul_batch(nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count, void* d_ws,
                                      size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st : cop_matmul_batch(ctx, jobs, count, d_ws, ws_bytes, stream);
}

nimbus_status nimbus_cop_workspace_size_batch_u64(const nimbus_ctx* ctx, const nimbus_cop_job_u64* jobs,
                                                  uint32_t count, size_t* bytes) {
    if (!ctx || !jobs || !bytes || count == 0) return NIMBUS_EINVAL;
    const std::vector<nimbus_cop_job> v = jobs_of(jobs, count);
    return nimbus_cop_workspace_size_batch(ctx, v.data(), count, bytes);
}

nimbus_status nimbus_cop_matmul_batch_u64(nimbus_ctx* ctx, const nimbus_cop_job_u64* jobs, uint32_t count,
                                          void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 8);
    if (st != NIMBUS_OK) return st;
    if (!jobs || count == 0) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    const std::vector<nimbus_cop_job> v = jobs_of(jobs, count);
    return cop_matmul_batch(ctx, v.data(), count, d_ws, ws_bytes, stream);
}

// ---------------------------------------------------------------- streamed path (Enc(W) in host memory)
nimbus_status nimbus_cop_stage_size(const nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count,
                                    size_t* bytes) {
    if (!ctx || !jobs || !bytes || count == 0) return NIMBUS_EINVAL;
    size_t mx = 0, mc = 0;
    for (uint32_t i = 0; i < count; i++) {
        if (!jobs[i].encw) return NIMBUS_EINVAL;
        const nimbus_encw* w = jobs[i].encw;
        if (!w->d_Et) mx = mx > w->bytes ? mx : w->bytes;
        if (!w->d_Et && !w->h_Et) mc = mc > w->canon_bytes ? mc : w->canon_bytes;   // file-backed
    }
    *bytes = 2 * al1k(mx) + al1k(mc);     // two tiled slots + one canonical buffer for file reads
    return NIMBUS_OK;
}

// stream-ordered read of a file-backed Enc(W) payload into a pinned buffer (cudaLaunchHostFunc)
struct FileRead {
    nimbus_ctx* ctx;
    std::string path;
    uint64_t off, bytes;
    uint8_t* dst;
};
static void CUDART_CB file_read_cb(void* p) {
    FileRead* r = static_cast<FileRead*>(p);
    if (!read_at(r->path.c_str(), r->off, r->dst, r->bytes)) r->ctx->io_error.store(1);
    delete r;
}

static nimbus_status cop_matmul_streamed(nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count, void* d_ws,
                                         size_t ws_bytes, void* d_stage, size_t stage_bytes, void* stream) {
    if (!ctx || !jobs || count == 0 || !d_ws) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    size_t need = 0;
    for (uint32_t i = 0; i < count; i++) {
        nimbus_status st = check_shape(ctx, jobs[i].encw, jobs[i].k_per_query, jobs[i].n_queries);
        if (st != NIMBUS_OK) return st;
        if (!jobs[i].d_X || !jobs[i].d_cts || !jobs[i].d_R) return set_err(ctx, NIMBUS_EINVAL, "null buffer");
        const size_t w = ws_layout(ctx, jobs[i].encw, jobs[i].k_per_query * jobs[i].n_queries).total;
        need = need > w ? need : w;
    }
    if (ws_bytes < need) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    if (ctx->io_error.exchange(0)) return set_err(ctx, NIMBUS_EIO, "an earlier file-backed Enc(W) read failed");
    size_t stage_need = 0;
    nimbus_cop_stage_size(ctx, jobs, count, &stage_need);
    if (stage_need && (!d_stage || stage_bytes < stage_need)) return set_err(ctx, NIMBUS_ESHAPE, "stage too small");
    size_t mx = 0, mc = 0;
    for (uint32_t i = 0; i < count; i++) {
        const nimbus_encw* w = jobs[i].encw;
        if (!w->d_Et) mx = std::max(mx, w->bytes);
        if (!w->d_Et && !w->h_Et) mc = std::max<size_t>(mc, w->canon_bytes);
    }
    const size_t slot = al1k(mx);
    uint32_t* d_canon = reinterpret_cast<uint32_t*>((uint8_t*)d_stage + 2 * slot);
    if (mc > ctx->h_read_bytes) {         // pinned read buffers (grow-only; none may be in flight)
        if (ctx->copy) CK(cudaStreamSynchronize(ctx->copy), "read buffers idle");
        for (uint8_t*& h : ctx->h_read) { if (h) cudaFreeHost(h); h = nullptr; }
        ctx->h_read_bytes = 0;
        for (uint8_t*& h : ctx->h_read) CK(cudaMallocHost(&h, mc), "pinned read buffer");
        ctx->h_read_bytes = mc;
    }
    uint32_t n_file = 0;
    cudaStream_t a = (cudaStream_t)stream;
    if (!ctx->copy) CK(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking), "copy stream");
    cudaStream_t b = ctx->copy;
    while (ctx->stream_ev.size() < 2 * (size_t)count + 1) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        ctx->stream_ev.push_back(e);
    }
    cudaEvent_t* loaded = ctx->stream_ev.data();           // Enc(W) of job i is in its slot (stream b)
    cudaEvent_t* used = ctx->stream_ev.data() + count;     // job i's kernels are done with its slot (stream a)
    // copies must not start before earlier work on `stream` that may still read the slots
    CK(cudaEventRecord(ctx->stream_ev[2 * count], a), "record");
    CK(cudaStreamWaitEvent(b, ctx->stream_ev[2 * count], 0), "wait");
    // host-resident jobs alternate between the two slots; job j's copy waits until the
    // job that last used its slot has finished, so copy j+1 overlaps the compute of job j
    std::vector<int> slot_of(count, -1), prev_user(count, -1);
    int last_user[2] = {-1, -1}, nh = 0;
    for (uint32_t i = 0; i < count; i++) {
        if (jobs[i].encw->d_Et) continue;
        const int sl = nh++ & 1;
        slot_of[i] = sl;
        prev_user[i] = last_user[sl];
        last_user[sl] = (int)i;
    }
    uint8_t* stage = (uint8_t*)d_stage;
    auto issue_copy = [&](uint32_t j) -> nimbus_status {
        const nimbus_encw* w = jobs[j].encw;
        if (prev_user[j] >= 0) CK(cudaStreamWaitEvent(b, used[prev_user[j]], 0), "wait slot");
        if (w->h_Et) {
            CK(cudaMemcpyAsync(stage + (size_t)slot_of[j] * slot, w->h_Et, w->bytes, cudaMemcpyHostToDevice, b),
               "stage copy");
        } else {
            // file-backed: read the canonical payload on the copy stream's host
            // callback into pinned buffer n_file % 2 (free again: its previous upload precedes this
            // callback on the same stream), upload it, and tile it into the slot
            uint8_t* hb = ctx->h_read[n_file++ & 1];
            FileRead* rd = new (std::nothrow) FileRead{ctx, w->file, w->file_off, w->canon_bytes, hb};
            if (!rd) return set_err(ctx, NIMBUS_ENOMEM, "host alloc");
            const cudaError_t e = cudaLaunchHostFunc(b, file_read_cb, rd);
            if (e != cudaSuccess) { delete rd; return cuda_err(ctx, e, "file read"); }
            CK(cudaMemcpyAsync(d_canon, hb, w->canon_bytes, cudaMemcpyHostToDevice, b), "stage upload");
            CK(launch_tile_encw(ctx, d_canon, w->m, w->KB, w->bn, stage + (size_t)slot_of[j] * slot, b), "stage tile");
        }
        CK(cudaEventRecord(loaded[j], b), "record");
        return NIMBUS_OK;
    };
    // prefetch the first two host-resident jobs (both slots are free)
    uint32_t issued = 0, n_issue = 0;
    for (uint32_t j = 0; j < count && n_issue < 2; j++)
        if (slot_of[j] >= 0) { nimbus_status st = issue_copy(j); if (st != NIMBUS_OK) return st; issued = j + 1; n_issue++; }
    if (n_issue < 2) issued = count;
    for (uint32_t i = 0; i < count; i++) {
        const nimbus_cop_job& J = jobs[i];
        nimbus_encw view = *J.encw;                        // same shape/layout, Enc(W) in its slot
        view.h_Et = nullptr;
        if (slot_of[i] >= 0) {
            view.d_Et = stage + (size_t)slot_of[i] * slot;
            CK(cudaStreamWaitEvent(a, loaded[i], 0), "wait load");
        }
        nimbus_status st = cop_matmul(ctx, &view, J.d_X, J.k_per_query, J.n_queries, J.mask_seed, J.d_cts,
                                      J.d_R, d_ws, ws_bytes, a);
        view.d_Et = nullptr;                               // the view owns nothing
        if (st != NIMBUS_OK) return st;
        CK(cudaEventRecord(used[i], a), "record");
        // next host-resident job not yet in flight: its slot frees when job i (or earlier) is done
        while (issued < count && slot_of[issued] < 0) issued++;
        if (issued < count && slot_of[i] >= 0) {
            nimbus_status st2 = issue_copy(issued);
            if (st2 != NIMBUS_OK) return st2;
            issued++;
        }
    }
    return NIMBUS_OK;
}

nimbus_status nimbus_cop_matmul_streamed(nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count, void* d_ws,
                                         size_t ws_bytes, void* d_stage, size_t stage_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st : cop_matmul_streamed(ctx, jobs, count, d_ws, ws_bytes, d_stage, stage_bytes, stream);
}

nimbus_status nimbus_cop_stage_size_u64(const nimbus_ctx* ctx, const nimbus_cop_job_u64* jobs, uint32_t count,
                                        size_t* bytes) {
    if (!ctx || !jobs || !bytes || count == 0) return NIMBUS_EINVAL;
    const std::vector<nimbus_cop_job> v = jobs_of(jobs, count);
    return nimbus_cop_stage_size(ctx, v.data(), count, bytes);
}

nimbus_status nimbus_cop_matmul_streamed_u64(nimbus_ctx* ctx, const nimbus_cop_job_u64* jobs, uint32_t count,
                                             void* d_ws, size_t ws_bytes, void* d_stage, size_t stage_bytes,
                                             void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 8);
    if (st != NIMBUS_OK) return st;
    if (!jobs || count == 0) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    const std::vector<nimbus_cop_job> v = jobs_of(jobs, count);
    return cop_matmul_streamed(ctx, v.data(), count, d_ws, ws_bytes, d_stage, stage_bytes, stream);
}

nimbus_status nimbus_profile_enable(nimbus_ctx* ctx, int on) {
    if (!ctx) return NIMBUS_EINVAL;
    ctx->profile = on != 0;
    return NIMBUS_OK;
}

nimbus_status nimbus_profile_read(nimbus_ctx* ctx, double* ms, uint64_t* calls, int reset) {
    DevGuard dg_(ctx, __func__);
    if (!ctx) return NIMBUS_EINVAL;
    auto& P = ctx->ev_pending;
    // groups of 5: before slice, after slice, after contraction, before pack, after pack
    for (size_t i = 0; i + 5 <= P.size(); i += 5) {
        CK(cudaEventSynchronize(P[i + 4]), "profile sync");
        CK(cudaEventSynchronize(P[i + 2]), "profile sync");
        float a = 0, b = 0, c = 0;
        cudaEventElapsedTime(&a, P[i], P[i + 1]);
        cudaEventElapsedTime(&b, P[i + 1], P[i + 2]);
        cudaEventElapsedTime(&c, P[i + 3], P[i + 4]);
        ctx->prof_ms[0] += a; ctx->prof_ms[1] += b; ctx->prof_ms[2] += c;
        ctx->prof_calls++;
    }
    for (cudaEvent_t e : P) ctx->ev_pool.push_back(e);
    P.clear();
    if (ms) for (int i = 0; i < 3; i++) ms[i] = ctx->prof_ms[i];
    if (calls) *calls = ctx->prof_calls;
    if (reset) { ctx->prof_ms[0] = ctx->prof_ms[1] = ctx->prof_ms[2] = 0; ctx->prof_calls = 0; }
    return NIMBUS_OK;
}

static nimbus_status cop_matmul_host(nimbus_ctx* ctx, const nimbus_encw* w, const void* h_X, uint32_t kq,
                                     uint32_t nq, uint64_t seed, uint32_t* h_cts, void* h_R, void* d_ws,
                                     size_t ws_bytes, void* stream) {
    nimbus_status st = check_online(ctx, w, kq, nq);
    if (st != NIMBUS_OK) return st;
    if (!h_X || !h_cts || !h_R || !d_ws) return set_err(ctx, NIMBUS_EINVAL, "null buffer");
    const uint32_t k = kq * nq;
    const size_t es = elem_bytes(ctx->rns.ell);
    const WsLayout L = ws_layout(ctx, w, k);
    if (ws_bytes < L.total) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)d_ws;
    void* dX = ws + L.stage_x;
    uint32_t* dcts = reinterpret_cast<uint32_t*>(ws + L.stage_cts);
    void* dR = ws + L.stage_r;
    const uint32_t nct = cts_per_query(ctx, kq, w->n);
    const size_t cts_bytes = (size_t)nq * nct * 2 * ctx->rns.L_out * ctx->rns.N * 4;
    // R depends only on the mask seed: generate and download it on the side stream while
    // `stream` uploads X and runs the matmul (whose pack then skips R)
    if (!ctx->side) CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "side stream");
    cudaStream_t b = ctx->side;
    while (ctx->sync_ev.size() < 2) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        ctx->sync_ev.push_back(e);
    }
    CK(cudaEventRecord(ctx->sync_ev[0], s), "record");
    CK(cudaStreamWaitEvent(b, ctx->sync_ev[0], 0), "wait");          // after earlier work on `stream`
    CK(launch_mask_R(ctx, kq, nq, w->n, seed, dR, b), "mask R");
    CK(cudaMemcpyAsync(h_R, dR, (size_t)k * w->n * es, cudaMemcpyDeviceToHost, b), "d2h R");
    CK(cudaEventRecord(ctx->sync_ev[1], b), "record");
    CK(cudaMemcpyAsync(dX, h_X, (size_t)k * w->m * es, cudaMemcpyHostToDevice, s), "h2d X");
    st = cop_matmul(ctx, w, dX, kq, nq, seed, dcts, nullptr, d_ws, ws_bytes, stream, true);
    if (st != NIMBUS_OK) return st;
    CK(cudaMemcpyAsync(h_cts, dcts, cts_bytes, cudaMemcpyDeviceToHost, s), "d2h cts");
    CK(cudaStreamWaitEvent(s, ctx->sync_ev[1], 0), "join");
    CK(cudaStreamSynchronize(s), "host matmul sync");
    return NIMBUS_OK;
}

nimbus_status nimbus_cop_matmul_host(nimbus_ctx* ctx, const nimbus_encw* w, const uint32_t* h_X, uint32_t kq,
                                     uint32_t nq, uint64_t seed, uint32_t* h_cts, uint32_t* h_R, void* d_ws,
                                     size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st : cop_matmul_host(ctx, w, h_X, kq, nq, seed, h_cts, h_R, d_ws, ws_bytes, stream);
}

nimbus_status nimbus_cop_matmul_host_u64(nimbus_ctx* ctx, const nimbus_encw* w, const uint64_t* h_X, uint32_t kq,
                                         uint32_t nq, uint64_t seed, uint32_t* h_cts, uint64_t* h_R, void* d_ws,
                                         size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 8);
    return st != NIMBUS_OK ? st : cop_matmul_host(ctx, w, h_X, kq, nq, seed, h_cts, h_R, d_ws, ws_bytes, stream);
}

// ---------------------------------------------------------------- host-buffer job list, pipelined
// Workspace: the matmul workspace of the largest job (nimbus_cop_workspace_size),
// then kHostSlots staging slots (X | cts | R) sized for the largest job.
// staging slots of the host-buffer job list: a unit (one job, or a same-X group of up to 4) and
// the next one are in flight together and must not share a slot, so 8
static constexpr uint32_t kHostSlots = 8;
struct HostBatchLayout {
    size_t mm = 0, slot = 0, x = 0, cts = 0, r = 0, total = 0;   // x / cts / r: offsets inside a slot
};
static HostBatchLayout host_batch_layout(const nimbus_ctx* ctx, const nimbus_cop_host_job* jobs, uint32_t count) {
    auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
    HostBatchLayout H;
    const size_t es = elem_bytes(ctx->rns.ell);
    size_t xb = 0, cb = 0, rb = 0;
    for (uint32_t i = 0; i < count; i++) {
        const nimbus_cop_host_job& J = jobs[i];
        const uint32_t k = J.k_per_query * J.n_queries;
        const WsLayout L = ws_layout(ctx, J.encw, k);
        H.mm = H.mm > L.total ? H.mm : L.total;                     // what nimbus_cop_matmul checks for
        xb = std::max(xb, al((size_t)k * J.encw->m * es));
        cb = std::max(cb, al((size_t)J.n_queries * cts_per_query(ctx, J.k_per_query, J.encw->n) * 2 *
                             ctx->rns.L_out * ctx->rns.N * 4));
        rb = std::max(rb, al((size_t)k * J.encw->n * es));
    }
    // a same-X group runs as one resident-X launch: X planes + one C buffer per job of the group
    for (uint32_t i = 0; i < count;) {
        const uint32_t g = same_hx_group(ctx, jobs, count, i);
        if (g > 1) {
            const nimbus_cop_host_job& J = jobs[i];
            const uint32_t k = J.k_per_query * J.n_queries;
            const WsLayout L = ws_layout(ctx, J.encw, k);
            H.mm = std::max(H.mm, L.c + g * al((size_t)k * ncols(ctx) * 4));
        }
        i += g;
    }
    H.x = 0;
    H.cts = xb;
    H.r = xb + cb;
    H.slot = xb + cb + rb;
    H.total = H.mm + kHostSlots * H.slot;
    return H;
}

nimbus_status nimbus_cop_workspace_size_host_batch(const nimbus_ctx* ctx, const nimbus_cop_host_job* jobs,
                                                   uint32_t count, size_t* bytes) {
    if (!ctx || !jobs || !bytes || count == 0) return NIMBUS_EINVAL;
    for (uint32_t i = 0; i < count; i++)
        if (!jobs[i].encw || jobs[i].encw->ctx != ctx || jobs[i].k_per_query == 0 || jobs[i].n_queries == 0)
            return NIMBUS_EINVAL;
    *bytes = host_batch_layout(ctx, jobs, count).total;
    return NIMBUS_OK;
}

static nimbus_status cop_matmul_host_batch(nimbus_ctx* ctx, const nimbus_cop_host_job* jobs, uint32_t count,
                                           void* d_ws, size_t ws_bytes, void* stream) {
    if (!ctx || !jobs || count == 0 || !d_ws) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    for (uint32_t i = 0; i < count; i++) {
        nimbus_status st = check_online(ctx, jobs[i].encw, jobs[i].k_per_query, jobs[i].n_queries);
        if (st != NIMBUS_OK) return st;
        if (!jobs[i].h_X || !jobs[i].h_cts || !jobs[i].h_R) return set_err(ctx, NIMBUS_EINVAL, "null buffer");
    }
    const HostBatchLayout H = host_batch_layout(ctx, jobs, count);
    if (ws_bytes < H.total) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    const size_t es = elem_bytes(ctx->rns.ell);
    cudaStream_t s = (cudaStream_t)stream;
    if (!ctx->copy) CK(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking), "copy stream");
    if (!ctx->side) CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "side stream");
    cudaStream_t up = ctx->copy, down = ctx->side;
    while (ctx->host_ev.size() < 3 * kHostSlots + 1) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        ctx->host_ev.push_back(e);
    }
    cudaEvent_t* ev_x = ctx->host_ev.data();                    // slot's X uploaded
    cudaEvent_t* ev_c = ev_x + kHostSlots;                      // slot's matmul done
    cudaEvent_t* ev_o = ev_c + kHostSlots;                      // slot's outputs downloaded (slot free)
    cudaEvent_t start = ev_o[kHostSlots];
    // neither copy stream may touch the workspace before earlier work on `stream`
    CK(cudaEventRecord(start, s), "record");
    CK(cudaStreamWaitEvent(up, start, 0), "wait");
    CK(cudaStreamWaitEvent(down, start, 0), "wait");
    uint8_t* ws = (uint8_t*)d_ws;
    auto slot_of = [&](uint32_t i) { return ws + H.mm + (i % kHostSlots) * H.slot; };
    auto cts_bytes = [&](const nimbus_cop_host_job& J) {
        return (size_t)J.n_queries * cts_per_query(ctx, J.k_per_query, J.encw->n) * 2 * ctx->rns.L_out *
               ctx->rns.N * 4;
    };
    // upload job i's X into its slot once the matmul that last used the slot (job i - S) is done
    auto upload = [&](uint32_t i) -> nimbus_status {
        const nimbus_cop_host_job& J = jobs[i];
        if (i >= kHostSlots) CK(cudaStreamWaitEvent(up, ev_c[i % kHostSlots], 0), "wait slot X");
        CK(cudaMemcpyAsync(slot_of(i) + H.x, J.h_X, (size_t)J.k_per_query * J.n_queries * J.encw->m * es,
                           cudaMemcpyHostToDevice, up), "h2d X");
        CK(cudaEventRecord(ev_x[i % kHostSlots], up), "record");
        return NIMBUS_OK;
    };
    // `stream` may start job i once its X is up and its output buffers were read out (job i - S)
    auto admit = [&](uint32_t i) -> nimbus_status {
        CK(cudaStreamWaitEvent(s, ev_x[i % kHostSlots], 0), "wait X");
        if (i >= kHostSlots) CK(cudaStreamWaitEvent(s, ev_o[i % kHostSlots], 0), "wait slot out");
        return NIMBUS_OK;
    };
    // a unit is one job, or a same-X group of g jobs (one X upload into the first job's slot, one
    // resident-X launch; the group's outputs in the slots of its jobs)
    auto prepare = [&](uint32_t i, uint32_t g) -> nimbus_status {
        nimbus_status r = upload(i);
        for (uint32_t q = 1; q < g && r == NIMBUS_OK; q++) {
            // the other jobs' slots hold no X: their "X ready" is the group's
            if (cudaEventRecord(ev_x[(i + q) % kHostSlots], up) != cudaSuccess) r = set_err(ctx, NIMBUS_ECUDA, "record");
        }
        for (uint32_t q = 0; q < g && r == NIMBUS_OK; q++) r = admit(i + q);
        return r;
    };
    uint32_t g = same_hx_group(ctx, jobs, count, 0);
    nimbus_status st = prepare(0, g);
    const nimbus_encw* after = ctx->pf_next;               // the caller's hint: what follows the list
    for (uint32_t i = 0; i < count && st == NIMBUS_OK; i += g) {
        g = same_hx_group(ctx, jobs, count, i);
        const nimbus_cop_host_job& J = jobs[i];
        const uint32_t k = J.k_per_query * J.n_queries;
        uint8_t* slot = slot_of(i);
        ctx->pf_next = i + g < count ? jobs[i + g].encw : after;   // the list names each unit's successor
        // the next unit's prerequisites go into `stream` BEFORE this unit's kernels, so that its
        // pack and the next unit's slice stay adjacent (programmatic dependent launch across jobs)
        if (i + g < count) {
            st = prepare(i + g, same_hx_group(ctx, jobs, count, i + g));
            if (st != NIMBUS_OK) break;
        }
        if (g > 1) {
            nimbus_cop_job dj[4];
            for (uint32_t q = 0; q < g; q++) {
                const nimbus_cop_host_job& Jq = jobs[i + q];
                dj[q] = {Jq.encw, reinterpret_cast<const uint32_t*>(slot + H.x), Jq.k_per_query, Jq.n_queries,
                         Jq.mask_seed, reinterpret_cast<uint32_t*>(slot_of(i + q) + H.cts),
                         reinterpret_cast<uint32_t*>(slot_of(i + q) + H.r)};
            }
            const WsLayout L = ws_layout(ctx, J.encw, k);
            const cudaError_t e = run_x_group(ctx, dj, g, ws, L.c, al1k((size_t)k * ncols(ctx) * 4), s);
            if (e != cudaSuccess) { st = cuda_err(ctx, e, "host batch group"); break; }
        } else {
            st = cop_matmul(ctx, J.encw, slot + H.x, J.k_per_query, J.n_queries, J.mask_seed,
                            reinterpret_cast<uint32_t*>(slot + H.cts), slot + H.r, ws, H.mm, stream);
            if (st != NIMBUS_OK) break;
        }
        for (uint32_t q = 0; q < g; q++) {
            const nimbus_cop_host_job& Jq = jobs[i + q];
            uint8_t* sq = slot_of(i + q);
            CK(cudaEventRecord(ev_c[(i + q) % kHostSlots], s), "record");
            // download the job's outputs while the next jobs compute
            CK(cudaStreamWaitEvent(down, ev_c[(i + q) % kHostSlots], 0), "wait matmul");
            CK(cudaMemcpyAsync(Jq.h_cts, sq + H.cts, cts_bytes(Jq), cudaMemcpyDeviceToHost, down), "d2h cts");
            CK(cudaMemcpyAsync(Jq.h_R, sq + H.r, (size_t)k * Jq.encw->n * es, cudaMemcpyDeviceToHost, down), "d2h R");
            CK(cudaEventRecord(ev_o[(i + q) % kHostSlots], down), "record");
        }
    }
    if (st != NIMBUS_OK) {
        cudaStreamSynchronize(up);          // no copy may outlive the call into a buffer the caller frees
        cudaStreamSynchronize(down);
        return st;
    }
    CK(cudaStreamWaitEvent(s, ev_o[(count - 1) % kHostSlots], 0), "join");
    CK(cudaStreamSynchronize(s), "host batch sync");
    return NIMBUS_OK;
}

nimbus_status nimbus_cop_matmul_host_batch(nimbus_ctx* ctx, const nimbus_cop_host_job* jobs, uint32_t count,
                                           void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st : cop_matmul_host_batch(ctx, jobs, count, d_ws, ws_bytes, stream);
}

nimbus_status nimbus_cop_workspace_size_host_batch_u64(const nimbus_ctx* ctx, const nimbus_cop_host_job_u64* jobs,
                                                       uint32_t count, size_t* bytes) {
    return nimbus_cop_workspace_size_host_batch(ctx, reinterpret_cast<const nimbus_cop_host_job*>(jobs), count,
                                                bytes);
}

nimbus_status nimbus_cop_matmul_host_batch_u64(nimbus_ctx* ctx, const nimbus_cop_host_job_u64* jobs, uint32_t count,
                                               void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 8);
    return st != NIMBUS_OK ? st
                           : cop_matmul_host_batch(ctx, reinterpret_cast<const nimbus_cop_host_job*>(jobs), count,
                                                   d_ws, ws_bytes, stream);
}

static nimbus_status decrypt(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_cts, uint32_t kq, uint32_t n,
                             uint32_t nq, void* d_Z, void* d_M, void* stream) {
    if (!ctx || !sk || !d_cts || !d_Z || kq == 0 || nq == 0 || n == 0) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    if (n > ctx->rns.N) return set_err(ctx, NIMBUS_ESHAPE, "n > N");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t nct = cts_per_query(ctx, kq, n);
    uint32_t* U = nullptr;
    CK(cudaMallocAsync(&U, (size_t)nq * nct * ctx->rns.L_out * ctx->rns.N * 4, s), "decrypt alloc");
    cudaError_t e = launch_decrypt(ctx, sk->d_s_ntt, d_cts, nq * nct, nct, kq, n, U, d_Z, d_M, s);
    cudaFreeAsync(U, s);
    CK(e, "decrypt");
    return NIMBUS_OK;
}

nimbus_status nimbus_decrypt(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_cts, uint32_t kq, uint32_t n,
                             uint32_t nq, uint32_t* d_Z, uint32_t* d_M, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 4);
    return st != NIMBUS_OK ? st : decrypt(ctx, sk, d_cts, kq, n, nq, d_Z, d_M, stream);
}

nimbus_status nimbus_decrypt_u64(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_cts, uint32_t kq,
                                 uint32_t n, uint32_t nq, uint64_t* d_Z, uint64_t* d_M, void* stream) {
    DevGuard dg_(ctx, __func__);
    nimbus_status st = want_width(ctx, 8);
    return st != NIMBUS_OK ? st : decrypt(ctx, sk, d_cts, kq, n, nq, d_Z, d_M, stream);
}

// ---------------------------------------------------------------- server, step 5
nimbus_status nimbus_plain_weights_u64(nimbus_ctx* ctx, const uint64_t* d_W, uint32_t m, uint32_t n, void* stream,
                                       nimbus_plainw** out) {
    DevGuard dg_(ctx, __func__);
    if (want_width(ctx, 8) != NIMBUS_OK) return NIMBUS_EINVAL;          // ell > 32: t = 2^64 products
    if (!ctx || !d_W || !out || m == 0 || n == 0) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    if (m > 4096) return set_err(ctx, NIMBUS_ESHAPE, "m > 4096 at ell = 64 (int32 slice accumulators)");
    nimbus_plainw* w = new (std::nothrow) nimbus_plainw();
    if (!w) return set_err(ctx, NIMBUS_ENOMEM, "host alloc");
    w->ctx = ctx;
    w->m = m;
    w->n = n;
    w->KB = (m + kBK - 1) / kBK;
    w->bytes = (size_t)plain_col_tiles64(n) * w->KB * 8 * 128 * kBK;
    cudaError_t e = cudaMalloc(&w->d_Wt, w->bytes);
    if (e != cudaSuccess) { delete w; return cuda_err(ctx, e, "plain weights alloc"); }
    e = launch_tile_plainw64(ctx, d_W, m, n, w->KB, w->d_Wt, (cudaStream_t)stream);
    if (e != cudaSuccess) { cudaFree(w->d_Wt); delete w; return cuda_err(ctx, e, "tile plain weights"); }
    ctx_retain(ctx);
    *out = w;
    return NIMBUS_OK;
}

nimbus_status nimbus_plain_weights(nimbus_ctx* ctx, const uint32_t* d_W, uint32_t m, uint32_t n, void* stream,
                                   nimbus_plainw** out) {
    DevGuard dg_(ctx, __func__);
    if (want_width(ctx, 4) != NIMBUS_OK) return NIMBUS_EINVAL;          // ell <= 32 (ell = 64: _u64)
    if (!ctx || !d_W || !out || m == 0 || n == 0) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    nimbus_plainw* w = new (std::nothrow) nimbus_plainw();
    if (!w) return set_err(ctx, NIMBUS_ENOMEM, "host alloc");
    w->ctx = ctx;
    w->m = m;
    w->n = n;
    w->KB = (m + kBK - 1) / kBK;
    w->bytes = (size_t)plain_col_tiles(n) * w->KB * sx_of(ctx->rns.ell) * 64 * kBK;
    cudaError_t e = cudaMalloc(&w->d_Wt, w->bytes);
    if (e != cudaSuccess) { delete w; return cuda_err(ctx, e, "plain weights alloc"); }
    e = launch_tile_plainw(ctx, d_W, m, n, w->KB, w->d_Wt, (cudaStream_t)stream);
    if (e != cudaSuccess) { cudaFree(w->d_Wt); delete w; return cuda_err(ctx, e, "tile plain weights"); }
    ctx_retain(ctx);
    *out = w;
    return NIMBUS_OK;
}

void nimbus_plainw_destroy(nimbus_plainw* w) {
    DevGuard dg_(w ? w->ctx : nullptr, __func__);
    if (!w) return;
    if (w->d_Wt) cudaFree(w->d_Wt);
    nimbus_ctx* ctx = w->ctx;
    delete w;
    ctx_release(ctx);
}

struct ServerWs {
    size_t xt = 0, z = 0, u = 0, total = 0;
};
static ServerWs server_ws(const nimbus_ctx* ctx, const nimbus_plainw* w, uint32_t kq, uint32_t nq) {
    auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
    ServerWs L;
    const size_t k = (size_t)kq * (nq ? nq : 1);
    const size_t Mt = (k + kBM - 1) / kBM;
    const size_t es = elem_bytes(ctx->rns.ell);
    L.xt = 0;
    // X slices: 128-row tiles, or 32-row tiles for the ell = 64 kernel (k_plain_t64)
    const size_t xrows = es == 8 ? ((k + 31) / 32) * 32 : Mt * kBM;
    L.z = al(sx_of(ctx->rns.ell) * xrows * (size_t)w->KB * kBK);
    L.u = L.z + (nq ? al(k * w->n * es) : 0);
    size_t ubytes = 0;
    if (nq) {
        const uint32_t R = ctx->rns.N / w->n, nct = (kq + R - 1) / R;
        ubytes = al((size_t)nq * nct * ctx->rns.L_out * ctx->rns.N * 4);
    }
    L.total = L.u + ubytes;
    return L;
}

nimbus_status nimbus_server_workspace_size(const nimbus_ctx* ctx, const nimbus_plainw* w, uint32_t kq, uint32_t nq,
                                           size_t* bytes) {
    if (!ctx || !w || !bytes || kq == 0) return NIMBUS_EINVAL;
    if (nq && w->n > ctx->rns.N) return NIMBUS_ESHAPE;
    *bytes = server_ws(ctx, w, kq, nq).total;
    return NIMBUS_OK;
}

nimbus_status nimbus_plain_matmul(nimbus_ctx* ctx, const nimbus_plainw* w, const uint32_t* d_X, uint32_t k,
                                  const uint32_t* d_add, uint32_t* d_Y, void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !w || w->ctx != ctx || !d_X || !d_Y || !d_ws || k == 0) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    if (k > (1u << 24)) return set_err(ctx, NIMBUS_ESHAPE, "k too large");
    const ServerWs L = server_ws(ctx, w, k, 0);
    if (ws_bytes < L.total) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* xt = (uint8_t*)d_ws + L.xt;
    CK(launch_slice_x(ctx, d_X, k, w->m, w->KB, kBM, xt, s), "slice X");
    CK(launch_plain_matmul(ctx, xt, w->d_Wt, k, w->n, w->KB, d_add, d_Y, s), "plain matmul");
    return NIMBUS_OK;
}

nimbus_status nimbus_server_output(nimbus_ctx* ctx, const nimbus_sk* sk, const nimbus_plainw* w,
                                   const uint32_t* d_Xs, const uint32_t* d_cts, uint32_t kq, uint32_t nq,
                                   uint32_t* d_Ys, void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !sk || !w || w->ctx != ctx || !d_Xs || !d_cts || !d_Ys || !d_ws || kq == 0 || nq == 0)
        return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    if (w->n > ctx->rns.N) return set_err(ctx, NIMBUS_ESHAPE, "n > N");
    if ((uint64_t)kq * nq > (1u << 24)) return set_err(ctx, NIMBUS_ESHAPE, "k too large");
    const ServerWs L = server_ws(ctx, w, kq, nq);
    if (ws_bytes < L.total) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t k = kq * nq, R = ctx->rns.N / w->n, nct = (kq + R - 1) / R;
    uint8_t* ws = (uint8_t*)d_ws;
    uint32_t* Z = reinterpret_cast<uint32_t*>(ws + L.z);
    uint32_t* U = reinterpret_cast<uint32_t*>(ws + L.u);
    CK(launch_decrypt(ctx, sk->d_s_ntt, d_cts, nq * nct, nct, kq, w->n, U, Z, nullptr, s), "decrypt");
    CK(launch_slice_x(ctx, d_Xs, k, w->m, w->KB, kBM, ws + L.xt, s), "slice X_s");
    CK(launch_plain_matmul(ctx, ws + L.xt, w->d_Wt, k, w->n, w->KB, Z, d_Ys, s), "plain matmul");
    return NIMBUS_OK;
}

nimbus_status nimbus_plain_matmul_u64(nimbus_ctx* ctx, const nimbus_plainw* w, const uint64_t* d_X, uint32_t k,
                                      const uint64_t* d_add, uint64_t* d_Y, void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (want_width(ctx, 8) != NIMBUS_OK) return NIMBUS_EINVAL;
    if (!ctx || !w || w->ctx != ctx || !d_X || !d_Y || !d_ws || k == 0) return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    if (k > (1u << 24)) return set_err(ctx, NIMBUS_ESHAPE, "k too large");
    const ServerWs L = server_ws(ctx, w, k, 0);
    if (ws_bytes < L.total) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* xt = (uint8_t*)d_ws + L.xt;
    CK(launch_slice_x(ctx, d_X, k, w->m, w->KB, 32, xt, s), "slice X");
    CK(launch_plain_matmul64(ctx, xt, w->d_Wt, k, w->n, w->KB, d_add, d_Y, s), "plain matmul 64");
    return NIMBUS_OK;
}

nimbus_status nimbus_server_output_u64(nimbus_ctx* ctx, const nimbus_sk* sk, const nimbus_plainw* w,
                                       const uint64_t* d_Xs, const uint32_t* d_cts, uint32_t kq, uint32_t nq,
                                       uint64_t* d_Ys, void* d_ws, size_t ws_bytes, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (want_width(ctx, 8) != NIMBUS_OK) return NIMBUS_EINVAL;
    if (!ctx || !sk || !w || w->ctx != ctx || !d_Xs || !d_cts || !d_Ys || !d_ws || kq == 0 || nq == 0)
        return set_err(ctx, NIMBUS_EINVAL, "bad argument");
    if (w->n > ctx->rns.N) return set_err(ctx, NIMBUS_ESHAPE, "n > N");
    if ((uint64_t)kq * nq > (1u << 24)) return set_err(ctx, NIMBUS_ESHAPE, "k too large");
    const ServerWs L = server_ws(ctx, w, kq, nq);
    if (ws_bytes < L.total) return set_err(ctx, NIMBUS_ESHAPE, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t k = kq * nq, R = ctx->rns.N / w->n, nct = (kq + R - 1) / R;
    uint8_t* ws = (uint8_t*)d_ws;
    uint64_t* Z = reinterpret_cast<uint64_t*>(ws + L.z);
    uint32_t* U = reinterpret_cast<uint32_t*>(ws + L.u);
    CK(launch_decrypt(ctx, sk->d_s_ntt, d_cts, nq * nct, nct, kq, w->n, U, Z, nullptr, s), "decrypt");
    CK(launch_slice_x(ctx, d_Xs, k, w->m, w->KB, 32, ws + L.xt, s), "slice X_s");
    CK(launch_plain_matmul64(ctx, ws + L.xt, w->d_Wt, k, w->n, w->KB, Z, d_Ys, s), "plain matmul 64");
    return NIMBUS_OK;
}

nimbus_status nimbus_prg_words(uint64_t seed, uint32_t dom, uint64_t start, uint64_t count, uint64_t* d_out,
                               void* stream) {
    if (!d_out) return NIMBUS_EINVAL;
    return launch_prg_words(seed, dom, start, count, d_out, (cudaStream_t)stream) == cudaSuccess ? NIMBUS_OK
                                                                                                : NIMBUS_ECUDA;
}

nimbus_status nimbus_negacyclic_mul(nimbus_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t count,
                                    uint32_t* c, void* stream) {
    DevGuard dg_(ctx, __func__);
    if (!ctx || !a || !b || !c || count == 0) return NIMBUS_EINVAL;
    CK(launch_negacyclic_mul(ctx, a, b, count, c, (cudaStream_t)stream), "negacyclic_mul");
    return NIMBUS_OK;
}

}  // extern "C"
