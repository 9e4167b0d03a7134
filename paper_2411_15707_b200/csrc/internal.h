// internal.h -- host-side structures shared by the translation units of
// libnimbus_cop.so.  Not part of the public ABI (see include/nimbus_cop.h).
#pragma once
#include <cstdint>
#include <atomic>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/nimbus_cop.h"
#include "common.cuh"

typedef unsigned __int128 u128;

// Kernel-layout geometry of Enc(W) and of the sliced X.
constexpr uint32_t kBK = 128;      // beta (contraction) bytes per k-block = one 128-B swizzle row
constexpr uint32_t kBNT = 48;      // coefficient columns per Enc(W) tile, streaming kernel (4 planes -> MMA N = 192)
constexpr uint32_t kBNR = 32;      // tile width of the resident-X kernel (ell <= 16, m <= 768; MMA N = 128)
constexpr uint32_t kBNW = 128;     // tile width of the transposed ell = 32 kernel (E planes are the MMA A operand)
constexpr uint32_t kResMaxKB = 6;  // resident-X kernel: at most 6 k-blocks (m <= 768) of X in TMEM + smem
constexpr uint32_t kBM = 128;      // rows (alpha) per X tile = tcgen05 M
constexpr uint32_t kSW = 4;        // 8-bit slices of a 31-bit residue (S_w)

// unsigned big integer (6 x 64 bits, little-endian): q beyond 128 bits for ell = 64
struct Big {
    uint64_t w[6] = {0, 0, 0, 0, 0, 0};
};

struct nimbus_ctx {
    nimbus_params prm{};
    int device = 0;
    // the caller's reference + one per live handle (sk, pk, encw, plainw): the context is freed
    // when the last of them goes, so handles may be destroyed after it in any order
    std::atomic<int> refs{1};
    nimbus::Rns rns{};
    Big q;                         // q = prod of all L primes (up to 6 x 31 bits)
    u128 qout = 0;                 // q' = prod of the first L_out primes (< 2^95)
    uint32_t* d_tw = nullptr;      // per limb 4 x N: psi_rev, psi_rev_shoup, ipsi_rev, ipsi_rev_shoup
    uint32_t* d_flag = nullptr;    // device error flags (bit 0: input >= t)
    std::string err;
    uint64_t launches = 0;
    char last_contraction[48] = "";  // name of the last contraction kernel launched (nimbus_last_contraction)
    int num_sms = 148;
    int res_ring = 1;              // resident-X contraction: 1 = 3-slot ring + slice 1 in smem, 2 = deep ring (k_cop_tc_res2); env NIMBUS_RES
    int cluster = 1;               // CTAs per cluster of the streaming contraction (2 = X multicast); env NIMBUS_CLUSTER
    bool fuse_r1 = true;           // R = 1 layers: mod-switch + mask in the resident kernel's epilogue; env NIMBUS_NO_FUSE=1 off
    const nimbus_encw* pf_next = nullptr;   // nimbus_cop_prefetch_next: the Enc(W) of the call after the next one (one-shot hint)
    // stage profiling (nimbus_profile_*): pending event quadruples, accumulated ms
    bool profile = false;
    std::vector<cudaEvent_t> ev_pool, ev_pending;
    double prof_ms[3] = {0, 0, 0};
    uint64_t prof_calls = 0;
    // batched path (nimbus_cop_matmul_batch): side stream for the pack kernels + sync events
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> sync_ev;
    // streamed path (nimbus_cop_matmul_streamed): host -> device copy stream + events
    cudaStream_t copy = nullptr;
    std::vector<cudaEvent_t> stream_ev;
    // host-buffer job list (nimbus_cop_matmul_host_batch): per staging slot X-up / matmul / outputs-down events
    std::vector<cudaEvent_t> host_ev;
    // file-backed Enc(W) streaming: two pinned read buffers (grow-only) and the first read error of a
    // stream-ordered host callback (reported by nimbus_sync / the next streamed call)
    uint8_t* h_read[2] = {nullptr, nullptr};
    size_t h_read_bytes = 0;
    std::atomic<int> io_error{0};
    // grow-only device scratch for the canonical rows of Enc(W) during (re-)encryption
    void* d_scratch = nullptr;
    size_t scratch_bytes = 0;
    // kernels already opted into their dynamic shared memory on this context's device
    std::vector<const void*> smem_ok;
};

struct nimbus_sk {
    nimbus_ctx* ctx = nullptr;
    int8_t* d_s = nullptr;         // N ternary coefficients
    uint32_t* d_s_ntt = nullptr;   // L x N, NTT domain (bit-reversed order)
    uint32_t* d_s_enc = nullptr;   // 2 x L x N: s_hat in the fused encrypt's thread order + Shoup (N = 4096 / 8192)
};

// public key pk = (b, a) (reading 25)
struct nimbus_pk {
    nimbus_ctx* ctx = nullptr;
    uint32_t* d_pk = nullptr;      // [comp b=0, a=1][limb][N] coefficients (the exported form)
    uint32_t* d_pk_ntt = nullptr;  // same, NTT domain (bit-reversed), for the zero encryptions
};

struct nimbus_encw {
    nimbus_ctx* ctx = nullptr;
    uint32_t m = 0, n = 0, KB = 0; // KB = ceil(m / 128) k-blocks
    uint32_t bn = kBNT;            // tile width (columns) of the resident layout
    uint8_t* d_Et = nullptr;       // tiled byte planes [ct][kb][s][bn][128 swizzled]; null when offloaded
    uint32_t* d_corr = nullptr;    // packed contraction (cop_pk.cu): corr [2LN] then ColSum [2LN]; stays resident
    uint8_t* h_Et = nullptr;       // pinned host copy of the same bytes (nimbus_encw_offload)
    size_t bytes = 0;
    // file-backed (nimbus_encw_open): canonical payload of a store file, read per streamed matmul
    std::string file;
    uint64_t file_off = 0, canon_bytes = 0;
};

struct nimbus_plainw {
    nimbus_ctx* ctx = nullptr;
    uint32_t m = 0, n = 0, KB = 0;
    uint8_t* d_Wt = nullptr;       // S_x byte planes [ct][kb][j][64][128 swizzled] (plain.cu)
    size_t bytes = 0;
};

// number of 8-bit slices of an ell-bit X entry (S_x)
inline uint32_t sx_of(uint32_t ell) { return ell <= 8 ? 1 : ell <= 16 ? 2 : ell <= 32 ? 4 : 8; }
// bytes of one X / W / R / Z element at the boundary: uint32 up to ell = 32, uint64 beyond
inline uint32_t elem_bytes(uint32_t ell) { return ell <= 32 ? 4u : 8u; }
// number of 48-column Enc(W) tiles covering the 2 L N coefficient columns (last one zero padded)
// (rounded up to an even count so column tiles pair up in 2-CTA clusters)
inline uint32_t col_tiles(const nimbus_ctx* c, uint32_t bn) { return (((2 * c->rns.L * c->rns.N + bn - 1) / bn) + 1) & ~1u; }

// one matmul of the packed contraction (cop_pk.cu); d_Xp: its packed X slices in the workspace
struct PkHostJob {
    const nimbus_encw* w = nullptr;
    const uint32_t* d_X = nullptr;
    uint32_t kq = 0, nq = 0;
    uint64_t seed = 0;
    uint32_t* d_cts = nullptr;
    uint32_t* d_R = nullptr;       // null: R not written (the host-buffer call makes it separately)
    const uint8_t* d_Xp = nullptr;
};

// the matmuls of one pack launch (same shape; blockIdx.z = comp + 2 job)
struct PackJobs {
    const uint32_t* C[4] = {nullptr, nullptr, nullptr, nullptr};
    uint32_t* cts[4] = {nullptr, nullptr, nullptr, nullptr};
    void* R[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t key[4] = {0, 0, 0, 0};      // prg_key(mask_seed, 6)
    uint32_t nj = 0;
};
// the matmuls of one resident-X contraction launch (same X, same m: Q / K / V of a layer)
struct ResJobs {
    const uint8_t* Et[4] = {nullptr, nullptr, nullptr, nullptr};
    uint32_t* C[4] = {nullptr, nullptr, nullptr, nullptr};
    uint32_t nj = 0;
};

// First tiles of the NEXT resident-X contraction (nimbus_cop_prefetch_next): CTA b of this launch
// prefetches into L2 the Enc(W) tile CTA b of that launch starts with, once its own last copies are issued.
struct ResPf {
    const uint8_t* base = nullptr;
    uint32_t tile_bytes = 0, ntiles = 0, NT = 0, fuse = 0, grid = 0, count = 1;
    uint32_t self = 0, from = 2;     // own tiles [from, from + self) prefetched before the PDL wait
    uint32_t pol = 0;                // L2 policy of the prefetch (measurement switch)
};

// ---------------------------------------------------------------- launchers
namespace nimbus {
// ntt.cu
cudaError_t launch_keygen(nimbus_ctx* c, uint64_t seed, int8_t* d_s, uint32_t* d_s_ntt, cudaStream_t st);
cudaError_t launch_encrypt(nimbus_ctx* c, const uint32_t* d_s_ntt, const void* d_W, uint32_t m,
                           uint32_t n, uint64_t seed, uint32_t* d_encW, cudaStream_t st);
cudaError_t launch_negacyclic_mul(nimbus_ctx* c, const uint32_t* a, const uint32_t* b, uint32_t count,
                                  uint32_t* out, cudaStream_t st);
cudaError_t launch_decrypt(nimbus_ctx* c, const uint32_t* d_s_ntt, const uint32_t* cts, uint32_t nct_total,
                           uint32_t nct, uint32_t kq, uint32_t n, uint32_t* d_u_tmp, void* d_Z,
                           void* d_M, cudaStream_t st);
// public key (coefficients, [comp][limb][N]) from sk; then launch_ntt_rows for its NTT form
cudaError_t launch_keygen_pk(nimbus_ctx* c, const uint32_t* d_s_ntt, uint64_t seed, uint32_t* d_pk, cudaStream_t st);
// forward NTT of `count` x L polynomials [count][L][N] (limb i mod p_i)
cudaError_t launch_ntt_rows(nimbus_ctx* c, const uint32_t* in, uint32_t count, uint32_t* out, cudaStream_t st);
// n_cts public-key encryptions of zero [g][comp][limb][N] with F flooding bits (reading 26)
cudaError_t launch_rerand(nimbus_ctx* c, const uint32_t* d_pk_ntt, uint64_t seed, uint32_t n_cts, uint32_t F,
                          uint32_t* d_zero, cudaStream_t st);
cudaError_t launch_prg_words(uint64_t seed, uint32_t dom, uint64_t start, uint64_t count, uint64_t* out,
                             cudaStream_t st);
// layout.cu
// fused Encrypt rows -> resident planes (encrypt.cu; N = 4096 / 8192)
bool encrypt_planes_ok(const nimbus_ctx* c);
cudaError_t launch_perm_s(nimbus_ctx* c, const uint32_t* d_s_ntt, uint32_t* d_s_enc, cudaStream_t st);
cudaError_t launch_encrypt_planes(nimbus_ctx* c, const uint32_t* d_s_enc, const void* d_W, uint32_t m, uint32_t n,
                                  uint64_t seed, uint32_t KB, uint32_t bn, uint8_t* d_Et, cudaStream_t st);
cudaError_t launch_tile_encw(nimbus_ctx* c, const uint32_t* d_canon, uint32_t m, uint32_t KB, uint32_t bn,
                             uint8_t* d_Et, cudaStream_t st);
cudaError_t launch_untile_encw(nimbus_ctx* c, const uint8_t* d_Et, uint32_t m, uint32_t KB, uint32_t bn,
                               uint32_t* d_canon, cudaStream_t st);
// Outputs of the last kernel we launched on a stream that triggers its dependents early
// (griddepcontrol.launch_dependents at its start: k_pack, the fused R = 1 contraction,
// k_cop_pk, the server GEMMs).  The next kernel on that stream may start before it is done;
// the slice kernels read X before their PDL wait, which is only safe when X is not one of
// these outputs -- otherwise they load X after the wait (pdl_outputs_overlap).
void pdl_outputs_set(cudaStream_t st, const void* const* ptrs, const size_t* bytes, uint32_t n);
bool pdl_outputs_overlap(cudaStream_t st, const void* p, size_t bytes);
cudaError_t launch_slice_x(nimbus_ctx* c, const void* d_X, uint32_t k, uint32_t m, uint32_t KB, uint32_t rt,
                           uint8_t* d_Xt, cudaStream_t st);
// d_R may be null: then the pack writes only the ciphertexts (R comes from launch_mask_R).
// d_zero (nullable): public-key encryptions of zero [tg][comp][L][N] added before ModDown.
cudaError_t launch_pack(nimbus_ctx* c, const uint32_t* d_C, uint32_t kq, uint32_t nq, uint32_t n,
                        uint64_t seed, uint32_t* d_cts, void* d_R, cudaStream_t st, bool pdl,
                        const uint32_t* d_zero = nullptr);
cudaError_t launch_pack_jobs(nimbus_ctx* c, const PackJobs& P, uint32_t kq, uint32_t nq, uint32_t n, cudaStream_t st,
                             bool pdl, const uint32_t* Z0 = nullptr);
cudaError_t launch_mask_R(nimbus_ctx* c, uint32_t kq, uint32_t nq, uint32_t n, uint64_t seed, void* d_R,
                          cudaStream_t st);
// cop_cc.cu
cudaError_t launch_cop_cudacore(nimbus_ctx* c, const nimbus_encw* w, const uint32_t* d_X, uint32_t k,
                                uint32_t* d_C, cudaStream_t st);
// plain.cu (server step 5)
uint32_t plain_col_tiles(uint32_t n);
cudaError_t launch_tile_plainw(nimbus_ctx* c, const uint32_t* d_W, uint32_t m, uint32_t n, uint32_t KB,
                               uint8_t* d_Wt, cudaStream_t st);
cudaError_t launch_plain_matmul(nimbus_ctx* c, const uint8_t* d_Xt, const uint8_t* d_Wt, uint32_t k, uint32_t n,
                                uint32_t KB, const uint32_t* d_add, uint32_t* d_Y, cudaStream_t st);
// ell = 64: 8-plane W tiles of 128 columns, X slices of 32-row tiles (k_slice_x<8, 32>), uint64 Y / add
uint32_t plain_col_tiles64(uint32_t n);
cudaError_t launch_tile_plainw64(nimbus_ctx* c, const uint64_t* d_W, uint32_t m, uint32_t n, uint32_t KB,
                                 uint8_t* d_Wt, cudaStream_t st);
cudaError_t launch_plain_matmul64(nimbus_ctx* c, const uint8_t* d_Xt, const uint8_t* d_Wt, uint32_t k, uint32_t n,
                                  uint32_t KB, const uint64_t* d_add, uint64_t* d_Y, cudaStream_t st);
// cop_tc.cu
uint32_t transposed_rows(const nimbus_ctx* c);
cudaError_t launch_cop_tcgen05(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k,
                               uint32_t* d_C, cudaStream_t st);
// R = 1 fast path of cop_matmul: the resident-X contraction writes the output ciphertexts
// and R itself (mod-switch + mask fused in its epilogue); fused_r1_ok says when it applies
bool fused_r1_ok(const nimbus_ctx* c, const nimbus_encw* w, uint32_t k);
// the resident-X contraction (ell <= 16, k <= 128, m <= 768) applies to w: resident_ok; several
// such matmuls sharing X run as one launch (launch_res_jobs)
bool resident_ok(const nimbus_ctx* c, const nimbus_encw* w, uint32_t k);
cudaError_t launch_res_jobs(nimbus_ctx* c, const ResJobs& J, uint32_t KB, const uint8_t* d_Xt, uint32_t k,
                            cudaStream_t st);
cudaError_t launch_cop_fused_r1(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k, uint64_t seed,
                                uint32_t* d_cts, uint32_t* d_R, cudaStream_t st);
// cop_pk.cu: the contraction in the packed output layout with ModDown + mask in its epilogue
bool packed_layout_ok(const nimbus_ctx* c, const nimbus_encw* w);
bool packed_ok(const nimbus_ctx* c, const nimbus_encw* w, uint32_t kq, uint32_t nq);
uint32_t packed_rt(const nimbus_ctx* c, const PkHostJob* jobs, uint32_t count);
// the theta-tile heights the packed contraction is instantiated for at this context's S_x
void packed_rt_candidates(const nimbus_ctx* c, const uint32_t** rts, uint32_t* n);
// workspace bytes of one packed job (packed X slices, dropped-limb residues, flags)
size_t packed_xp_bytes(const nimbus_ctx* c, const nimbus_encw* w, uint64_t ntheta, uint32_t rt);
size_t packed_job_bytes(const nimbus_ctx* c, const PkHostJob& j, uint32_t rt);
// d_ctr: a 4-byte device word for the unit dispatch counter (zeroed by the launch itself)
cudaError_t launch_cop_packed(nimbus_ctx* c, const PkHostJob* jobs, uint32_t count, uint32_t rt, uint32_t* d_ctr,
                              cudaStream_t st, void (*mark)(nimbus_ctx*, cudaStream_t));
cudaError_t launch_pk_corr(nimbus_ctx* c, nimbus_encw* w, cudaStream_t st);
}  // namespace nimbus

// Opt `kernel` into `bytes` of dynamic shared memory on the context's device, once
// (the attribute is per device; a process may hold contexts on several devices).
template <typename K>
static inline cudaError_t ensure_smem(nimbus_ctx* c, K kernel, size_t bytes) {
    const void* key = reinterpret_cast<const void*>(kernel);
    for (const void* k : c->smem_ok)
        if (k == key) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) c->smem_ok.push_back(key);
    return e;
}

// Launch with programmatic dependent launch (PDL) allowed: the kernel may be
// scheduled while its stream predecessor is still running; it must call
// nimbus::pdl_wait() before touching data that predecessor produces.
template <typename K, typename... Args>
static inline cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}
