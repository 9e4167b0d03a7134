/*
 * nimbus_cop.h -- C ABI of libnimbus_cop.so, the B200 (sm_100a) hot path of
 * Nimbus' client-side outer-product (COP) homomorphic matmul
 * (arXiv 2411.15707, Alg. 1).
 *
 * Citations: PAPER.md:<line> = /root/reference/PAPER.md (section / algorithm);
 * SURVEY.md §8(c) #<n> = the reading taken where the paper is silent or
 * ambiguous (repeated in DESIGN.md "Readings").
 *
 * Conventions for every entry point
 *  - Return value: nimbus_status, 0 = NIMBUS_OK.  Shape / parameter / noise
 *    budget errors are detected on the host BEFORE any launch, and nothing is
 *    written.  Asynchronous CUDA faults surface as NIMBUS_ECUDA on the next
 *    call that synchronises; nimbus_last_error() has the text.
 *  - d_* pointers are DEVICE pointers owned by the caller (e.g. torch tensor
 *    data_ptr()), contiguous, 16-byte aligned, with the sizes annotated.
 *    h_* pointers are HOST pointers (pinned memory recommended).
 *  - stream is a cudaStream_t (NULL = legacy default stream).  All device work
 *    is enqueued on it; functions return without synchronising unless noted.
 *  - Residues are little-endian uint32 in [0, p_i).  Prime order is
 *    p_0 > p_1 > ....
 *  - Opaque handles are allocated by the library and released by *_destroy.
 *    A context is not thread-safe; distinct contexts are independent.  Every call
 *    runs on its context's device and leaves the caller's current device as it was;
 *    streams passed in must belong to that device.
 */
#ifndef NIMBUS_COP_H
#define NIMBUS_COP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NIMBUS_OK = 0,
    NIMBUS_EINVAL = -1,  /* null pointer, zero dimension, unsupported N/L/ell */
    NIMBUS_ESHAPE = -2,  /* n > N (PAPER.md:232 assumes n < N), dims mismatch, buffer too small */
    NIMBUS_ERANGE = -3,  /* an input entry >= t (only when NIMBUS_FLAG_CHECK_RANGE) */
    NIMBUS_ENOISE = -4,  /* parameters fail the worst-case decryption bound */
    NIMBUS_ECUDA = -5,   /* CUDA runtime error, text in nimbus_last_error */
    NIMBUS_ENOMEM = -6,  /* device allocation failed */
    NIMBUS_EIO = -7,     /* store file unreadable, corrupt, or made for other parameters */
    NIMBUS_EARCH = -8    /* device is not sm_100 (B200) */
} nimbus_status;

enum { NIMBUS_IMPL_TCGEN05 = 0, NIMBUS_IMPL_CUDACORE = 1 };
/* NIMBUS_FLAG_CHECK_RANGE: check X, W < t on the device (reported by nimbus_sync).
 * NIMBUS_FLAG_LARGE_K: 9 <= ell <= 32 only -- lay Enc(W) out for the transposed
 *   contraction (128-column tiles, Enc(W) planes as the MMA A operand), which also feeds
 *   the packed contraction (matmuls with >= 48 packed ciphertexts and n % 128 == 0: the
 *   C5 pass); for matmuls with k >= 512 rows (C5), slower at k = 128 (C4). */
enum { NIMBUS_FLAG_CHECK_RANGE = 1, NIMBUS_FLAG_LARGE_K = 2 };

/* RLWE / workload parameters (App. B.1 {N, q, t}).
 *  N      ring degree, power of two, 64 <= N <= 8192
 *  L      number of 31-bit NTT primes in q (1..6, each with 2^32 mod p < 2^21);
 *         q = p_0 ... p_{L-1}
 *  ell    plaintext bits, t = 2^ell, 1 <= ell <= 64 (> 32: the _u64 entry points)
 *  L_out  limbs kept by the mod-switch of the output (1..min(L, 3))
 *  impl   NIMBUS_IMPL_TCGEN05 (tcgen05 int8 tensor cores) or
 *         NIMBUS_IMPL_CUDACORE (lazy-reduction CUDA-core ablation)
 *  flags  NIMBUS_FLAG_* */
typedef struct {
    uint32_t N, L, ell, L_out, impl, flags;
} nimbus_params;

typedef struct nimbus_ctx nimbus_ctx;
typedef struct nimbus_sk nimbus_sk;
typedef struct nimbus_encw nimbus_encw;
typedef struct nimbus_plainw nimbus_plainw;
typedef struct nimbus_pk nimbus_pk;

/* Context: validates params, derives the primes (the L largest p < 2^31 with
 * p = 1 mod 2N), uploads NTT twiddles and RNS constants to
 * `device`.  Fails with NIMBUS_EARCH off sm_100. */
nimbus_status nimbus_ctx_create(const nimbus_params* params, int device, nimbus_ctx** out);
/* Drops the caller's reference.  Every handle made from the context (sk, pk, encw,
 * plainw) holds one too, so handles may be destroyed before or after the context, in
 * any order; the device memory of the context goes with the last reference. */
void nimbus_ctx_destroy(nimbus_ctx* ctx);
/* Writes the L primes to out_primes[L] (host). */
nimbus_status nimbus_ctx_primes(const nimbus_ctx* ctx, uint32_t* out_primes);
/* Last error text of this context ("" if none).  Valid until the next call. */
const char* nimbus_last_error(const nimbus_ctx* ctx);
/* Blocks until `stream` drains; reports async faults (NIMBUS_ECUDA) and, if
 * range checking is on, NIMBUS_ERANGE for any input seen >= t since the last call. */
nimbus_status nimbus_sync(nimbus_ctx* ctx, void* stream);

/* ---------------------------------------------------------------- setup ---- */
/* KeyGen: ternary secret s in {-1,0,1}^N (SURVEY.md §8(c) #7,
 * symmetric key per #8), drawn from the PRG with domain 1,
 * kept on the device together with its per-limb NTT form. */
nimbus_status nimbus_keygen(nimbus_ctx* ctx, uint64_t seed, void* stream, nimbus_sk** out);
void nimbus_sk_destroy(nimbus_sk* sk);
/* Copies s (N int8 values in {-1,0,1}) to d_s. */
nimbus_status nimbus_sk_export(const nimbus_sk* sk, int8_t* d_s, void* stream);

/* Public key ("KeyGen. Generate the RLWE key pair (sk, pk)";
 * DESIGN.md reading 25), for the client's re-randomisation below:
 *   a_i = uniform mod p_i (PRG domain 7, index i N + j), e = CBD(21) (domain 8, index j),
 *   b_i = a_i s + e mod p_i.
 * The handle owns the key on the device (coefficients and NTT form).
 * export: d_out 2 x L x N uint32 [comp b=0, a=1][limb][j] (what the server sends);
 * import: the same layout, entries must be residues < p_i (not checked). */
nimbus_status nimbus_keygen_pk(nimbus_ctx* ctx, const nimbus_sk* sk, uint64_t seed, void* stream, nimbus_pk** out);
void nimbus_pk_destroy(nimbus_pk* pk);
nimbus_status nimbus_pk_export(const nimbus_pk* pk, uint32_t* d_out, void* stream);
nimbus_status nimbus_pk_import(nimbus_ctx* ctx, const uint32_t* d_in, void* stream, nimbus_pk** out);

/* Alg. 1 step 1, server side: row-wise encode each weight row
 * (Eq. 2: w_hat[j] = W[beta][j] for j < n, 0 beyond) and
 * encrypt it: b = a*s + Emb_q(w_hat) + e mod p_i, a uniform mod p_i (domain 2),
 * e CBD(21) (domain 3), Emb_q(w) = floor((q w + t/2)/t) (SURVEY.md §8(c) #4,#6).
 *  d_W   m x n uint32, row-major, entries < t
 * The handle keeps Enc(W) resident in HBM in the kernel layout (DESIGN.md
 * "Data layout").  Errors: n > N -> ESHAPE; m or n == 0 -> EINVAL;
 * noise bound violated for this (m, n) -> ENOISE. */
nimbus_status nimbus_encrypt_weights(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_W,
                                     uint32_t m, uint32_t n, uint64_t seed, void* stream,
                                     nimbus_encw** out);
/* ell > 32 (up to the paper's ell = 64): X, W, R and Z
 * are uint64 arrays, through the _u64 entry points below; the 32-bit entry
 * points return NIMBUS_EINVAL for such a context and the _u64 ones for ell <= 32.
 * ell > 32 needs L >= 4 limbs for the noise bound (5 at N = 8192), uses S_x = 8
 * X slices (11 shifted accumulators, the transposed kernel) and m <= 4096; the
 * CUDA-core ablation, the server-side calls and nimbus_cop_accumulate /
 * nimbus_cop_pack are 32-bit only. */
nimbus_status nimbus_encrypt_weights_u64(nimbus_ctx* ctx, const nimbus_sk* sk, const uint64_t* d_W,
                                         uint32_t m, uint32_t n, uint64_t seed, void* stream,
                                         nimbus_encw** out);
/* Re-encrypt new weights (same m x n, same layout) into an existing resident handle,
 * e.g. a weight update or a new key: nothing is allocated beyond a stream-ordered
 * temporary for the canonical rows.  Same semantics and PRG indices as
 * nimbus_encrypt_weights with this seed.  NIMBUS_EINVAL for an offloaded handle. */
nimbus_status nimbus_encrypt_weights_into(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_W, uint64_t seed,
                                          void* stream, nimbus_encw* encw);
nimbus_status nimbus_encrypt_weights_into_u64(nimbus_ctx* ctx, const nimbus_sk* sk, const uint64_t* d_W,
                                              uint64_t seed, void* stream, nimbus_encw* encw);
void nimbus_encw_destroy(nimbus_encw* encw);
/* Bytes of device memory held by the handle. */
size_t nimbus_encw_bytes(const nimbus_encw* encw);
/* Canonical layout export / import: d_buf is m x 2 x L x N uint32,
 * [beta][comp b=0,a=1][limb][j] (the store format). */
nimbus_status nimbus_encw_export(const nimbus_encw* encw, uint32_t* d_out, void* stream);
nimbus_status nimbus_encw_import(nimbus_ctx* ctx, const uint32_t* d_in, uint32_t m, uint32_t n,
                                 void* stream, nimbus_encw** out);

/* Store file (the client keeps Enc(W) on disk between sessions, PAPER.md:300;
 * SPEC.md:470).  Little-endian: "NIMBUSEW", u32 version (1), N, L, ell, m, n, the
 * L primes (u32 each), u64 payload bytes, then Enc(W) in the canonical layout of
 * nimbus_encw_export, then a u64 FNV-1a checksum of the payload.  Loading checks
 * every header field against the context and the checksum: NIMBUS_EIO otherwise. */
nimbus_status nimbus_encw_save(const nimbus_encw* encw, const char* path);
nimbus_status nimbus_encw_load(nimbus_ctx* ctx, const char* path, nimbus_encw** out);

/* ---------------------------------------------------------------- online --- */
/* Number of packed output ciphertexts of a call, n_queries * ceil(k_q / floor(N/n))
 * (Table 1, "Pad with zeros"; each query packed apart). */
nimbus_status nimbus_cop_out_count(const nimbus_ctx* ctx, uint32_t k_per_query, uint32_t n,
                                   uint32_t n_queries, uint32_t* n_cts);
/* Device workspace bytes needed by nimbus_cop_matmul / nimbus_cop_accumulate
 * for k = n_queries * k_per_query rows. */
nimbus_status nimbus_cop_workspace_size(const nimbus_ctx* ctx, const nimbus_encw* encw, uint32_t k,
                                        size_t* bytes);

/* Alg. 1 steps 2-4, client side, the timed hot path:
 *   step 2  c[alpha] = sum_beta X[alpha][beta] (x) Enc(W_beta)
 *   step 3  ct~[theta] = sum_r RShift(c[theta R + r], r n), R = floor(N/n)
 *           (stride n per SURVEY.md §8(c) #11)
 *   mod-switch to L_out limbs, iterated round(c/p_last)
 *   step 4  b -= Emb_{q'}(r_theta), r uniform in Z_t for all N slots (domain 6,
 *           index theta_global*N + J)
 *  d_X     k x m uint32 (k = n_queries * k_per_query; query-major), entries < t
 *          (unsigned representative)
 *  d_cts   n_queries x n_cts x 2 x L_out x N uint32  [query][theta][comp][limb][J]
 *  d_R     k x n uint32: the client's output share Y_c = R
 *  d_ws    workspace of at least nimbus_cop_workspace_size bytes (16-byte aligned)
 * No allocation, no host synchronisation: the call (like nimbus_cop_matmul_batch)
 * may be captured into a CUDA graph and replayed; a replay reads the captured
 * buffers as they are at replay time (tests/test_gpu_graph.py).  Do one call
 * per context and kernel variant before capturing (it sets kernel attributes). */
nimbus_status nimbus_cop_matmul(nimbus_ctx* ctx, const nimbus_encw* encw, const uint32_t* d_X,
                                uint32_t k_per_query, uint32_t n_queries, uint64_t mask_seed,
                                uint32_t* d_cts, uint32_t* d_R, void* d_ws, size_t ws_bytes,
                                void* stream);
/* ell > 32: d_X k x m uint64, d_R k x n uint64 (see nimbus_encrypt_weights_u64). */
nimbus_status nimbus_cop_matmul_u64(nimbus_ctx* ctx, const nimbus_encw* encw, const uint64_t* d_X,
                                    uint32_t k_per_query, uint32_t n_queries, uint64_t mask_seed,
                                    uint32_t* d_cts, uint64_t* d_R, void* d_ws, size_t ws_bytes,
                                    void* stream);

/* Circuit privacy of the client's output (the key owner must learn
 * nothing about X_c from the ciphertexts it decrypts; reading 26).
 * Offline, input-independent: nimbus_rerand_prepare writes one public-key
 * encryption of zero per output ciphertext,
 *   z_b = v b_pk + e1 + f,  z_a = v a_pk + e2  (mod each of the L primes),
 *   v ternary (domain 9), e1, e2 CBD(21) (domains 10, 11), f uniform in
 *   [-2^F, 2^F) (F = flood_bits <= 126, 0 = none): the top F + 1 bits of the word
 *   of domain 12 (F <= 62) or of the 128-bit (domain 13 word) 2^64 + (domain 12 word);
 *   PRG index g N + j for output ciphertext g (query-major, as d_cts).
 * Online, nimbus_cop_matmul_rr is nimbus_cop_matmul with z[g] added to packed
 * ciphertext g at the full modulus, before the mod-switch: the output's a
 * component is re-randomised, its noise grows by at most 2 eta N + eta + 2^F
 * before the limb drops, and it decrypts to the same (X.W - R) mod t.
 *  d_zero   n_cts x 2 x L x N uint32 [g][comp][limb][j] (n_cts of nimbus_cop_out_count);
 *           prepare it with the same encw, k_per_query, n_queries, and a fresh seed per call.
 * nimbus_rerand_flood_max: the largest F (<= 126) that keeps decryption exact for
 * this encw and k_per_query (NIMBUS_ENOISE if none); prepare returns NIMBUS_ENOISE
 * for a larger F.  Statistical smudging (F >= 40 bits above the worst-case COP noise
 * R m (t-1)(eta + 1/2)) needs headroom in q: e.g. N = 4096, L = 3, ell = 16, L_out = 1
 * gives F = 73 at the C2 shape (41 bits over 2^32.3); L = 2 allows only F = 44. */
nimbus_status nimbus_rerand_flood_max(const nimbus_ctx* ctx, const nimbus_encw* encw, uint32_t k_per_query,
                                      uint32_t* flood_bits);
nimbus_status nimbus_rerand_prepare(nimbus_ctx* ctx, const nimbus_pk* pk, const nimbus_encw* encw,
                                    uint32_t k_per_query, uint32_t n_queries, uint64_t seed, uint32_t flood_bits,
                                    uint32_t* d_zero, void* stream);
nimbus_status nimbus_cop_matmul_rr(nimbus_ctx* ctx, const nimbus_encw* encw, const uint32_t* d_X,
                                   uint32_t k_per_query, uint32_t n_queries, uint64_t mask_seed,
                                   const uint32_t* d_zero, uint32_t* d_cts, uint32_t* d_R, void* d_ws,
                                   size_t ws_bytes, void* stream);
nimbus_status nimbus_cop_matmul_rr_u64(nimbus_ctx* ctx, const nimbus_encw* encw, const uint64_t* d_X,
                                       uint32_t k_per_query, uint32_t n_queries, uint64_t mask_seed,
                                       const uint32_t* d_zero, uint32_t* d_cts, uint64_t* d_R, void* d_ws,
                                       size_t ws_bytes, void* stream);

/* A sequence of COP matmuls (e.g. all linear layers of a model pass, SURVEY.md
 * config C5): equivalent to nimbus_cop_matmul for jobs[0..count-1] in order,
 * with identical outputs, but the memory-bound pack/mod-switch/mask of job i
 * runs on a library-owned side stream concurrently with the tensor-bound
 * contraction of job i+1 (two C buffers in the workspace, event-ordered).
 * Everything is complete in `stream` order when the call's work on `stream` is.
 * Workspace: nimbus_cop_workspace_size_batch.  Each job's buffers as in
 * nimbus_cop_matmul.  Errors are checked for all jobs before any launch. */
typedef struct {
    const nimbus_encw* encw;
    const uint32_t* d_X;          /* k x m, k = n_queries * k_per_query */
    uint32_t k_per_query, n_queries;
    uint64_t mask_seed;
    uint32_t* d_cts;              /* n_queries x n_cts x 2 x L_out x N */
    uint32_t* d_R;                /* k x n */
} nimbus_cop_job;
nimbus_status nimbus_cop_workspace_size_batch(const nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count,
                                              size_t* bytes);
nimbus_status nimbus_cop_matmul_batch(nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count, void* d_ws,
                                      size_t ws_bytes, void* stream);
/* ell > 32: the same with uint64 X and R. */
typedef struct {
    const nimbus_encw* encw;
    const uint64_t* d_X;          /* k x m uint64 */
    uint32_t k_per_query, n_queries;
    uint64_t mask_seed;
    uint32_t* d_cts;
    uint64_t* d_R;                /* k x n uint64 */
} nimbus_cop_job_u64;
nimbus_status nimbus_cop_workspace_size_batch_u64(const nimbus_ctx* ctx, const nimbus_cop_job_u64* jobs,
                                                  uint32_t count, size_t* bytes);
nimbus_status nimbus_cop_matmul_batch_u64(nimbus_ctx* ctx, const nimbus_cop_job_u64* jobs, uint32_t count,
                                          void* d_ws, size_t ws_bytes, void* stream);

/* Asynchronous weight loading: keep
 * Enc(W) in pinned host memory and stage each matrix into HBM right before its
 * matmul, overlapping the copy with the previous matmul's compute.
 *  nimbus_encw_offload  moves the handle's Enc(W) to pinned host memory (synchronous
 *                       on `stream`) and frees the device copy; nimbus_cop_matmul
 *                       then returns EINVAL for it;
 *  nimbus_encw_reload   copies it back into a fresh device allocation (async on `stream`);
 *  nimbus_cop_stage_size  bytes of the device staging buffer for a job list
 *                       (2 x the largest non-resident tiled Enc(W), plus the largest
 *                       file-backed canonical payload; 0 if all are resident);
 *  nimbus_cop_matmul_streamed  runs the jobs in order on `stream` exactly as
 *                       nimbus_cop_matmul would (same outputs, bit for bit); the
 *                       host-resident ones are copied into alternating halves of
 *                       d_stage on the context's copy stream, job j+2's copy
 *                       overlapping job j+1's compute.  d_ws as for the largest job. */
/*  nimbus_encw_open     a FILE-backed handle on a store file written by nimbus_encw_save
 *                       (header, parameters and file size checked; verify != 0 also checks the
 *                       payload checksum in one streaming pass; NIMBUS_EIO otherwise).  Nothing is
 *                       read into memory: nimbus_cop_matmul_streamed reads the payload for each job
 *                       on its copy stream (a stream-ordered host callback into one of two pinned
 *                       buffers), uploads and tiles it while earlier jobs compute -- the paper's
 *                       Enc(W) kept on the client's disk and loaded for the next layer
 *                       (PAPER.md:300, 312-317).  A read failure during streaming is reported as
 *                       NIMBUS_EIO by nimbus_sync or the next streamed call.  nimbus_cop_matmul
 *                       refuses the handle; nimbus_encw_reload reads it into HBM. */
nimbus_status nimbus_encw_open(nimbus_ctx* ctx, const char* path, int verify, nimbus_encw** out);
nimbus_status nimbus_encw_offload(nimbus_encw* encw, void* stream);
nimbus_status nimbus_encw_reload(nimbus_encw* encw, void* stream);
int nimbus_encw_is_resident(const nimbus_encw* encw);
nimbus_status nimbus_cop_stage_size(const nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count,
                                    size_t* bytes);
nimbus_status nimbus_cop_matmul_streamed(nimbus_ctx* ctx, const nimbus_cop_job* jobs, uint32_t count, void* d_ws,
                                         size_t ws_bytes, void* d_stage, size_t stage_bytes, void* stream);
nimbus_status nimbus_cop_stage_size_u64(const nimbus_ctx* ctx, const nimbus_cop_job_u64* jobs, uint32_t count,
                                        size_t* bytes);
nimbus_status nimbus_cop_matmul_streamed_u64(nimbus_ctx* ctx, const nimbus_cop_job_u64* jobs, uint32_t count,
                                             void* d_ws, size_t ws_bytes, void* d_stage, size_t stage_bytes,
                                             void* stream);

/* Same computation with HOST buffers: copies h_X in, runs nimbus_cop_matmul,
 * copies h_cts and h_R out, and synchronises `stream` before returning. */
nimbus_status nimbus_cop_matmul_host(nimbus_ctx* ctx, const nimbus_encw* encw, const uint32_t* h_X,
                                     uint32_t k_per_query, uint32_t n_queries, uint64_t mask_seed,
                                     uint32_t* h_cts, uint32_t* h_R, void* d_ws, size_t ws_bytes,
                                     void* stream);
nimbus_status nimbus_cop_matmul_host_u64(nimbus_ctx* ctx, const nimbus_encw* encw, const uint64_t* h_X,
                                         uint32_t k_per_query, uint32_t n_queries, uint64_t mask_seed,
                                         uint32_t* h_cts, uint64_t* h_R, void* d_ws, size_t ws_bytes,
                                         void* stream);

/* A list of independent matmuls with HOST buffers (e.g. many queries, or every
 * layer of many queries' passes), pipelined: job i+1's X upload (copy stream) and
 * job i-1's ciphertext/R download (a second copy stream) run while job i computes
 * on `stream`, through 8 device staging slots.  Consecutive jobs with the same h_X
 * pointer and shape that nimbus_cop_matmul_batch would run as a same-X group (Q, K,
 * V of a layer) are uploaded once and run as one contraction launch.
 * Each job's outputs are identical to nimbus_cop_matmul_host's for it; jobs must be
 * independent (no job's h_X is another job's output).  Host buffers should be pinned (pageable
 * memory works but the copies then do not overlap).  Synchronises `stream` before
 * returning, so all h_cts / h_R are filled.  Workspace (device):
 * nimbus_cop_workspace_size_host_batch.  Errors are checked for all jobs before
 * any copy or launch. */
typedef struct {
    const nimbus_encw* encw;
    const uint32_t* h_X;          /* host, k x m, k = n_queries * k_per_query */
    uint32_t k_per_query, n_queries;
    uint64_t mask_seed;
    uint32_t* h_cts;              /* host, n_queries x n_cts x 2 x L_out x N */
    uint32_t* h_R;                /* host, k x n */
} nimbus_cop_host_job;
nimbus_status nimbus_cop_workspace_size_host_batch(const nimbus_ctx* ctx, const nimbus_cop_host_job* jobs,
                                                   uint32_t count, size_t* bytes);
nimbus_status nimbus_cop_matmul_host_batch(nimbus_ctx* ctx, const nimbus_cop_host_job* jobs, uint32_t count,
                                           void* d_ws, size_t ws_bytes, void* stream);
/* ell > 32: the same with uint64 X and R (same struct layout). */
typedef struct {
    const nimbus_encw* encw;
    const uint64_t* h_X;
    uint32_t k_per_query, n_queries;
    uint64_t mask_seed;
    uint32_t* h_cts;
    uint64_t* h_R;
} nimbus_cop_host_job_u64;
nimbus_status nimbus_cop_workspace_size_host_batch_u64(const nimbus_ctx* ctx, const nimbus_cop_host_job_u64* jobs,
                                                       uint32_t count, size_t* bytes);
nimbus_status nimbus_cop_matmul_host_batch_u64(nimbus_ctx* ctx, const nimbus_cop_host_job_u64* jobs, uint32_t count,
                                               void* d_ws, size_t ws_bytes, void* stream);

/* Step 2 alone (verification of the contraction): d_C is k x 2 x L x N uint32,
 * [alpha][comp][limb][j], the unpacked ciphertexts c[alpha] reduced mod p_i. */
nimbus_status nimbus_cop_accumulate(nimbus_ctx* ctx, const nimbus_encw* encw, const uint32_t* d_X,
                                    uint32_t k, uint32_t* d_C, void* d_ws, size_t ws_bytes,
                                    void* stream);

/* Steps 3-4 alone on an unpacked d_C (k x 2 x L x N, as produced above). */
nimbus_status nimbus_cop_pack(nimbus_ctx* ctx, const uint32_t* d_C, uint32_t k_per_query,
                              uint32_t n_queries, uint32_t n, uint64_t mask_seed, uint32_t* d_cts,
                              uint32_t* d_R, void* stream);

/* Server step 5 decryption: u = b - a*s mod q'
 * (NTT), m = floor((2 t u + q')/(2 q')) mod t, unpacked
 * Z[alpha][j] = m_theta[(alpha mod R) n + j]; Z = (X.W - R) mod t.
 *  d_cts  as written by nimbus_cop_matmul;  d_Z  k x n uint32.
 *  d_M    optional (may be NULL): n_queries x n_cts x N full decrypted slots. */
nimbus_status nimbus_decrypt(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_cts,
                             uint32_t k_per_query, uint32_t n, uint32_t n_queries, uint32_t* d_Z,
                             uint32_t* d_M, void* stream);
/* ell > 32: d_Z k x n uint64, d_M (optional) n_queries x n_cts x N uint64. */
nimbus_status nimbus_decrypt_u64(nimbus_ctx* ctx, const nimbus_sk* sk, const uint32_t* d_cts,
                                 uint32_t k_per_query, uint32_t n, uint32_t n_queries, uint64_t* d_Z,
                                 uint64_t* d_M, void* stream);

/* ------------------------------------------------------ server, step 5 --- */
/* Alg. 1 step 5: the server computes W<X>_s locally and outputs
 * <Y>_s = W<X>_s + (W<X>_c - R), the second term being its decryption of the
 * client's masked ciphertexts; the client's share is <Y>_c = R.  Orientation
 * Y = X.W.  Plaintext products are exact mod t = 2^ell
 * (int8 slices on the tensor cores, the same slicing as the contraction).
 *
 * Server plaintext weights in the tensor-core layout (the server owns W).
 *  d_W  m x n uint32 row-major; entries are taken mod 2^(8 S_x) >= t, so the
 *       products are exact mod t for any input. */
nimbus_status nimbus_plain_weights(nimbus_ctx* ctx, const uint32_t* d_W, uint32_t m, uint32_t n,
                                   void* stream, nimbus_plainw** out);
void nimbus_plainw_destroy(nimbus_plainw* w);
/* Workspace bytes for nimbus_plain_matmul (n_queries = 0) or nimbus_server_output
 * with k = k_per_query * n_queries rows. */
nimbus_status nimbus_server_workspace_size(const nimbus_ctx* ctx, const nimbus_plainw* w,
                                           uint32_t k_per_query, uint32_t n_queries, size_t* bytes);
/* d_Y = (d_X . W + d_add) mod t.  d_X k x m uint32, d_add k x n uint32 or NULL,
 * d_Y k x n uint32 (may alias d_add). */
nimbus_status nimbus_plain_matmul(nimbus_ctx* ctx, const nimbus_plainw* w, const uint32_t* d_X, uint32_t k,
                                  const uint32_t* d_add, uint32_t* d_Y, void* d_ws, size_t ws_bytes,
                                  void* stream);
/* d_Ys = (d_Xs . W + unpack(Dec(d_cts))) mod t, k = k_per_query * n_queries rows of
 * n = w's n columns; d_cts as written by nimbus_cop_matmul for the same n.
 * Decryption as nimbus_decrypt (L_out limbs, NTT, exact rounding). */
nimbus_status nimbus_server_output(nimbus_ctx* ctx, const nimbus_sk* sk, const nimbus_plainw* w,
                                   const uint32_t* d_Xs, const uint32_t* d_cts, uint32_t k_per_query,
                                   uint32_t n_queries, uint32_t* d_Ys, void* d_ws, size_t ws_bytes,
                                   void* stream);

/* The paper's t = 2^64, ell > 32 contexts: W, X, Y,
 * the added term and the shares are uint64 (k x m, m x n, k x n row-major).  Products are
 * exact mod 2^64: 8 byte slices of each operand on the int8 tensor cores, the 36 slice
 * pairs with shift < 64 (m <= 4096, NIMBUS_ESHAPE beyond).  Workspace:
 * nimbus_server_workspace_size as for the 32-bit calls. */
nimbus_status nimbus_plain_weights_u64(nimbus_ctx* ctx, const uint64_t* d_W, uint32_t m, uint32_t n,
                                       void* stream, nimbus_plainw** out);
nimbus_status nimbus_plain_matmul_u64(nimbus_ctx* ctx, const nimbus_plainw* w, const uint64_t* d_X, uint32_t k,
                                      const uint64_t* d_add, uint64_t* d_Y, void* d_ws, size_t ws_bytes,
                                      void* stream);
/* d_Ys = (d_Xs . W + unpack(Dec(d_cts))) mod 2^64 (Alg. 1 step 5 at the paper's t). */
nimbus_status nimbus_server_output_u64(nimbus_ctx* ctx, const nimbus_sk* sk, const nimbus_plainw* w,
                                       const uint64_t* d_Xs, const uint32_t* d_cts, uint32_t k_per_query,
                                       uint32_t n_queries, uint64_t* d_Ys, void* d_ws, size_t ws_bytes,
                                       void* stream);

/* ---------------------------------------------------------- test helpers --- */
/* PRG words word(seed, dom, start + i), i < count. */
nimbus_status nimbus_prg_words(uint64_t seed, uint32_t dom, uint64_t start, uint64_t count,
                               uint64_t* d_out, void* stream);
/* Negacyclic products c = a*b mod (X^N+1, p_i) through the library's NTT
 * (PAPER.md:606, 180).  d_a, d_b, d_c: count x L x N uint32. */
nimbus_status nimbus_negacyclic_mul(nimbus_ctx* ctx, const uint32_t* d_a, const uint32_t* d_b,
                                    uint32_t count, uint32_t* d_c, void* stream);
/* Software pipelining across calls: names the Enc(W) of the matmul that will FOLLOW the next
 * nimbus_cop_matmul / nimbus_cop_matmul_batch call on this context (a model's layer order is
 * static; the weights are the asynchronously loaded operand of PAPER.md:312-317).  When that next
 * call runs the resident-X contraction (k <= 128, ell <= 16), each of its CTAs, once its own last
 * Enc(W) copy is issued, prefetches into L2 the first two tiles of the same CTA of the following
 * contraction, so that launch does not start with a cold DRAM round trip.  The job-list calls
 * (nimbus_cop_matmul_batch, nimbus_cop_matmul_host_batch) do this themselves between consecutive
 * units of a list; a hint set before them names what follows the list's last unit.  A hint only:
 * never changes a result, one-shot (consumed by the next contraction launch, ignored by the other
 * kernels), `next` stays owned by the caller and must be resident and alive until that launch has
 * run (destroying it first drops the hint).  next = NULL clears a pending hint.  Returns
 * NIMBUS_EINVAL for a null ctx or an Enc(W) of another context. */
nimbus_status nimbus_cop_prefetch_next(nimbus_ctx* ctx, const nimbus_encw* next);
/* Number of library kernels launched through this context since creation. */
uint64_t nimbus_launch_count(const nimbus_ctx* ctx);
/* Name of the last contraction kernel the context launched ("k_cop_pk<4, 52>", "k_cop_tc_res<true>",
 * ...; "" before the first), owned by the context and valid until its next call.  Measurement
 * support: bench.py matches it against the kernel of the ncu capture it takes `traffic` from. */
const char* nimbus_last_contraction(const nimbus_ctx* ctx);

/* Per-stage CUDA-event timing of nimbus_cop_matmul (for the bench's live
 * roofline numbers).  When enabled, each stage -- [0] slice X (K4),
 * [1] contraction (K5/K6), [2] pack + mod-switch + mask (K7) -- is bracketed by
 * events recorded on the caller's stream.  nimbus_profile_read synchronises
 * those events and returns the accumulated milliseconds per stage in ms[3]
 * and the number of profiled calls; reset != 0 clears the totals. */
nimbus_status nimbus_profile_enable(nimbus_ctx* ctx, int on);
nimbus_status nimbus_profile_read(nimbus_ctx* ctx, double* ms, uint64_t* calls, int reset);

#ifdef __cplusplus
}
#endif
#endif /* NIMBUS_COP_H */
