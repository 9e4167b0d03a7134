"""ctypes wrapper around oracle/liboracle.so (plain C, see nimbus_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg.  Never imported by the product
package paper_2411_15707_b200/.  Numpy in, numpy out; all arithmetic happens
in the C file, whose functions cite the paper passages they implement -- except
the server's plaintext product X.W mod 2^ell (plain_matmul), a textbook numpy
integer matmul.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nimbus_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP over independent rows only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's parallel loops (execution only, no arithmetic change);
    returns the thread count now in effect (for the bench's cpu_baseline `cores`)."""
    lib()
    gomp = C.CDLL("libgomp.so.1")
    gomp.omp_set_num_threads(int(n))
    return max_threads()


def max_threads() -> int:
    lib()
    gomp = C.CDLL("libgomp.so.1")
    gomp.omp_get_max_threads.restype = C.c_int
    return int(gomp.omp_get_max_threads())


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_word.restype = C.c_uint64
        L.orc_word.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
        L.orc_words.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, u64p]
        L.orc_is_prime.restype = C.c_int
        L.orc_is_prime.argtypes = [C.c_uint64]
        L.orc_primes.restype = C.c_int
        L.orc_primes.argtypes = [C.c_uint32, C.c_uint32, u32p]
        L.orc_negacyclic_schoolbook.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, u32p]
        L.orc_negacyclic_ntt.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, u32p]
        L.orc_keygen.argtypes = [C.c_uint32, C.c_uint64, i8p]
        L.orc_encrypt_rows.argtypes = [C.c_uint32, C.c_uint32, u32p, C.c_uint32, i8p, u32p,
                                       C.c_uint32, C.c_uint32, C.c_uint64, u32p]
        L.orc_decrypt_ct.argtypes = [C.c_uint32, C.c_uint32, u32p, C.c_uint32, i8p, u32p, u32p,
                                     C.POINTER(C.c_double)]
        L.orc_cop_accumulate.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, u32p, C.c_uint32,
                                         C.c_uint32, u32p]
        L.orc_cts_per_query.restype = C.c_uint32
        L.orc_cts_per_query.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_pack_moddown_mask.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_uint32,
                                            u32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                            u32p, u32p]
        L.orc_cop_matmul.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_uint32, u32p,
                                     C.c_uint32, C.c_uint32, u32p, C.c_uint32, C.c_uint32,
                                     C.c_uint64, u32p, u32p]
        L.orc_cop_matmul_sampled.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_uint32,
                                             u32p, C.c_uint32, C.c_uint32, u32p, C.c_uint32,
                                             C.c_uint32, C.c_uint64, C.c_uint32, u32p, u32p, u32p,
                                             u32p]
        L.orc_decrypt_unpack.argtypes = [C.c_uint32, C.c_uint32, u32p, C.c_uint32, i8p, u32p,
                                         C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_void_p,
                                         C.POINTER(C.c_double)]
        L.orc_pack_moddown_mask_rr.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_uint32,
                                               u32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                               C.c_void_p, u32p, u32p]
        L.orc_cop_matmul_rr.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_uint32, u32p,
                                        C.c_uint32, C.c_uint32, u32p, C.c_uint32, C.c_uint32,
                                        C.c_uint64, u32p, u32p, u32p]
        L.orc_keygen_pk.argtypes = [C.c_uint32, C.c_uint32, u32p, i8p, C.c_uint64, u32p]
        L.orc_rerand_zero.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, C.c_uint64, C.c_uint32,
                                      C.c_uint32, u32p]
        L.orc_emb.argtypes = [u32p, C.c_uint32, C.c_uint32, C.c_uint64, u32p]
        L.orc_moddown.argtypes = [u32p, C.c_uint32, C.c_uint32, u32p]
        L.orc_sample_uniform_mod.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                             C.c_uint32, u32p]
        L.orc_sample_cbd21.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, i32p]
    return _lib


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def word(seed: int, dom: int, i: int) -> int:
    return int(lib().orc_word(seed, dom, i))


def words(seed: int, dom: int, start: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    lib().orc_words(seed, dom, start, count, out)
    return out


def is_prime(n: int) -> bool:
    return bool(lib().orc_is_prime(n))


def primes(N: int, L: int) -> np.ndarray:
    out = np.empty(L, np.uint32)
    if lib().orc_primes(N, L, out) != 0:
        raise ValueError("not enough primes")
    return out


def negacyclic_schoolbook(N, p, a, b):
    out = np.empty(N, np.uint32)
    lib().orc_negacyclic_schoolbook(N, p, _u32(a), _u32(b), out)
    return out


def negacyclic_ntt(N, p, a, b):
    out = np.empty(N, np.uint32)
    lib().orc_negacyclic_ntt(N, p, _u32(a), _u32(b), out)
    return out


def keygen(N: int, seed: int) -> np.ndarray:
    s = np.empty(N, np.int8)
    lib().orc_keygen(N, seed, s)
    return s


def encrypt_rows(N, L, pr, ell, s, W, seed) -> np.ndarray:
    W = _u32(W)
    m, n = W.shape
    out = np.empty((m, 2, L, N), np.uint32)
    lib().orc_encrypt_rows(N, L, _u32(pr), ell, np.ascontiguousarray(s, np.int8), W, m, n, seed, out)
    return out


def decrypt_ct(N, Lc, pr, ell, s, ct):
    m = np.empty(N, np.uint32)
    tv = C.c_double(0)
    lib().orc_decrypt_ct(N, Lc, _u32(pr), ell, np.ascontiguousarray(s, np.int8), _u32(ct), m,
                         C.byref(tv))
    return m, tv.value


def cop_accumulate(N, L, pr, encW, X) -> np.ndarray:
    X = _u32(X)
    k, m = X.shape
    out = np.empty((k, 2, L, N), np.uint32)
    lib().orc_cop_accumulate(N, L, _u32(pr), _u32(encW), X, k, m, out)
    return out


def cts_per_query(N, n, kq) -> int:
    return int(lib().orc_cts_per_query(N, n, kq))


def pack_moddown_mask(N, L, L_out, pr, ell, C_unpacked, kq, n_queries, n, mask_seed):
    nct = cts_per_query(N, n, kq)
    cts = np.empty((n_queries, nct, 2, L_out, N), np.uint32)
    R = np.zeros((n_queries * kq, n), np.uint32)
    lib().orc_pack_moddown_mask(N, L, L_out, _u32(pr), ell, _u32(C_unpacked), kq, n_queries, n,
                                mask_seed, cts, R)
    return cts, R


def cop_matmul(N, L, L_out, pr, ell, encW, X, n, kq, n_queries, mask_seed):
    """Alg. 1 steps 2-4 for n_queries stacked queries: returns (cts, R)."""
    encW = _u32(encW)
    X = _u32(X)
    m = encW.shape[0]
    nct = cts_per_query(N, n, kq)
    cts = np.empty((n_queries, nct, 2, L_out, N), np.uint32)
    R = np.zeros((n_queries * kq, n), np.uint32)
    lib().orc_cop_matmul(N, L, L_out, _u32(pr), ell, encW, m, n, X, kq, n_queries, mask_seed,
                         cts, R)
    return cts, R


def keygen_pk(N, L, pr, s, seed) -> np.ndarray:
    """Public key pk[comp b=0, a=1][limb][j] (reading 25)."""
    pk = np.empty((2, L, N), np.uint32)
    lib().orc_keygen_pk(N, L, _u32(pr), np.ascontiguousarray(s, np.int8), seed, pk)
    return pk


def rerand_zero(N, L, pr, pk, seed, n_cts, flood_bits) -> np.ndarray:
    """Public-key encryptions of zero z[g][comp][limb][j] for circuit privacy
    (reading 26)."""
    z = np.empty((n_cts, 2, L, N), np.uint32)
    lib().orc_rerand_zero(N, L, _u32(pr), _u32(pk), seed, n_cts, flood_bits, z)
    return z


def cop_matmul_rr(N, L, L_out, pr, ell, encW, X, n, kq, n_queries, mask_seed, Z0):
    """Alg. 1 steps 2-4 with the zero encryptions Z0 added before ModDown."""
    encW = _u32(encW)
    X = _u32(X)
    m = encW.shape[0]
    nct = cts_per_query(N, n, kq)
    cts = np.empty((n_queries, nct, 2, L_out, N), np.uint32)
    R = np.zeros((n_queries * kq, n), np.uint32)
    lib().orc_cop_matmul_rr(N, L, L_out, _u32(pr), ell, encW, m, n, X, kq, n_queries, mask_seed,
                            _u32(Z0), cts, R)
    return cts, R


def cop_matmul_sampled(N, L, L_out, pr, ell, encW, X, n, kq, n_queries, mask_seed,
                       s_query, s_theta, s_J):
    encW = _u32(encW)
    X = _u32(X)
    m = encW.shape[0]
    ns = len(s_query)
    out = np.empty((ns, 2, L_out), np.uint32)
    lib().orc_cop_matmul_sampled(N, L, L_out, _u32(pr), ell, encW, m, n, X, kq, n_queries,
                                 mask_seed, ns, _u32(s_query), _u32(s_theta), _u32(s_J), out)
    return out


def decrypt_unpack(N, L_out, pr, ell, s, cts, kq, n_queries, n, want_full=False):
    cts = _u32(cts)
    nct = cts_per_query(N, n, kq)
    Z = np.zeros((n_queries * kq, n), np.uint32)
    full = np.empty((n_queries * nct, N), np.uint32) if want_full else None
    tv = C.c_double(0)
    lib().orc_decrypt_unpack(N, L_out, _u32(pr), ell, np.ascontiguousarray(s, np.int8), cts, kq,
                             n_queries, n, Z,
                             full.ctypes.data_as(C.c_void_p) if full is not None else None,
                             C.byref(tv))
    return Z, full, tv.value


def plain_matmul(X, W, ell) -> np.ndarray:
    """X.W mod 2^ell (Alg. 1 step 5's W<X>_s; orientation SURVEY.md
    §8(c) #10): the textbook product in uint64 -- exact mod 2^64, hence mod 2^ell
    for ell <= 32 -- then reduced mod t."""
    t_mask = np.uint64((1 << ell) - 1)
    Y = _u32(X).astype(np.uint64) @ _u32(W).astype(np.uint64)
    return (Y & t_mask).astype(np.uint32)


def server_output(N, L_out, pr, ell, s, cts, Xs, W, kq, n_queries):
    """Alg. 1 step 5: <Y>_s = W<X>_s + (W<X>_c - R) mod 2^ell, the
    second term being the server's decryption + unpack of the client's ciphertexts."""
    Z, _, _ = decrypt_unpack(N, L_out, pr, ell, s, cts, kq, n_queries, _u32(W).shape[1])
    t_mask = np.uint64((1 << ell) - 1)
    return ((plain_matmul(Xs, W, ell).astype(np.uint64) + Z.astype(np.uint64)) & t_mask).astype(np.uint32)


def emb(pr, ell, w) -> np.ndarray:
    out = np.empty(len(pr), np.uint32)
    lib().orc_emb(_u32(pr), len(pr), ell, w, out)
    return out


def moddown(res, L_out, pr) -> np.ndarray:
    r = _u32(res).copy()
    lib().orc_moddown(r, len(pr), L_out, _u32(pr))
    return r[:L_out]


def sample_uniform_mod(seed, dom, start, count, p):
    out = np.empty(count, np.uint32)
    lib().orc_sample_uniform_mod(seed, dom, start, count, p, out)
    return out


def sample_cbd21(seed, dom, start, count):
    out = np.empty(count, np.int32)
    lib().orc_sample_cbd21(seed, dom, start, count, out)
    return out
