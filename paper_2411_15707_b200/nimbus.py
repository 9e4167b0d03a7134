"""Thin ctypes binding of libnimbus_cop.so (include/nimbus_cop.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  Functions carry the C names; tensors are torch CUDA tensors
(contiguous, the dtype the header states), passed as data_ptr(); the stream
defaults to torch's current stream.  There is no CPU fallback: if the library
is missing or no sm_100 device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# NIMBUS_LIB selects an experiment build of the same library (e.g. libnimbus_cop_<variant>.so)
LIB_PATH = os.path.join(_PKG, os.environ.get("NIMBUS_LIB", "libnimbus_cop.so"))

STATUS = {0: "NIMBUS_OK", -1: "NIMBUS_EINVAL", -2: "NIMBUS_ESHAPE", -3: "NIMBUS_ERANGE",
          -4: "NIMBUS_ENOISE", -5: "NIMBUS_ECUDA", -6: "NIMBUS_ENOMEM", -7: "NIMBUS_EIO", -8: "NIMBUS_EARCH"}
IMPL_TCGEN05, IMPL_CUDACORE = 0, 1
FLAG_CHECK_RANGE = 1
FLAG_LARGE_K = 2


class NimbusError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


class nimbus_params(C.Structure):
    _fields_ = [("N", C.c_uint32), ("L", C.c_uint32), ("ell", C.c_uint32),
                ("L_out", C.c_uint32), ("impl", C.c_uint32), ("flags", C.c_uint32)]


_lib = None
_vp, _u32, _u64, _sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_size_t
_SIGS = {
    "nimbus_ctx_create": (C.c_int, [C.POINTER(nimbus_params), C.c_int, C.POINTER(_vp)]),
    "nimbus_ctx_destroy": (None, [_vp]),
    "nimbus_ctx_primes": (C.c_int, [_vp, C.POINTER(_u32)]),
    "nimbus_last_error": (C.c_char_p, [_vp]),
    "nimbus_sync": (C.c_int, [_vp, _vp]),
    "nimbus_keygen": (C.c_int, [_vp, _u64, _vp, C.POINTER(_vp)]),
    "nimbus_sk_destroy": (None, [_vp]),
    "nimbus_sk_export": (C.c_int, [_vp, _vp, _vp]),
    "nimbus_encrypt_weights": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, C.POINTER(_vp)]),
    "nimbus_encw_destroy": (None, [_vp]),
    "nimbus_encw_bytes": (_sz, [_vp]),
    "nimbus_encw_export": (C.c_int, [_vp, _vp, _vp]),
    "nimbus_encw_import": (C.c_int, [_vp, _vp, _u32, _u32, _vp, C.POINTER(_vp)]),
    "nimbus_cop_out_count": (C.c_int, [_vp, _u32, _u32, _u32, C.POINTER(_u32)]),
    "nimbus_cop_workspace_size": (C.c_int, [_vp, _vp, _u32, C.POINTER(_sz)]),
    "nimbus_cop_matmul": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, _vp, _vp, _sz, _vp]),
    "nimbus_cop_matmul_host": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, _vp, _vp, _sz, _vp]),
    "nimbus_cop_accumulate": (C.c_int, [_vp, _vp, _vp, _u32, _vp, _vp, _sz, _vp]),
    "nimbus_cop_pack": (C.c_int, [_vp, _vp, _u32, _u32, _u32, _u64, _vp, _vp, _vp]),
    "nimbus_decrypt": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u32, _vp, _vp, _vp]),
    "nimbus_prg_words": (C.c_int, [_u64, _u32, _u64, _u64, _vp, _vp]),
    "nimbus_negacyclic_mul": (C.c_int, [_vp, _vp, _vp, _u32, _vp, _vp]),
    "nimbus_launch_count": (_u64, [_vp]),
    "nimbus_last_contraction": (C.c_char_p, [_vp]),
    "nimbus_cop_prefetch_next": (C.c_int, [_vp, _vp]),
    "nimbus_cop_workspace_size_batch": (C.c_int, [_vp, _vp, _u32, C.POINTER(_sz)]),
    "nimbus_cop_matmul_batch": (C.c_int, [_vp, _vp, _u32, _vp, _sz, _vp]),
    "nimbus_profile_enable": (C.c_int, [_vp, C.c_int]),
    "nimbus_profile_read": (C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(_u64), C.c_int]),
    "nimbus_encrypt_weights_u64": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, C.POINTER(_vp)]),
    "nimbus_cop_matmul_u64": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, _vp, _vp, _sz, _vp]),
    "nimbus_decrypt_u64": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u32, _vp, _vp, _vp]),
    "nimbus_cop_matmul_host_u64": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, _vp, _vp, _sz, _vp]),
    "nimbus_cop_workspace_size_host_batch": (C.c_int, [_vp, _vp, _u32, C.POINTER(_sz)]),
    "nimbus_cop_matmul_host_batch": (C.c_int, [_vp, _vp, _u32, _vp, _sz, _vp]),
    "nimbus_cop_workspace_size_host_batch_u64": (C.c_int, [_vp, _vp, _u32, C.POINTER(_sz)]),
    "nimbus_cop_matmul_host_batch_u64": (C.c_int, [_vp, _vp, _u32, _vp, _sz, _vp]),
    "nimbus_cop_workspace_size_batch_u64": (C.c_int, [_vp, _vp, _u32, C.POINTER(_sz)]),
    "nimbus_cop_matmul_batch_u64": (C.c_int, [_vp, _vp, _u32, _vp, _sz, _vp]),
    "nimbus_cop_stage_size_u64": (C.c_int, [_vp, _vp, _u32, C.POINTER(_sz)]),
    "nimbus_cop_matmul_streamed_u64": (C.c_int, [_vp, _vp, _u32, _vp, _sz, _vp, _sz, _vp]),
    "nimbus_encw_save": (C.c_int, [_vp, C.c_char_p]),
    "nimbus_encw_load": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "nimbus_encw_open": (C.c_int, [_vp, C.c_char_p, C.c_int, C.POINTER(_vp)]),
    "nimbus_encw_offload": (C.c_int, [_vp, _vp]),
    "nimbus_encw_reload": (C.c_int, [_vp, _vp]),
    "nimbus_encw_is_resident": (C.c_int, [_vp]),
    "nimbus_cop_stage_size": (C.c_int, [_vp, _vp, _u32, C.POINTER(_sz)]),
    "nimbus_cop_matmul_streamed": (C.c_int, [_vp, _vp, _u32, _vp, _sz, _vp, _sz, _vp]),
    "nimbus_plain_weights": (C.c_int, [_vp, _vp, _u32, _u32, _vp, C.POINTER(_vp)]),
    "nimbus_plainw_destroy": (None, [_vp]),
    "nimbus_server_workspace_size": (C.c_int, [_vp, _vp, _u32, _u32, C.POINTER(_sz)]),
    "nimbus_plain_matmul": (C.c_int, [_vp, _vp, _vp, _u32, _vp, _vp, _vp, _sz, _vp]),
    "nimbus_server_output": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _u32, _u32, _vp, _vp, _sz, _vp]),
    "nimbus_plain_weights_u64": (C.c_int, [_vp, _vp, _u32, _u32, _vp, C.POINTER(_vp)]),
    "nimbus_plain_matmul_u64": (C.c_int, [_vp, _vp, _vp, _u32, _vp, _vp, _vp, _sz, _vp]),
    "nimbus_server_output_u64": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _u32, _u32, _vp, _vp, _sz, _vp]),
    "nimbus_encrypt_weights_into": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp]),
    "nimbus_encrypt_weights_into_u64": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp]),
    "nimbus_keygen_pk": (C.c_int, [_vp, _vp, _u64, _vp, C.POINTER(_vp)]),
    "nimbus_pk_destroy": (None, [_vp]),
    "nimbus_pk_export": (C.c_int, [_vp, _vp, _vp]),
    "nimbus_pk_import": (C.c_int, [_vp, _vp, _vp, C.POINTER(_vp)]),
    "nimbus_rerand_flood_max": (C.c_int, [_vp, _vp, _u32, C.POINTER(_u32)]),
    "nimbus_rerand_prepare": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _u32, _vp, _vp]),
    "nimbus_cop_matmul_rr": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "nimbus_cop_matmul_rr_u64": (C.c_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, _vp, _vp, _vp, _sz, _vp]),
}
EXPORTED = tuple(_SIGS)


def lib():
    """Load the in-tree library (built by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if "NIMBUS_LIB" in os.environ and not hasattr(L, name):
                continue          # an older experiment build may lack newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _stream(stream):
    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def _ptr(t: torch.Tensor, dtype=None, what=""):
    if t is None:
        return None
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{what}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


class _Handle:
    _destroy = None

    def __init__(self, ptr, owner=None):
        self.ptr = ptr
        self.owner = owner

    def close(self):
        if self.ptr:
            getattr(lib(), self._destroy)(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context(_Handle):
    _destroy = "nimbus_ctx_destroy"

    def __init__(self, ptr, params: nimbus_params, device: int):
        super().__init__(ptr)
        self.params = params
        self.device = device

    @property
    def N(self):
        return self.params.N

    @property
    def L(self):
        return self.params.L

    @property
    def L_out(self):
        return self.params.L_out

    @property
    def ell(self):
        return self.params.ell


class SecretKey(_Handle):
    _destroy = "nimbus_sk_destroy"


class PublicKey(_Handle):
    _destroy = "nimbus_pk_destroy"


class EncW(_Handle):
    _destroy = "nimbus_encw_destroy"

    def __init__(self, ptr, ctx, m, n):
        super().__init__(ptr, ctx)
        self.m, self.n = m, n


class PlainW(_Handle):
    _destroy = "nimbus_plainw_destroy"

    def __init__(self, ptr, ctx, m, n):
        super().__init__(ptr, ctx)
        self.m, self.n = m, n


def _check(st: int, ctx=None):
    if st != 0:
        msg = lib().nimbus_last_error(ctx.ptr if ctx is not None else None)
        raise NimbusError(st, msg.decode() if msg else "")


# ------------------------------------------------------------------ C-named API
def nimbus_ctx_create(N, L, ell, L_out, impl=IMPL_TCGEN05, flags=0, device=0) -> Context:
    prm = nimbus_params(N, L, ell, L_out, impl, flags)
    out = C.c_void_p()
    _check(lib().nimbus_ctx_create(C.byref(prm), device, C.byref(out)))
    return Context(out, prm, device)


def nimbus_ctx_primes(ctx: Context):
    arr = (_u32 * ctx.L)()
    _check(lib().nimbus_ctx_primes(ctx.ptr, arr), ctx)
    return [int(x) for x in arr]


def nimbus_sync(ctx: Context, stream=None):
    _check(lib().nimbus_sync(ctx.ptr, _stream(stream)), ctx)


def nimbus_keygen(ctx: Context, seed: int, stream=None) -> SecretKey:
    out = C.c_void_p()
    _check(lib().nimbus_keygen(ctx.ptr, seed, _stream(stream), C.byref(out)), ctx)
    return SecretKey(out, ctx)


def nimbus_sk_export(sk: SecretKey, stream=None) -> torch.Tensor:
    ctx = sk.owner
    s = torch.empty(ctx.N, dtype=torch.int8, device=f"cuda:{ctx.device}")
    _check(lib().nimbus_sk_export(sk.ptr, _ptr(s), _stream(stream)), ctx)
    return s


def nimbus_encrypt_weights(ctx: Context, sk: SecretKey, W: torch.Tensor, seed: int, stream=None) -> EncW:
    m, n = W.shape
    out = C.c_void_p()
    _check(lib().nimbus_encrypt_weights(ctx.ptr, sk.ptr, _ptr(W, torch.int32, "W"), m, n, seed,
                                        _stream(stream), C.byref(out)), ctx)
    return EncW(out, ctx, m, n)


def nimbus_encrypt_weights_u64(ctx: Context, sk: SecretKey, W: torch.Tensor, seed: int, stream=None) -> EncW:
    """ell > 32: W is an int64 tensor holding uint64 values."""
    m, n = W.shape
    out = C.c_void_p()
    _check(lib().nimbus_encrypt_weights_u64(ctx.ptr, sk.ptr, _ptr(W, torch.int64, "W"), m, n, seed,
                                            _stream(stream), C.byref(out)), ctx)
    return EncW(out, ctx, m, n)


def nimbus_encrypt_weights_into(ctx: Context, sk: SecretKey, W: torch.Tensor, seed: int, w: EncW, stream=None):
    """Re-encrypt W (same shape as the handle's) into the existing handle w."""
    if tuple(W.shape) != (w.m, w.n):
        raise ValueError(f"W shape {tuple(W.shape)} != handle ({w.m}, {w.n})")
    wide = ctx.ell > 32
    fn = lib().nimbus_encrypt_weights_into_u64 if wide else lib().nimbus_encrypt_weights_into
    _check(fn(ctx.ptr, sk.ptr, _ptr(W, torch.int64 if wide else torch.int32, "W"), seed, _stream(stream), w.ptr), ctx)
    return w


def nimbus_encw_bytes(w: EncW) -> int:
    return int(lib().nimbus_encw_bytes(w.ptr))


def nimbus_encw_export(w: EncW, stream=None) -> torch.Tensor:
    ctx = w.owner
    out = torch.empty((w.m, 2, ctx.L, ctx.N), dtype=torch.int32, device=f"cuda:{ctx.device}")
    _check(lib().nimbus_encw_export(w.ptr, _ptr(out), _stream(stream)), ctx)
    return out


def nimbus_encw_import(ctx: Context, canon: torch.Tensor, n: int, stream=None) -> EncW:
    m = canon.shape[0]
    out = C.c_void_p()
    _check(lib().nimbus_encw_import(ctx.ptr, _ptr(canon, torch.int32, "canon"), m, n, _stream(stream),
                                    C.byref(out)), ctx)
    return EncW(out, ctx, m, n)


def nimbus_cop_out_count(ctx: Context, k_per_query: int, n: int, n_queries: int = 1) -> int:
    """Packed output ciphertexts of a call (per query with the default n_queries = 1)."""
    out = _u32()
    _check(lib().nimbus_cop_out_count(ctx.ptr, k_per_query, n, n_queries, C.byref(out)), ctx)
    return int(out.value)


def nimbus_cop_workspace_size(ctx: Context, w: EncW, k: int) -> int:
    out = _sz()
    _check(lib().nimbus_cop_workspace_size(ctx.ptr, w.ptr, k, C.byref(out)), ctx)
    return int(out.value)


def alloc_workspace(ctx: Context, w: EncW, k: int) -> torch.Tensor:
    return torch.empty(nimbus_cop_workspace_size(ctx, w, k), dtype=torch.uint8, device=f"cuda:{ctx.device}")


def alloc_outputs(ctx: Context, w: EncW, k_per_query: int, n_queries: int, pin: bool = False,
                  device=None):
    nct = nimbus_cop_out_count(ctx, k_per_query, w.n)
    dev = device if device is not None else f"cuda:{ctx.device}"
    kw = dict(dtype=torch.int32, device=dev)
    if pin:
        kw["pin_memory"] = True
    cts = torch.empty((n_queries, nct, 2, ctx.L_out, ctx.N), **kw)
    R = torch.empty((n_queries * k_per_query, w.n), **kw)
    return cts, R


def nimbus_cop_matmul(ctx: Context, w: EncW, X: torch.Tensor, k_per_query: int, n_queries: int,
                      mask_seed: int, cts: torch.Tensor, R: torch.Tensor, ws: torch.Tensor,
                      stream=None):
    _check(lib().nimbus_cop_matmul(ctx.ptr, w.ptr, _ptr(X, torch.int32, "X"), k_per_query, n_queries,
                                   mask_seed, _ptr(cts, torch.int32, "cts"), _ptr(R, torch.int32, "R"),
                                   _ptr(ws), ws.numel(), _stream(stream)), ctx)
    return cts, R


def alloc_outputs_u64(ctx: Context, w: EncW, k_per_query: int, n_queries: int):
    nct = nimbus_cop_out_count(ctx, k_per_query, w.n)
    dev = f"cuda:{ctx.device}"
    cts = torch.empty((n_queries, nct, 2, ctx.L_out, ctx.N), dtype=torch.int32, device=dev)
    R = torch.empty((n_queries * k_per_query, w.n), dtype=torch.int64, device=dev)
    return cts, R


def nimbus_cop_matmul_u64(ctx: Context, w: EncW, X: torch.Tensor, k_per_query: int, n_queries: int,
                          mask_seed: int, cts: torch.Tensor, R: torch.Tensor, ws: torch.Tensor, stream=None):
    """ell > 32: X and R are int64 tensors holding uint64 values."""
    _check(lib().nimbus_cop_matmul_u64(ctx.ptr, w.ptr, _ptr(X, torch.int64, "X"), k_per_query, n_queries,
                                       mask_seed, _ptr(cts, torch.int32, "cts"), _ptr(R, torch.int64, "R"),
                                       _ptr(ws), ws.numel(), _stream(stream)), ctx)
    return cts, R


def nimbus_keygen_pk(ctx: Context, sk: SecretKey, seed: int, stream=None) -> PublicKey:
    out = C.c_void_p()
    _check(lib().nimbus_keygen_pk(ctx.ptr, sk.ptr, seed, _stream(stream), C.byref(out)), ctx)
    return PublicKey(out, ctx)


def nimbus_pk_export(pk: PublicKey, stream=None) -> torch.Tensor:
    ctx = pk.owner
    out = torch.empty((2, ctx.L, ctx.N), dtype=torch.int32, device=f"cuda:{ctx.device}")
    _check(lib().nimbus_pk_export(pk.ptr, _ptr(out), _stream(stream)), ctx)
    return out


def nimbus_pk_import(ctx: Context, pk: torch.Tensor, stream=None) -> PublicKey:
    out = C.c_void_p()
    _check(lib().nimbus_pk_import(ctx.ptr, _ptr(pk, torch.int32, "pk"), _stream(stream), C.byref(out)), ctx)
    return PublicKey(out, ctx)


def nimbus_rerand_flood_max(ctx: Context, w: EncW, k_per_query: int) -> int:
    out = _u32()
    _check(lib().nimbus_rerand_flood_max(ctx.ptr, w.ptr, k_per_query, C.byref(out)), ctx)
    return int(out.value)


def alloc_zero(ctx: Context, w: EncW, k_per_query: int, n_queries: int) -> torch.Tensor:
    nct = nimbus_cop_out_count(ctx, k_per_query, w.n, n_queries)
    return torch.empty((nct, 2, ctx.L, ctx.N), dtype=torch.int32, device=f"cuda:{ctx.device}")


def nimbus_rerand_prepare(ctx: Context, pk: PublicKey, w: EncW, k_per_query: int, n_queries: int, seed: int,
                          flood_bits: int, zero: torch.Tensor = None, stream=None) -> torch.Tensor:
    if zero is None:
        zero = alloc_zero(ctx, w, k_per_query, n_queries)
    _check(lib().nimbus_rerand_prepare(ctx.ptr, pk.ptr, w.ptr, k_per_query, n_queries, seed, flood_bits,
                                       _ptr(zero, torch.int32, "zero"), _stream(stream)), ctx)
    return zero


def nimbus_cop_matmul_rr(ctx: Context, w: EncW, X: torch.Tensor, k_per_query: int, n_queries: int,
                         mask_seed: int, zero: torch.Tensor, cts: torch.Tensor, R: torch.Tensor, ws: torch.Tensor,
                         stream=None):
    _check(lib().nimbus_cop_matmul_rr(ctx.ptr, w.ptr, _ptr(X, torch.int32, "X"), k_per_query, n_queries,
                                      mask_seed, _ptr(zero, torch.int32, "zero"), _ptr(cts, torch.int32, "cts"),
                                      _ptr(R, torch.int32, "R"), _ptr(ws), ws.numel(), _stream(stream)), ctx)
    return cts, R


def nimbus_cop_matmul_rr_u64(ctx: Context, w: EncW, X: torch.Tensor, k_per_query: int, n_queries: int,
                             mask_seed: int, zero: torch.Tensor, cts: torch.Tensor, R: torch.Tensor,
                             ws: torch.Tensor, stream=None):
    _check(lib().nimbus_cop_matmul_rr_u64(ctx.ptr, w.ptr, _ptr(X, torch.int64, "X"), k_per_query, n_queries,
                                          mask_seed, _ptr(zero, torch.int32, "zero"),
                                          _ptr(cts, torch.int32, "cts"), _ptr(R, torch.int64, "R"), _ptr(ws),
                                          ws.numel(), _stream(stream)), ctx)
    return cts, R


class nimbus_cop_job(C.Structure):
    _fields_ = [("encw", _vp), ("d_X", _vp), ("k_per_query", _u32), ("n_queries", _u32),
                ("mask_seed", _u64), ("d_cts", _vp), ("d_R", _vp)]


def _jobs(jobs, wide=False):
    """jobs: sequence of dicts with encw, X, k_per_query, n_queries, mask_seed, cts, R
    (X and R int64 holding uint64 when wide, i.e. ell > 32: nimbus_cop_job_u64, same layout)."""
    dt = torch.int64 if wide else torch.int32
    arr = (nimbus_cop_job * len(jobs))()
    for i, j in enumerate(jobs):
        arr[i] = nimbus_cop_job(j["encw"].ptr, _ptr(j["X"], dt, "X"), j["k_per_query"], j["n_queries"],
                                j["mask_seed"], _ptr(j["cts"], torch.int32, "cts"), _ptr(j["R"], dt, "R"))
    return arr


def nimbus_cop_workspace_size_batch(ctx: Context, jobs) -> int:
    out = _sz()
    _check(lib().nimbus_cop_workspace_size_batch(ctx.ptr, _jobs(jobs), len(jobs), C.byref(out)), ctx)
    return int(out.value)


def nimbus_cop_matmul_batch(ctx: Context, jobs, ws: torch.Tensor, stream=None):
    arr = _jobs(jobs)
    _check(lib().nimbus_cop_matmul_batch(ctx.ptr, arr, len(jobs), _ptr(ws), ws.numel(), _stream(stream)), ctx)


def nimbus_encw_save(w: EncW, path: str):
    _check(lib().nimbus_encw_save(w.ptr, path.encode()), w.owner)


def nimbus_encw_load(ctx: Context, path: str, m: int = None, n: int = None) -> EncW:
    """Enc(W) from a store file; m, n are read from the file (the arguments only label the handle)."""
    out = C.c_void_p()
    _check(lib().nimbus_encw_load(ctx.ptr, path.encode(), C.byref(out)), ctx)
    import struct
    with open(path, "rb") as f:
        hdr = struct.unpack("<8s6I", f.read(32))
    return EncW(out, ctx, hdr[5], hdr[6])


def nimbus_encw_open(ctx: Context, path: str, verify: bool = False) -> EncW:
    """File-backed Enc(W) handle on a store file: its payload is read from disk per
    nimbus_cop_matmul_streamed job; m, n come from the file header."""
    out = C.c_void_p()
    _check(lib().nimbus_encw_open(ctx.ptr, path.encode(), 1 if verify else 0, C.byref(out)), ctx)
    import struct
    with open(path, "rb") as f:
        hdr = struct.unpack("<8s6I", f.read(32))
    return EncW(out, ctx, hdr[5], hdr[6])


def nimbus_encw_offload(w: EncW, stream=None):
    _check(lib().nimbus_encw_offload(w.ptr, _stream(stream)), w.owner)


def nimbus_encw_reload(w: EncW, stream=None):
    _check(lib().nimbus_encw_reload(w.ptr, _stream(stream)), w.owner)


def nimbus_encw_is_resident(w: EncW) -> bool:
    return bool(lib().nimbus_encw_is_resident(w.ptr))


def nimbus_cop_stage_size(ctx: Context, jobs) -> int:
    out = _sz()
    _check(lib().nimbus_cop_stage_size(ctx.ptr, _jobs(jobs), len(jobs), C.byref(out)), ctx)
    return int(out.value)


def nimbus_cop_matmul_streamed(ctx: Context, jobs, ws: torch.Tensor, stage: torch.Tensor = None, stream=None):
    arr = _jobs(jobs)
    _check(lib().nimbus_cop_matmul_streamed(ctx.ptr, arr, len(jobs), _ptr(ws), ws.numel(),
                                            _ptr(stage) if stage is not None else None,
                                            stage.numel() if stage is not None else 0, _stream(stream)), ctx)


def nimbus_cop_workspace_size_batch_u64(ctx: Context, jobs) -> int:
    out = _sz()
    _check(lib().nimbus_cop_workspace_size_batch_u64(ctx.ptr, _jobs(jobs, True), len(jobs), C.byref(out)), ctx)
    return int(out.value)


def nimbus_cop_matmul_batch_u64(ctx: Context, jobs, ws: torch.Tensor, stream=None):
    arr = _jobs(jobs, True)
    _check(lib().nimbus_cop_matmul_batch_u64(ctx.ptr, arr, len(jobs), _ptr(ws), ws.numel(), _stream(stream)), ctx)


def nimbus_cop_stage_size_u64(ctx: Context, jobs) -> int:
    out = _sz()
    _check(lib().nimbus_cop_stage_size_u64(ctx.ptr, _jobs(jobs, True), len(jobs), C.byref(out)), ctx)
    return int(out.value)


def nimbus_cop_matmul_streamed_u64(ctx: Context, jobs, ws: torch.Tensor, stage: torch.Tensor = None, stream=None):
    arr = _jobs(jobs, True)
    _check(lib().nimbus_cop_matmul_streamed_u64(ctx.ptr, arr, len(jobs), _ptr(ws), ws.numel(),
                                                _ptr(stage) if stage is not None else None,
                                                stage.numel() if stage is not None else 0, _stream(stream)), ctx)


def nimbus_cop_matmul_host(ctx: Context, w: EncW, X_host: torch.Tensor, k_per_query: int,
                           n_queries: int, mask_seed: int, cts_host: torch.Tensor,
                           R_host: torch.Tensor, ws: torch.Tensor, stream=None):
    for t, nm in ((X_host, "X"), (cts_host, "cts"), (R_host, "R")):
        if t.is_cuda:
            raise ValueError(f"{nm} must be a host tensor")
    _check(lib().nimbus_cop_matmul_host(ctx.ptr, w.ptr, _ptr(X_host, torch.int32, "X"), k_per_query,
                                        n_queries, mask_seed, _ptr(cts_host, torch.int32, "cts"),
                                        _ptr(R_host, torch.int32, "R"), _ptr(ws), ws.numel(),
                                        _stream(stream)), ctx)
    return cts_host, R_host


def nimbus_cop_matmul_host_u64(ctx: Context, w: EncW, X_host: torch.Tensor, k_per_query: int,
                               n_queries: int, mask_seed: int, cts_host: torch.Tensor,
                               R_host: torch.Tensor, ws: torch.Tensor, stream=None):
    for t, nm in ((X_host, "X"), (cts_host, "cts"), (R_host, "R")):
        if t.is_cuda:
            raise ValueError(f"{nm} must be a host tensor")
    _check(lib().nimbus_cop_matmul_host_u64(ctx.ptr, w.ptr, _ptr(X_host, torch.int64, "X"), k_per_query,
                                            n_queries, mask_seed, _ptr(cts_host, torch.int32, "cts"),
                                            _ptr(R_host, torch.int64, "R"), _ptr(ws), ws.numel(),
                                            _stream(stream)), ctx)
    return cts_host, R_host


class nimbus_cop_host_job(C.Structure):
    _fields_ = [("encw", _vp), ("h_X", _vp), ("k_per_query", _u32), ("n_queries", _u32),
                ("mask_seed", _u64), ("h_cts", _vp), ("h_R", _vp)]


def _host_jobs(jobs, wide=False):
    """jobs: sequence of dicts with encw, X, k_per_query, n_queries, mask_seed, cts, R -- all HOST
    tensors (pinned for overlap); X and R int64 holding uint64 when wide (ell > 32)."""
    dt = torch.int64 if wide else torch.int32
    arr = (nimbus_cop_host_job * len(jobs))()
    for i, j in enumerate(jobs):
        for nm in ("X", "cts", "R"):
            if j[nm].is_cuda:
                raise ValueError(f"job {i}: {nm} must be a host tensor")
        arr[i] = nimbus_cop_host_job(j["encw"].ptr, _ptr(j["X"], dt, "X"), j["k_per_query"], j["n_queries"],
                                     j["mask_seed"], _ptr(j["cts"], torch.int32, "cts"), _ptr(j["R"], dt, "R"))
    return arr


def nimbus_cop_workspace_size_host_batch(ctx: Context, jobs, wide=False) -> int:
    out = _sz()
    fn = lib().nimbus_cop_workspace_size_host_batch_u64 if wide else lib().nimbus_cop_workspace_size_host_batch
    _check(fn(ctx.ptr, _host_jobs(jobs, wide), len(jobs), C.byref(out)), ctx)
    return int(out.value)


def nimbus_cop_matmul_host_batch(ctx: Context, jobs, ws: torch.Tensor, stream=None, wide=False):
    """Pipelined host-buffer job list (uploads / downloads overlap the compute); returns
    when every job's cts and R are in host memory."""
    arr = _host_jobs(jobs, wide)
    fn = lib().nimbus_cop_matmul_host_batch_u64 if wide else lib().nimbus_cop_matmul_host_batch
    _check(fn(ctx.ptr, arr, len(jobs), _ptr(ws), ws.numel(), _stream(stream)), ctx)


def nimbus_cop_accumulate(ctx: Context, w: EncW, X: torch.Tensor, ws: torch.Tensor, C_out=None,
                          stream=None) -> torch.Tensor:
    k = X.shape[0]
    if C_out is None:
        C_out = torch.empty((k, 2, ctx.L, ctx.N), dtype=torch.int32, device=X.device)
    _check(lib().nimbus_cop_accumulate(ctx.ptr, w.ptr, _ptr(X, torch.int32, "X"), k,
                                       _ptr(C_out, torch.int32, "C"), _ptr(ws), ws.numel(),
                                       _stream(stream)), ctx)
    return C_out


def nimbus_cop_pack(ctx: Context, C_in: torch.Tensor, k_per_query: int, n_queries: int, n: int,
                    mask_seed: int, stream=None):
    nct = nimbus_cop_out_count(ctx, k_per_query, n)
    cts = torch.empty((n_queries, nct, 2, ctx.L_out, ctx.N), dtype=torch.int32, device=C_in.device)
    R = torch.empty((n_queries * k_per_query, n), dtype=torch.int32, device=C_in.device)
    _check(lib().nimbus_cop_pack(ctx.ptr, _ptr(C_in, torch.int32, "C"), k_per_query, n_queries, n,
                                 mask_seed, _ptr(cts), _ptr(R), _stream(stream)), ctx)
    return cts, R


def nimbus_decrypt(ctx: Context, sk: SecretKey, cts: torch.Tensor, k_per_query: int, n_queries: int,
                   n: int, want_full: bool = False, stream=None):
    Z = torch.zeros((n_queries * k_per_query, n), dtype=torch.int32, device=cts.device)
    M = None
    if want_full:
        nct = nimbus_cop_out_count(ctx, k_per_query, n)
        M = torch.empty((n_queries * nct, ctx.N), dtype=torch.int32, device=cts.device)
    _check(lib().nimbus_decrypt(ctx.ptr, sk.ptr, _ptr(cts, torch.int32, "cts"), k_per_query, n,
                                n_queries, _ptr(Z), _ptr(M) if M is not None else None, _stream(stream)), ctx)
    return Z, M


def nimbus_decrypt_u64(ctx: Context, sk: SecretKey, cts: torch.Tensor, k_per_query: int, n_queries: int,
                       n: int, want_full: bool = False, stream=None):
    Z = torch.zeros((n_queries * k_per_query, n), dtype=torch.int64, device=cts.device)
    M = None
    if want_full:
        nct = nimbus_cop_out_count(ctx, k_per_query, n)
        M = torch.empty((n_queries * nct, ctx.N), dtype=torch.int64, device=cts.device)
    _check(lib().nimbus_decrypt_u64(ctx.ptr, sk.ptr, _ptr(cts, torch.int32, "cts"), k_per_query, n,
                                    n_queries, _ptr(Z), _ptr(M) if M is not None else None, _stream(stream)), ctx)
    return Z, M


def from_numpy_u64(a, device) -> torch.Tensor:
    import numpy as np
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(device)


def to_numpy_u64(t: torch.Tensor):
    import numpy as np
    return t.detach().cpu().contiguous().numpy().view(np.uint64)


def nimbus_prg_words(seed: int, dom: int, start: int, count: int, device="cuda:0", stream=None):
    out = torch.empty(count, dtype=torch.int64, device=device)
    st = lib().nimbus_prg_words(seed, dom, start, count, _ptr(out), _stream(stream))
    if st != 0:
        raise NimbusError(st, "prg_words")
    return out


def nimbus_negacyclic_mul(ctx: Context, a: torch.Tensor, b: torch.Tensor, stream=None) -> torch.Tensor:
    count = a.shape[0]
    c = torch.empty_like(a)
    _check(lib().nimbus_negacyclic_mul(ctx.ptr, _ptr(a, torch.int32, "a"), _ptr(b, torch.int32, "b"),
                                       count, _ptr(c), _stream(stream)), ctx)
    return c


def nimbus_launch_count(ctx: Context) -> int:
    return int(lib().nimbus_launch_count(ctx.ptr))


def nimbus_last_contraction(ctx: Context) -> str:
    return lib().nimbus_last_contraction(ctx.ptr).decode()


def nimbus_cop_prefetch_next(ctx: Context, nxt=None):
    """Hint: `nxt` is the Enc(W) of the matmul after the next call (see the header)."""
    _check(lib().nimbus_cop_prefetch_next(ctx.ptr, nxt.ptr if nxt is not None else None), ctx)


def nimbus_profile_enable(ctx: Context, on: bool = True):
    _check(lib().nimbus_profile_enable(ctx.ptr, int(on)), ctx)


def nimbus_profile_read(ctx: Context, reset: bool = True):
    """-> (ms[slice, contraction, pack] accumulated, number of profiled calls)."""
    ms = (C.c_double * 3)()
    calls = _u64()
    _check(lib().nimbus_profile_read(ctx.ptr, ms, C.byref(calls), int(reset)), ctx)
    return [float(x) for x in ms], int(calls.value)


# ------------------------------------------------------------------ server, Alg. 1 step 5
def nimbus_plain_weights(ctx: Context, W: torch.Tensor, stream=None) -> PlainW:
    m, n = W.shape
    out = C.c_void_p()
    _check(lib().nimbus_plain_weights(ctx.ptr, _ptr(W, torch.int32, "W"), m, n, _stream(stream), C.byref(out)), ctx)
    return PlainW(out, ctx, m, n)


def nimbus_server_workspace_size(ctx: Context, w: PlainW, k_per_query: int, n_queries: int) -> int:
    out = _sz()
    _check(lib().nimbus_server_workspace_size(ctx.ptr, w.ptr, k_per_query, n_queries, C.byref(out)), ctx)
    return int(out.value)


def nimbus_plain_matmul(ctx: Context, w: PlainW, X: torch.Tensor, add: torch.Tensor = None, Y=None, ws=None,
                        stream=None) -> torch.Tensor:
    k = X.shape[0]
    if Y is None:
        Y = torch.empty((k, w.n), dtype=torch.int32, device=X.device)
    if ws is None:
        ws = torch.empty(nimbus_server_workspace_size(ctx, w, k, 0), dtype=torch.uint8, device=X.device)
    _check(lib().nimbus_plain_matmul(ctx.ptr, w.ptr, _ptr(X, torch.int32, "X"), k,
                                     _ptr(add, torch.int32, "add") if add is not None else None,
                                     _ptr(Y, torch.int32, "Y"), _ptr(ws), ws.numel(), _stream(stream)), ctx)
    return Y


def nimbus_server_output(ctx: Context, sk: SecretKey, w: PlainW, Xs: torch.Tensor, cts: torch.Tensor,
                         k_per_query: int, n_queries: int, Ys=None, ws=None, stream=None) -> torch.Tensor:
    k = k_per_query * n_queries
    if Ys is None:
        Ys = torch.empty((k, w.n), dtype=torch.int32, device=Xs.device)
    if ws is None:
        ws = torch.empty(nimbus_server_workspace_size(ctx, w, k_per_query, n_queries), dtype=torch.uint8,
                         device=Xs.device)
    _check(lib().nimbus_server_output(ctx.ptr, sk.ptr, w.ptr, _ptr(Xs, torch.int32, "Xs"),
                                      _ptr(cts, torch.int32, "cts"), k_per_query, n_queries,
                                      _ptr(Ys, torch.int32, "Ys"), _ptr(ws), ws.numel(), _stream(stream)), ctx)
    return Ys


def nimbus_plain_weights_u64(ctx: Context, W: torch.Tensor, stream=None) -> PlainW:
    """ell > 32 (the paper's t = 2^64): W is an int64 tensor holding uint64 values."""
    m, n = W.shape
    out = C.c_void_p()
    _check(lib().nimbus_plain_weights_u64(ctx.ptr, _ptr(W, torch.int64, "W"), m, n, _stream(stream), C.byref(out)),
           ctx)
    return PlainW(out, ctx, m, n)


def nimbus_plain_matmul_u64(ctx: Context, w: PlainW, X: torch.Tensor, add: torch.Tensor = None, Y=None, ws=None,
                            stream=None) -> torch.Tensor:
    k = X.shape[0]
    if Y is None:
        Y = torch.empty((k, w.n), dtype=torch.int64, device=X.device)
    if ws is None:
        ws = torch.empty(nimbus_server_workspace_size(ctx, w, k, 0), dtype=torch.uint8, device=X.device)
    _check(lib().nimbus_plain_matmul_u64(ctx.ptr, w.ptr, _ptr(X, torch.int64, "X"), k,
                                         _ptr(add, torch.int64, "add") if add is not None else None,
                                         _ptr(Y, torch.int64, "Y"), _ptr(ws), ws.numel(), _stream(stream)), ctx)
    return Y


def nimbus_server_output_u64(ctx: Context, sk: SecretKey, w: PlainW, Xs: torch.Tensor, cts: torch.Tensor,
                             k_per_query: int, n_queries: int, Ys=None, ws=None, stream=None) -> torch.Tensor:
    k = k_per_query * n_queries
    if Ys is None:
        Ys = torch.empty((k, w.n), dtype=torch.int64, device=Xs.device)
    if ws is None:
        ws = torch.empty(nimbus_server_workspace_size(ctx, w, k_per_query, n_queries), dtype=torch.uint8,
                         device=Xs.device)
    _check(lib().nimbus_server_output_u64(ctx.ptr, sk.ptr, w.ptr, _ptr(Xs, torch.int64, "Xs"),
                                          _ptr(cts, torch.int32, "cts"), k_per_query, n_queries,
                                          _ptr(Ys, torch.int64, "Ys"), _ptr(ws), ws.numel(), _stream(stream)), ctx)
    return Ys


# ------------------------------------------------------------------ helpers
def as_u32(t: torch.Tensor) -> torch.Tensor:
    """View a uint32-valued int32 tensor as int64 with values in [0, 2^32)."""
    return t.to(torch.int64) & 0xFFFFFFFF


def from_numpy_u32(a, device) -> torch.Tensor:
    import numpy as np
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to(device)


def to_numpy_u32(t: torch.Tensor):
    import numpy as np
    return t.detach().cpu().contiguous().numpy().view(np.uint32)
