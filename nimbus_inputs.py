"""Seeded synthetic inputs and workload table shared by the tests, the bench and
the oracle harness.

This module holds NO arithmetic of the method (no encryption, no contraction,
no packing).  It only
  * names the five workloads of BASELINE.json (C1..C5) and their parameters,
  * derives the per-config / per-matrix seeds (SURVEY.md App. B "Seeds"),
  * draws the client share X and the server weights W from the counter-based
    SplitMix64 stream (SURVEY.md App. B "PRG", domains 4 and 5), uniform in
    Z_t = [0, 2^ell) (§2.1 notation; §2.3 shares are
    uniform).

The oracle (oracle/) and the CUDA library each implement the same PRG
contract independently; this module is the third, numpy, implementation, used
only to produce X and W, which both sides then receive as inputs.
"""
from __future__ import annotations

import dataclasses
import numpy as np

GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1

DOM_SK, DOM_A, DOM_E, DOM_X, DOM_W, DOM_MASK = 1, 2, 3, 4, 5, 6


def _mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= np.uint64(_M1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(_M2)
    z ^= z >> np.uint64(31)
    return z


def _mix64_int(z: int) -> int:
    z &= _MASK64
    z ^= z >> 30
    z = (z * _M1) & _MASK64
    z ^= z >> 27
    z = (z * _M2) & _MASK64
    z ^= z >> 31
    return z


def prg_words(seed: int, dom: int, start: int, count: int) -> np.ndarray:
    """word(seed, dom, i) = mix64(mix64(seed ^ (dom<<56)) + GAMMA*(i+1)) for
    i in [start, start+count), all arithmetic mod 2^64."""
    key = _mix64_int((seed ^ (dom << 56)) & _MASK64)
    i = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + np.uint64(GAMMA) * (i + np.uint64(1))
    return _mix64_np(z)


def uniform_mod_t(seed: int, dom: int, count: int, ell: int, start: int = 0) -> np.ndarray:
    """uniform in Z_t, t = 2^ell: word >> (64 - ell); uint32 for ell <= 32, uint64 beyond."""
    w = prg_words(seed, dom, start, count)
    return (w >> np.uint64(64 - ell)).astype(np.uint32 if ell <= 32 else np.uint64)


@dataclasses.dataclass(frozen=True)
class Layer:
    """One COP matmul: X (k x m) . W (m x n)  (Alg. 1 inputs)."""
    name: str
    k_per_query: int
    n_queries: int
    m: int
    n: int

    @property
    def k(self) -> int:
        return self.k_per_query * self.n_queries


@dataclasses.dataclass(frozen=True)
class Config:
    """RLWE parameters + workload.  N ring degree, L limbs of 31-bit NTT primes,
    ell plaintext bits (t = 2^ell), L_out limbs after the mod-switch.  shared_x: every
    matmul of the step multiplies the SAME client share X (Q, K, V of one layer)."""
    cid: int
    name: str
    N: int
    L: int
    ell: int
    L_out: int
    layers: tuple  # tuple[(layer_idx, proj, Layer)]
    shared_x: bool = False

    @property
    def seed_cfg(self) -> int:
        return seed_cfg(self.cid)


def seed_cfg(cid: int) -> int:
    """SURVEY.md §8(d) 'Seeds': 0x4E494D4255530000 ^ (cfg << 32)."""
    return (0x4E494D4255530000 ^ (cid << 32)) & _MASK64


def seed_mm(cid: int, layer: int = 0, proj: int = 0) -> int:
    """seed_cfg ^ (layer<<16) ^ (proj<<8); proj 0..5 = Q,K,V,O,FFN-up,FFN-down."""
    return (seed_cfg(cid) ^ (layer << 16) ^ (proj << 8)) & _MASK64


_PROJ = ("Q", "K", "V", "O", "up", "down")


def _bert_layer_stack(layers: int, seq: int, batch: int):
    out = []
    for li in range(layers):
        for proj in range(6):
            m, n = (768, 768) if proj < 4 else ((768, 3072) if proj == 4 else (3072, 768))
            out.append((li, proj, Layer(f"L{li}.{_PROJ[proj]}", seq, batch, m, n)))
    return tuple(out)


def _single(name, k, m, n):
    return ((0, 0, Layer(name, k, 1, m, n)),)


# BASELINE.json "configs", in order (C1..C5).  ell / L_out per SURVEY.md §8(c) #2, #14.
CONFIGS = {
    1: Config(1, "C1", 4096, 2, 16, 1, _single("C1", 16, 64, 64)),
    2: Config(2, "C2", 4096, 2, 16, 1, _single("attn_proj", 128, 768, 768)),
    3: Config(3, "C3", 4096, 2, 16, 1, _single("ffn_up", 128, 768, 3072)),
    4: Config(4, "C4", 8192, 3, 32, 2, _single("ffn_down", 128, 3072, 768)),
    5: Config(5, "C5", 8192, 3, 32, 2, _bert_layer_stack(12, 512, 4)),
}
# The three same-X attention projections of one layer at C2's shape (Q, K, V: X 128x768 . W 768x768
# each), one batched call per step -- the k = 128 stream as the model issues it.
CONFIG_QKV = Config(2, "C2-QKV", 4096, 2, 16, 1,
                    tuple((0, p, Layer(f"L0.{_PROJ[p]}", 128, 1, 768, 768)) for p in range(3)), shared_x=True)

# Secondary lines named by SURVEY.md §8(d): C4/C5 at ell=16 (L_out=1).
CONFIGS_L16 = {
    4: dataclasses.replace(CONFIGS[4], ell=16, L_out=1, name="C4@l16"),
    5: dataclasses.replace(CONFIGS[5], ell=16, L_out=1, name="C5@l16"),
}


# The paper's own t (ell = 64): q = 5 x 31-bit primes,
# 3-limb output (the noise bound at m = 3072, R = 10 needs q > 2^148 and q' > 2^86).
CONFIGS_L64 = {
    4: dataclasses.replace(CONFIGS[4], L=5, ell=64, L_out=3, name="C4@l64"),
    5: dataclasses.replace(CONFIGS[5], L=5, ell=64, L_out=3, name="C5@l64"),
}


def gen_X(seed: int, k: int, m: int, ell: int) -> np.ndarray:
    """Client share X, k x m, uniform in Z_t; domain 4, index alpha*m + beta."""
    return uniform_mod_t(seed, DOM_X, k * m, ell).reshape(k, m)


def gen_W(seed: int, m: int, n: int, ell: int) -> np.ndarray:
    """Server weights W, m x n, uniform in Z_t; domain 5, index beta*n + j."""
    return uniform_mod_t(seed, DOM_W, m * n, ell).reshape(m, n)


def modmacs(k: int, m: int, N: int, L: int) -> int:
    """Algorithmic work of one COP matmul: k*m*2*L*N modular MACs
    (App. D, O(kmN) per component and limb)."""
    return k * m * 2 * L * N
