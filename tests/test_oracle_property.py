"""Property-based pins of the oracle's end-to-end identity (hypothesis): for
random small parameter sets that satisfy the worst-case noise bound (SURVEY.md
§8(c)), Dec(COP(X, Enc(W))) unpacks to (X.W - R) mod t by Python-integer brute
force, the invalid slots decrypt to -r, R is the mask at the
valid slots, the measured noise stays under the analytic bound, and the
re-randomised output (reading 26) decrypts to the same shares.
CPU only; sizes keep each example well under a second."""
import numpy as np
import pytest
from hypothesis import HealthCheck, assume, given, settings
from hypothesis import strategies as st

import nimbus_inputs as ni
from test_oracle_pins import _check_e2e, noise_bound_after_moddown, py_matmul_mod
from test_oracle_rerand import max_flood_bits


@st.composite
def params(draw):
    N = draw(st.sampled_from([16, 32, 64, 128]))
    L = draw(st.integers(1, 3))
    L_out = draw(st.integers(1, L))
    ell = draw(st.sampled_from([4, 8, 12, 16, 24, 32]))
    m = draw(st.integers(1, 24))
    n = draw(st.integers(1, N))
    kq = draw(st.integers(1, 20))
    nq = draw(st.integers(1, 3))
    seed = draw(st.integers(0, 2**32 - 1))
    return N, L, L_out, ell, m, n, kq, nq, seed


@settings(max_examples=120, deadline=None, suppress_health_check=[HealthCheck.filter_too_much])
@given(params())
def test_e2e_identity_random_params(oracle, p):
    N, L, L_out, ell, m, n, kq, nq, seed = p
    pr = [int(x) for x in oracle.primes(N, L)]
    t = 1 << ell
    R_eff = min(N // n, kq)
    q_out = 1
    for x in pr[:L_out]:
        q_out *= x
    q = 1
    for x in pr:
        q *= x
    # worst case before and after the mod-switch (SURVEY.md §8(c) "Worst-case noise guarantee")
    assume(R_eff * m * (t - 1) * 21.5 < q / (2 * t) - 1)
    assume(noise_bound_after_moddown(N, pr, ell, L_out, m, R_eff) < q_out / (2 * t))
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, m, n, ell)
    X = ni.gen_X(seed ^ 1, kq * nq, m, ell)
    E = oracle.encrypt_rows(N, L, np.array(pr, np.uint32), ell, s, W, seed)
    cts, R = oracle.cop_matmul(N, L, L_out, np.array(pr, np.uint32), ell, E, X, n, kq, nq, seed)
    d = dict(s=s, W=W, X=X, cts=cts, R=R, seed=seed)
    v = _check_e2e(oracle, d, N, pr, ell, L_out, kq, n, nq)
    assert v <= noise_bound_after_moddown(N, pr, ell, L_out, m, R_eff)
    # circuit privacy leaves the shares unchanged
    F = max_flood_bits(N, pr, ell, L_out, m, R_eff)
    pk = oracle.keygen_pk(N, L, np.array(pr, np.uint32), s, seed ^ 2)
    z = oracle.rerand_zero(N, L, np.array(pr, np.uint32), pk, seed ^ 3, cts.shape[0] * cts.shape[1], F)
    cts2, R2 = oracle.cop_matmul_rr(N, L, L_out, np.array(pr, np.uint32), ell, E, X, n, kq, nq, seed, z)
    Z2, _, _ = oracle.decrypt_unpack(N, L_out, np.array(pr[:L_out], np.uint32), ell, s, cts2, kq, nq, n)
    Y = py_matmul_mod(X, W, t)
    assert (R2 == R).all()
    assert (Z2.astype(np.uint64) == (Y + np.uint64(t) - R.astype(np.uint64)) % np.uint64(t)).all()
