"""The Cooley-Tukey factorization of SlotToCoeffs (chain.py) and the chain oracle, on the CPU:
the grouped butterfly maps compose to the dense map M of stc.py, and three oracle BSGS maps on a level-4
toy ciphertext decrypt to the App. A coefficient layout the PCMM consumes."""
import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200 import HeParams, slots
from paper_2601_18511_b200.chain import apply_diagonals, bsgs_shape, special_fft_layers, stc_factors
from paper_2601_18511_b200.stc import slot_of_coeff, slot_vectors


def dense_apply(N, z):
    """M z: the slots of sum_s z_s X^(bitReverse(s)) (complex coefficients), evaluated directly."""
    e = slots.slot_exponents(N)
    c = np.argsort(slot_of_coeff(N))
    zeta = np.exp(1j * np.pi / N)
    return np.array([np.sum(z * zeta ** ((ej * c) % (2 * N))) for ej in e])


@pytest.mark.parametrize("N", [64, 512, 2048])
def test_layers_compose_to_the_dense_map(N):
    z = np.random.default_rng(N).standard_normal(N // 2) + 1j * np.random.default_rng(N + 1).standard_normal(N // 2)
    v = z.copy()
    for L in special_fft_layers(N):
        assert len(L) <= 3
        v = apply_diagonals(L, v)
    assert np.abs(v - dense_apply(N, z)).max() < 1e-9 * N


@pytest.mark.parametrize("N,levels", [(512, 3), (4096, 3), (65536, 3), (4096, 2)])
def test_grouped_maps(N, levels):
    n = N // 2
    fs = stc_factors(N, levels)
    z = np.random.default_rng(1).standard_normal(n) + 0j
    v = z.copy()
    for f in fs:
        assert len(f["diags"]) <= f["count"]
        span = n // f["stride"]
        for o in f["diags"]:
            assert o % f["stride"] == 0
            t = o // f["stride"]
            assert min(t, span - t) <= f["T"] or f["T"] == 0     # offsets within +-T strides (or wrapped)
        assert max(np.abs(d).max() for d in f["diags"].values()) <= 1 + 1e-12
        v = apply_diagonals(f["diags"], v)
    # reference: the slots of the coefficient-encoded polynomial (slots.decode of sum_s z_s X^(c(s)))
    m = np.zeros(N)
    m[np.argsort(slot_of_coeff(N))] = z.real
    ref = slots.decode(m, N, 1.0, real=False)
    assert np.abs(v - ref).max() < 1e-8 * np.sqrt(N)
    if N == 65536:
        assert [f["count"] for f in fs] == [63, 63, 32]
        assert [bsgs_shape(f["count"]) for f in fs] == [(16, 4), (16, 4), (16, 2)]


def test_oracle_factorized_stc_toy():
    """Three oracle chain maps (levels 4 -> 1) on a slot-encoded toy activation block: the result decrypts to
    the coefficient encoding `encrypt_acts` produces (the PCMM's input)."""
    from paper_2601_18511_b200.chain import stc_factors

    P = HeParams.toy_chain()
    N, n, k = P.N, P.N // 2, P.mlwe_rank
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (P.tokens, k))
    s = O.keygen(P, 7)
    shift = 10
    z = slot_vectors(P, A)[0]
    ct = O.encrypt(P, 13, s, slots.encode(z, N, P.delta * 2 ** (3 * shift))[None], level=4)[0]
    lvl = 4
    for kk, f in enumerate(stc_factors(N, 3)):
        b, g = bsgs_shape(f["count"])
        st, T = f["stride"], f["T"]
        scale = P.moduli[lvl] / 2 ** shift
        pts = np.zeros((b * g, lvl + 1, N), np.uint32)
        for j in range(g):
            for i in range(b):
                t = i + j * b
                d = f["diags"].get(((t - T) * st) % n) if t < f["count"] else None
                if d is not None:
                    m = slots.encode(np.roll(d, (j * b - T) * st), N, scale)
                    pts[t] = np.stack([(m % q).astype(np.uint32) for q in P.moduli[:lvl + 1]])
        kb = O.chain_rotation_keys(P, 21 + kk, s, [i * st for i in range(1, b)], lvl)
        kg = O.chain_rotation_keys(P, 21 + kk, s, [(j * b - T) * st for j in range(g)], lvl)
        ct = O.chain_bsgs(P, ct, pts, lvl, b, g, st, T, kb, kg)
        lvl -= 1
    assert ct.shape == (2, 2, N)
    ph = O.decrypt_rlwe(P, ct[None], s)[0]
    want = O.encode_acts(P, A)[0]
    err = np.abs(ph - want).max() / P.delta
    assert err < 2 ** -14, err


@pytest.mark.parametrize("N,levels", [(512, 3), (4096, 3), (65536, 3), (4096, 2)])
def test_cts_maps_invert_the_stc_maps(N, levels):
    """CoeffToSlots (cts_factors) = M^-1: applied to the slots of a real polynomial m it returns the coefficient
    pairs z_s = m_(c(s)) + i m_(N/2 + c(s)), c = bitReverse -- the first half of the Half-Bootstrap."""
    from paper_2601_18511_b200.chain import cts_factors

    n = N // 2
    m = np.random.default_rng(3).standard_normal(N)
    w = slots.decode(m, N, 1.0, real=False)
    fs = cts_factors(N, levels)
    assert [(f["stride"], f["T"], f["count"]) for f in fs] == [(f["stride"], f["T"], f["count"])
                                                            for f in stc_factors(N, levels)][::-1]
    v = w.copy()
    for f in fs:
        assert max(np.abs(d).max() for d in f["diags"].values()) <= 1 + 1e-12
        v = apply_diagonals(f["diags"], v)
    c = np.argsort(slot_of_coeff(N))           # c[s] = bitReverse(s)
    want = m[c] + 1j * m[n + c]
    assert np.abs(v - want).max() < 1e-9 * np.sqrt(N)
