"""The CPU oracle pinned before it is trusted: against an independent pure-Python
restatement, the schoolbook product, the seeded integer fixtures, the reference's float
semantics (hesim clear_pcmm / pcmm_bsgs golden values, BASELINE config 1) and the
decryption identity of the RLWE -> MLWE decomposition."""

from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200.params import HeParams

GOLD = Path(__file__).parent / "golden"
P = HeParams.toy()


@pytest.fixture(scope="module")
def toy():
    rng = np.random.default_rng(0)
    n_in, n_out = 32, 48
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    Wt = O.encode_weights(P, W)
    return A, W, s, ct, Wt


def test_ntt_product_equals_schoolbook():
    rng = np.random.default_rng(1)
    for q in P.moduli:
        a = rng.integers(0, q, P.N).astype(np.uint32)
        s = rng.integers(-1, 2, P.N).astype(np.int32)
        assert np.array_equal(O.negacyclic_mul(a, s, q), O.negacyclic_mul_schoolbook(a, s, q))


def test_encrypt_decrypt_roundtrip(toy):
    A, W, s, ct, Wt = toy
    for limb in (0, 1):
        ph = O.decrypt_rlwe(P, ct, s, limb)
        if limb == 0:
            assert np.abs(O.decode_acts(P, ph, A.shape[1]) - A).max() < 2 ** -20


def test_imaginary_half_is_empty(toy):
    A, W, s, ct, Wt = toy
    ph = O.decrypt_rlwe(P, ct, s, 0)
    assert np.abs(ph[:, P.N // 2:]).max() < 64  # only the fresh noise


def test_c_oracle_equals_pure_python_restatement(toy):
    A, W, s, ct, Wt = toy
    rows = [0, 7, 16, 47]
    assert np.array_equal(O.pcmm(P, Wt, ct, rows=rows), O.py_pcmm_rows(P, Wt, ct, rows))


def test_mlwe_decomposition_decrypts_under_the_component_key(toy):
    """b_t + sum_j a~_{t,j} * s_j == (b + a s)_t for every component t."""
    A, W, s, ct, Wt = toy
    d, k, q = P.mlwe_degree, P.mlwe_rank, P.moduli[0]
    a = [int(v) for v in ct[0, 0, 0]]
    b = [int(v) for v in ct[0, 0, 1]]
    full = O.decrypt_rlwe(P, ct[:1], s, 0)[0] % q
    at = O.py_mlwe_components(P, a, q)
    for t in range(k):
        for m in range(d):
            acc = b[t + k * m]
            for j in range(k):
                for mp in range(d):
                    idx = m - mp
                    sv = s[j + k * idx] if idx >= 0 else -s[j + k * (idx + d)]
                    acc += at[t][j][mp] * int(sv)
            assert acc % q == full[t + k * m]


def test_pcmm_decrypts_to_float_product(toy):
    A, W, s, ct, Wt = toy
    out = O.pcmm(P, Wt, ct)
    ph = O.decrypt_mlwe(P, s, out)
    ref = O.clear_pcmm(W, A)
    vals = O.decode_mlwe_rows(P, ph, list(range(W.shape[0])))
    err = max(np.abs(v - ref[br, col]).max() for col, (br, v) in vals.items())
    assert err < 2 ** -14, err


def test_rescale_rule():
    q0, q1 = P.moduli
    inv = pow(q1, q0 - 2, q0)
    for x0, x1 in [(0, 0), (5, 1), (q0 - 1, q1 - 1), (123, q1 // 2), (123, q1 // 2 + 1), (q0 - 1, 0)]:
        x1c = x1 - q1 if x1 > q1 // 2 else x1
        assert O.rescale(P, x0, x1) == (x0 - x1c) * inv % q0


def test_seeded_integer_fixture():
    """Regression pin of the oracle's integer outputs (tests/golden/make_oracle_golden.py)."""
    g = np.load(GOLD / "oracle_toy_int.npz")
    s = O.keygen(P, 7)
    assert np.array_equal(s, g["s"])
    gt = np.load(GOLD / "pcmm_toy_golden.npz")
    A = gt["M"].T.copy()
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    assert np.array_equal(ct, g["ct"])
    Wt = O.encode_weights(P, gt["W"])
    assert np.array_equal(Wt, g["Wt"])
    assert np.array_equal(O.pcmm(P, Wt, ct), g["out"])


def test_baseline_config1_matches_hesim():
    """BASELINE config 1: the 16x16x16 toy PCMM decrypts to hesim's clear_pcmm and to
    hesim's own slot-domain pcmm_bsgs (golden values from the reference)."""
    g = np.load(GOLD / "oracle_toy_int.npz")
    gt = np.load(GOLD / "pcmm_toy_golden.npz")
    W, M = gt["W"], gt["M"]
    ph = O.decrypt_mlwe(P, g["s"], g["out"])
    vals = O.decode_mlwe_rows(P, ph, list(range(16)))
    got = np.zeros((16, 16))                      # tokens x n_out = (W @ M)^T
    for col, (br, v) in vals.items():
        got[br, col] = v
    np.testing.assert_allclose(got.T, gt["hesim_clear"], atol=2 ** -16)
    np.testing.assert_allclose(got.T, gt["hesim_bsgs"], atol=2 ** -16)
    np.testing.assert_array_equal(gt["pin_clear_2x2_power1"], [[1.0, 8.0], [6.0, 2.0]])
    assert int(gt["hesim_level_drop"]) == 1      # the reference kernel also consumes one level


def test_ring_pack_decrypts_to_product_in_activation_layout():
    """§8f1 oracle: PCMM at level 1 + PackLWEs over Z[X^k] + rescale gives level-0 RLWE blocks whose
    decryption, decoded in the INPUT activation layout, is A @ W^T; and BASELINE config 1's toy
    product packs to hesim's golden values."""
    rng = np.random.default_rng(3)
    n_out, n_in = 32, 48
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    gal = O.ring_pack_keys(P, 5, s)
    out = O.pcmm_ring_pack(P, O.encode_weights(P, W), ct, gal)
    assert out.shape == (n_out // P.mlwe_rank, 2, P.N)
    ph = np.stack([O.decrypt_under(P, out[b, 0], out[b, 1], s, P.moduli[0]) for b in range(out.shape[0])])
    dec = O.decode_acts(P, ph, n_out)
    ref = A @ W.T
    assert np.abs(dec - ref).max() < np.abs(ref).max() * 2.0 ** -14
    gt = np.load(GOLD / "pcmm_toy_golden.npz")
    ct = O.encrypt(P, 11, s, O.encode_acts(P, gt["M"].T.copy()))
    out = O.pcmm_ring_pack(P, O.encode_weights(P, gt["W"]), ct, gal)
    ph = O.decrypt_under(P, out[0, 0], out[0, 1], s, P.moduli[0])[None]
    np.testing.assert_allclose(O.decode_acts(P, ph, 16).T, gt["hesim_clear"], atol=2 ** -14)


def test_ring_pack_leaves_trace_keeps_component_zero():
    """The leaf construction: component 0 of C_y's phase (A_y s + B_y, scaled back by k) is the MLWE
    row's phase -- the identity the subring trace relies on."""
    rng = np.random.default_rng(4)
    n_out, n_in = 16, 32
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    Wt = O.encode_weights(P, W)
    raw = [O.pcmm_limb(P, Wt, ct, L) for L in range(2)]
    leaves = O.ring_pack_leaves(P, raw)
    d, k, q = P.mlwe_degree, P.mlwe_rank, int(P.moduli[0])
    for y in (0, 5, 15):
        ph = O.decrypt_under(P, leaves[y, 0, 0], leaves[y, 0, 1], s, q)[::k] * k % q
        row = np.concatenate([raw[0][y]])[None]
        # MLWE phase of row y at level 1, limb 0 (decrypt_mlwe takes level-0 words; compare mod q0)
        ref = O.decrypt_mlwe(P, s, row)[0] % q
        assert np.array_equal(ph % q, ref)


def test_mlwe_keyswitch_packing_matches_trace_packing_plaintext():
    """The two packings (MLWE -> RLWE key switch; subring PackLWEs) give ciphertexts of the same
    plaintext: decryptions agree to the key-switching noise and decode to A @ W^T."""
    rng = np.random.default_rng(6)
    n_out, n_in = 32, 32
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    raw = [O.pcmm_limb(P, O.encode_weights(P, W), ct, L) for L in range(2)]
    ks = O.mlwe_to_rlwe(P, *O.raw_device_layout(P, raw), O.mlwe_ks_keys(P, 5, s))
    tr = O.ring_pack(P, O.ring_pack_leaves(P, raw), O.ring_pack_keys(P, 5, s))[1]
    q = P.moduli[0]
    ph_ks = np.stack([O.decrypt_under(P, ks[b, 0], ks[b, 1], s, q) for b in range(ks.shape[0])])
    ph_tr = np.stack([O.decrypt_under(P, tr[b, 0], tr[b, 1], s, q) for b in range(tr.shape[0])])
    assert np.abs(ph_ks - ph_tr).max() < 64
    ref = A @ W.T
    assert np.abs(O.decode_acts(P, ph_ks, n_out) - ref).max() < np.abs(ref).max() * 2.0 ** -14


def test_oracle_one_digit_ring_packing_decrypts():
    """or_mlwe_to_rlwe1 (one digit, special modulus P1 P2) packs the toy PCMM output to the same plaintext as the
    two-digit or_mlwe_to_rlwe (both decrypt to A W^T within 2^-16)."""
    P = HeParams.toy()
    rng = np.random.default_rng(1)
    n_out, n_in = 32, 48
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    raw = [O.pcmm_limb(P, O.encode_weights(P, W), ct, L) for L in range(2)]
    rb, ra = O.raw_device_layout(P, raw)
    assert O.ring_pack_special2(P) not in (*P.moduli, P.special_prime)
    for out in (O.mlwe_to_rlwe1(P, rb, ra, O.mlwe_ks_keys1(P, 5, s)), O.mlwe_to_rlwe(P, rb, ra, O.mlwe_ks_keys(P, 5, s))):
        dec = O.decode_acts(P, O.decrypt_rlwe(P, out[:, None], s), n_out)
        assert np.abs(dec - A @ W.T).max() < 2 ** -16


@pytest.mark.parametrize("L", [32, 64, 128])
def test_spectral_restatement_equals_direct_every_word(toy, L):
    """he_oracle_spectral.c (overlap-save correlations, any L > k) == or_pcmm (BCHPS24 Alg. 2) on every word,
    including row slices, and both equal the seeded golden output."""
    A, W, s, ct, Wt = toy
    ref = O.pcmm(P, Wt, ct)
    assert np.array_equal(O.pcmm_spectral(P, Wt, ct, L=L), ref)
    assert np.array_equal(O.pcmm_spectral(P, Wt, ct, row0=5, n_rows=17, L=L), ref[5:22])
    g = np.load(GOLD / "oracle_toy_int.npz")
    gt = np.load(GOLD / "pcmm_toy_golden.npz")
    ct2 = O.encrypt(P, 11, O.keygen(P, 7), O.encode_acts(P, gt["M"].T.copy()))
    assert np.array_equal(O.pcmm_spectral(P, O.encode_weights(P, gt["W"]), ct2, L=L), g["out"])


def test_spectral_restatement_equals_direct_llama_ring():
    """At the Llama ring (N = 2^16, MLWE (256, 256), L = 1024): 6 output rows x all 65 792 columns, 2 input
    ciphertexts, every word equal to the direct oracle."""
    PL = HeParams.llama()
    rng = np.random.default_rng(3)
    n_in, n_out = 2 * PL.mlwe_rank, 6
    A = rng.uniform(-1, 1, (PL.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    ct = O.encrypt(PL, 11, O.keygen(PL, 7), O.encode_acts(PL, A))
    Wt = O.encode_weights(PL, W)
    assert np.array_equal(O.pcmm_spectral(PL, Wt, ct), O.pcmm(PL, Wt, ct))
