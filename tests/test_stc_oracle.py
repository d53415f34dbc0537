"""SlotToCoeffs on the CPU: the slot layout of PAPER.md:656, the fused bit-reversal of
PAPER.md:661, the BSGS plaintexts, and the integer oracle (or_slot_bsgs, stride 1) decrypting to the App. A
coefficient encoding (or_encode_acts) of the same activations."""
import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200 import HeParams, slots
from paper_2601_18511_b200.layout import bit_reverse, rotate_bits_down
from paper_2601_18511_b200.stc import slot_of_coeff, slot_vectors, stc_plaintexts, stc_split

P = HeParams.toy()


def test_slot_layout_is_the_papers():
    """ct_s[i + (d/2) j] = A[i][k r + f(j, log k)], and slot bitReverse(c) carries the value
    the App. A coefficient encoding puts at c."""
    rng = np.random.default_rng(1)
    d, k = P.mlwe_degree, P.mlwe_rank
    A = rng.uniform(-1, 1, (d // 2, 2 * k))
    z = slot_vectors(P, A)
    lk, half = k.bit_length() - 1, d // 2
    for r in range(2):
        for i in range(half):
            for j in range(k):
                assert z[r, i + half * j] == A[i, k * r + rotate_bits_down(j, lk)]
    pt = O.encode_acts(P, A)
    rev = slot_of_coeff(P.N)
    n = P.N // 2
    assert np.array_equal(np.rint(z[:, rev] * P.delta).astype(np.int64), pt[:, :n])
    assert not pt[:, n:].any()
    assert all(rev[c] == bit_reverse(c, n.bit_length() - 1) for c in range(n))


def test_plaintexts_are_the_rotated_diagonals():
    """pt_(i,j)[s] = M[s - j b][s + i] with M[j][s] = zeta^(e_j bitReverse(s)) (decoded at scale q1)."""
    N, n = P.N, P.N // 2
    split = stc_split(n)
    b = split.baby
    assert split.baby * split.giant == n and split.baby >= split.giant
    e = slots.slot_exponents(N)
    c = slot_of_coeff(N)
    M = np.exp(1j * np.pi / N * ((e[:, None] * c[None, :]) % (2 * N)))
    for k0 in (0, 37, n - 3):
        pts = stc_plaintexts(P, split, k0, 3).numpy()
        for t in range(3):
            k = k0 + t
            i, j = k % b, k // b
            s = np.arange(n)
            want = M[(s - j * b) % n, (s + i) % n]
            got = slots.decode(pts[t], N, float(P.delta_w), real=False)
            assert np.abs(got - want).max() < 1e-3


@pytest.mark.parametrize("lazy,plain", [(False, False), (True, False), (True, True)])
def test_oracle_stc_decrypts_to_app_a_coefficients(lazy, plain):
    """Both BSGS forms (per-rotation ModDown; lazy ModDown in the PQ basis, plaintexts also mod P), the lazy
    one also with plain dnum-2 giant keys."""
    rng = np.random.default_rng(2)
    d, k = P.mlwe_degree, P.mlwe_rank
    N, n = P.N, P.N // 2
    A = rng.uniform(-1, 1, (d // 2, k))
    split = stc_split(n)
    b, g = split.baby, split.giant
    pt = stc_plaintexts(P, split, 0, n).numpy()
    mods = P.ks_moduli if lazy else P.moduli
    pts = np.stack([np.stack([(pt[t] % q).astype(np.uint32) for q in mods]) for t in range(n)])
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, slots.encode(slot_vectors(P, A)[0], N, P.delta)[None])[0]
    kb = O.rotation_keys(P, 13, s, list(range(1, b)))
    kg = (O.rotation_keys_plain if plain else O.rotation_keys)(P, 13, s, [j * b for j in range(1, g)])
    out = O.slot_bsgs(P, ct, pts, 1, b, g, kb, kg, lazy=lazy)
    ph = O.decrypt_under(P, out[0], out[1], s, P.moduli[0])
    want = O.encode_acts(P, A)[0]
    err = np.abs(ph - want)
    assert err[:n].max() < P.delta * 2.0 ** -12          # the activations, 12+ bits
    assert err[n:].max() < P.delta * 2.0 ** -12          # imaginary half: noise only
    np.testing.assert_allclose(O.decode_acts(P, ph[None], k), A, atol=2.0 ** -12)
    with pytest.raises(ValueError):
        O.slot_bsgs(P, ct, pts, 2, b, g, kb, kg, lazy=lazy)   # 2 b g > N/2


def test_llama_ring_layout_matches_paper_numbers():
    """At the paper's sizes (N = 2^16, 128 x 256 per ct): ct_s[i + 128 j] = A[i][f(j, 8)] and
    slot bitReverse(c, 15) lands at coefficient c = t + 256 m <-> A[bitReverse(m, 7)][sigma(t)]."""
    from paper_2601_18511_b200.layout import sigma_table

    L = HeParams()
    assert (L.N, L.mlwe_degree, L.mlwe_rank) == (65536, 256, 256)
    rng = np.random.default_rng(9)
    A = rng.standard_normal((128, 512))
    z = slot_vectors(L, A)
    i = rng.integers(0, 128, 64)
    j = rng.integers(0, 256, 64)
    for r in range(2):
        assert np.array_equal(z[r, i + 128 * j], A[i, 256 * r + np.array([rotate_bits_down(int(v), 8) for v in j])])
    c = rng.integers(0, 32768, 64)
    t, m = c % 256, c // 256
    sig = sigma_table(256)
    s = np.array([bit_reverse(int(v), 15) for v in c])
    want = A[[bit_reverse(int(v), 7) for v in m], sig[t]]
    assert np.array_equal(z[0, s], want)


def test_split_and_shape_errors():
    assert (stc_split(32768).baby, stc_split(32768).giant) == (256, 128)
    assert (stc_split(256).baby, stc_split(256).giant) == (16, 16)
    with pytest.raises(ValueError):
        slot_vectors(P, np.zeros((P.mlwe_degree // 2 + 1, P.mlwe_rank)))
    with pytest.raises(ValueError):
        slot_vectors(P, np.zeros((P.mlwe_degree // 2, P.mlwe_rank + 1)))
