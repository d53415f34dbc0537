"""App. A index maps against the reference's own behaviour (golden tables generated from
hesim.bitrev by tests/golden/make_golden.py) and the anchors of pkg/tests/test_bitrev.py."""

from pathlib import Path

import numpy as np
import pytest

from paper_2601_18511_b200 import layout as L

G = np.load(Path(__file__).parent / "golden" / "bitrev_golden.npz")


@pytest.mark.parametrize("k", [3, 7, 8, 11])
def test_bit_reverse_matches_reference_table(k):
    assert [L.bit_reverse(x, k) for x in range(1 << k)] == G[f"bit_reverse_{k}"].tolist()
    assert np.array_equal(L.bit_reverse_table(k), G[f"bit_reverse_{k}"])


def test_rotate_bits_down_matches_reference():
    assert [L.rotate_bits_down(x, 8) for x in range(256)] == G["rotate_bits_down_8"].tolist()


def test_byte_mix_matches_reference():
    assert [L.byte_mix(x) for x in range(256)] == G["byte_mix"].tolist()


def test_half_reverse_matches_reference():
    assert [L.half_reverse(x) for x in range(4096)] == G["half_reverse"].tolist()


def test_shuffle_matrix_matches_reference():
    assert np.array_equal(L.shuffle_matrix(G["shuffle_input"]), G["shuffle_output"])


def test_reference_check_all_passed_when_fixtures_were_made():
    assert all(G["check_all_values"]), dict(zip(G["check_all_names"], G["check_all_values"]))


# anchors of pkg/tests/test_bitrev.py:12-87
def test_anchor_values():
    assert L.bit_reverse(1, 3) == 4 and L.bit_reverse(1, 8) == 128 and L.bit_reverse(6, 3) == 3
    assert L.rotate_bits_down(1, 8) == 128 and L.rotate_bits_down(3, 8) == 129
    assert L.byte_mix(1) == 4 and L.byte_mix(4) == 1 and L.byte_mix(0) == 0 and L.byte_mix(255) == 255
    assert L.half_reverse(1) == 1024 and L.half_reverse(2048) == 2048


def test_error_contract_matches_reference():
    for fn, args in ((L.bit_reverse, (8, 3)), (L.bit_reverse, (-1, 3)), (L.byte_mix, (256,)),
                     (L.half_reverse, (4096,)), (L.rotate_bits_down, (256, 8))):
        with pytest.raises(ValueError):
            fn(*args)
    with pytest.raises(ValueError):
        L.shuffle_matrix(np.ones((2, 3)))
    with pytest.raises(ValueError):
        L.shuffle_matrix(np.ones((16, 16)))  # byte_mix needs 256 rows


def test_nibble_identity_width_8():
    # byte_mix(16i + j) == f(bitReverse(i + 16 j, 8), 8): the width-8 reading of PAPER.md:663
    for i in range(16):
        for j in range(16):
            assert L.byte_mix(16 * i + j) == L.rotate_bits_down(L.bit_reverse(i + 16 * j, 8), 8)


def test_sigma_is_g_after_nibble_swap():
    sig = L.sigma_table(256)
    for t in range(256):
        assert sig[t] == L.byte_mix(L.nibble_swap(t))
    assert sorted(sig) == list(range(256))


def test_block_conjugation_is_papers_g_shuffle_in_component_order():
    """The plan's block conjugation by sigma equals hesim.shuffle_matrix(B, g) reindexed by
    the nibble swap between MLWE index x and component t."""
    B = G["shuffle_input"]
    perm = L.block_permutation(256, 256)
    ours = B[np.ix_(perm, perm)]                 # rows/cols in component order
    swap = np.array([L.nibble_swap(t) for t in range(256)])
    paper = G["shuffle_output"]                  # B'[x][x'] = B[g(x)][g(x')], MLWE-index order
    assert np.array_equal(ours, paper[np.ix_(swap, swap)])


def test_coeff_table_covers_each_block_entry_once():
    for d, k in ((32, 16), (256, 256)):
        token, col = L.coeff_table(d, k)
        live = token >= 0
        assert live.sum() == (d // 2) * k
        pairs = set(zip(token[live].tolist(), col[live].tolist()))
        assert len(pairs) == (d // 2) * k


def test_coeff_layout_is_bitreversed_slot_layout():
    """ct_c[c] = ct_s[bitReverse(c, 15)] and ct_s[i + 128 j] = A[i][f(j, 8)]."""
    d = k = 256
    token, col = L.coeff_table(d, k)
    for c in [0, 1, 255, 256, 257, 4097, 32767]:
        s = L.bit_reverse(c, 15)
        i, j = s % 128, s // 128
        assert token[c] == i and col[c] == L.rotate_bits_down(j, 8)
