"""Slot-domain τ-PCMM on CPU: the CKKS slot encoder, and the integer oracle
(or_slot_pcmm: hoisted BSGS rotations + key switching on real ciphertexts) decrypting to the
reference's own pcmm_bsgs values (golden file from hesim, tests/golden/make_slot_pcmm_golden.py)."""
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200 import slots
from paper_2601_18511_b200.params import HeParams
from paper_2601_18511_b200.slotpcmm import (BsgsSplit, SlotPcmmPlan, clear_slot_pcmm, col_shear, default_split,
                                            encode_blocks, shift_rows)

GOLD = Path(__file__).parent / "golden"
P = HeParams.toy()


def test_encoder_round_trip_rotation_and_product():
    rng = np.random.default_rng(0)
    N = P.N
    z = rng.uniform(-1, 1, N // 2)
    m = slots.encode(z, N, P.delta)
    assert np.abs(slots.decode(m, N, P.delta) - z).max() < 1e-6
    g = slots.rotation_galois(N, 5)
    mr = np.zeros(N, np.int64)
    for i in range(N):
        j = i * g % (2 * N)
        mr[j if j < N else j - N] += m[i] if j < N else -m[i]
    assert np.abs(slots.decode(mr, N, P.delta) - np.roll(z, -5)).max() < 1e-6
    w = rng.uniform(-1, 1, N // 2)
    q = P.moduli[0]
    m16 = slots.encode(z, N, 2.0 ** 16)   # product scale 2^28 < q0 / 2
    prod = O.negacyclic_mul((m16 % q).astype(np.uint32), slots.encode(w, N, 2.0 ** 12).astype(np.int32), q)
    prod = np.where(prod > q // 2, prod.astype(np.int64) - q, prod.astype(np.int64))
    assert np.abs(slots.decode(prod, N, 2.0 ** 28) - z * w).max() < 1e-2


def _oracle_run(W, B, shear, split=None):
    d = W.shape[0]
    split = split or default_split(d)
    plan = SlotPcmmPlan(d, shear, split, col_shear(shift_rows(W), shear))
    pt = encode_blocks(P, plan)
    pts = np.stack([np.stack([(pt[k] % q).astype(np.uint32) for q in P.moduli]) for k in range(d)])
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, slots.encode(col_shear(B, shear + 1).reshape(-1), P.N, P.delta)[None])[0]
    b, g = split.baby, split.giant
    kb = O.rotation_keys(P, 13, s, [i * d for i in range(1, b)])
    kg = O.rotation_keys(P, 13, s, [j * b * d for j in range(1, g)])
    out = O.slot_pcmm(P, ct, pts, d, b, g, kb, kg)
    ph = O.decrypt_under(P, out[0], out[1], s, P.moduli[0])
    return slots.decode(ph, P.N, P.delta, d * d).reshape(d, d)


@pytest.mark.parametrize("key", ["d16_l0", "d16_l2", "d8_l1"])
def test_oracle_decrypts_to_hesim_pcmm_bsgs(key):
    g = np.load(GOLD / "slot_pcmm_golden.npz")
    W, B, ref = g[key + "_W"], g[key + "_B"], g[key + "_hesim_bsgs"]
    shear = int(key.split("_l")[1])
    split = BsgsSplit(*(int(v) for v in g[key + "_split"]))
    got = _oracle_run(W, B, shear, split)
    np.testing.assert_allclose(ref, clear_slot_pcmm(W, B, shear), atol=1e-12)
    assert np.abs(got - ref).max() < 2.0 ** -13
