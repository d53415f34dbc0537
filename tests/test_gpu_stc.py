"""SlotToCoeffs on the GPU: bit-exact against the integer oracle (or_slot_bsgs, stride 1)
at toy size, decrypting to the App. A coefficient layout the MLWE PCMM consumes (decrypt_acts), the ledger
and error contract; at N = 2^16 (32 768 slots, 256 x 128 BSGS) the decryption matches the activations."""
import time

import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200 import HeContext, HeParams, slots
from paper_2601_18511_b200.errors import NeedsBootstrapError
from paper_2601_18511_b200.pcmm import make_mlwe_pcmm_plan, pcmm_mlwe
from paper_2601_18511_b200.slotpcmm import BsgsSplit
from paper_2601_18511_b200.stc import (SlotBlocks, encrypt_slots, make_slot_to_coeffs_plan, slot_to_coeffs,
                                       slot_to_coeffs_keygen, slot_vectors, stc_plaintexts)

pytestmark = pytest.mark.gpu


def u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("lazy", [False, True])
def test_toy_bit_exact_and_layout(lazy):
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    d, k, N, n = P.mlwe_degree, P.mlwe_rank, P.N, P.N // 2
    A = np.random.default_rng(3).uniform(-1, 1, (d // 2, 2 * k))
    plan = make_slot_to_coeffs_plan(ctx, lazy=lazy)
    b, g = plan.split.baby, plan.split.giant
    keys = slot_to_coeffs_keygen(ctx, sk, plan, seed=13)
    X = encrypt_slots(ctx, sk, A, seed=11)
    before = ctx.ledger.snapshot()
    Y = slot_to_coeffs(ctx, plan, keys, X)
    diff = ctx.ledger.diff(before)
    assert diff["ct_rotations"] == 2 * ((b - 1) + (g - 1)) and diff["pc_mults"] == 2 * n and diff["rescales"] == 2
    assert Y.level == 0 and Y.layout == "app_a_coeff" and Y.n_cols == 2 * k
    # the oracle on the same integers (ct 0)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, slots.encode(slot_vectors(P, A)[0], N, plan.input_scale)[None])[0]
    assert np.array_equal(u32(X.data[0]), ct)
    pt = stc_plaintexts(P, plan.split, 0, n, pt_shift=plan.pt_shift).numpy()
    mods = P.ks_moduli if lazy else P.moduli
    pts = np.stack([np.stack([(pt[t] % q).astype(np.uint32) for q in mods]) for t in range(n)])
    want = O.slot_bsgs(P, ct, pts, 1, b, g, O.rotation_keys(P, 13, s, list(range(1, b))),
                       (O.rotation_keys_plain if lazy else O.rotation_keys)(P, 13, s, [j * b for j in range(1, g)]), lazy=lazy)
    got = u32(Y.data[0, 0])
    assert np.array_equal(got, want), f"{int((got != want).sum())} words differ"
    # decrypts to the App. A coefficient layout of A: exactly what encrypt_acts encodes
    np.testing.assert_allclose(ctx.decrypt_acts(sk, Y), A, atol=2.0 ** -14)
    ph = ctx.decrypt_phase(sk, Y).cpu().numpy()
    assert np.abs(ph - O.encode_acts(P, A)).max() < P.delta * 2.0 ** -14


@pytest.mark.parametrize("n_ct,lazy,halves", [(4, False, 0), (4, True, 0), (7, True, 2), (7, False, 2)])
def test_toy_batched_shared_path_bit_exact(n_ct, lazy, halves, monkeypatch):
    """The shared-memory multi-ciphertext products (forced at toy size; up to 6 cts per plaintext read, the
    baby range optionally split in two accumulating passes) give the oracle's words for every ciphertext."""
    monkeypatch.setenv("HE_SD_SHARED", "1")
    if halves:
        monkeypatch.setenv("HE_SD_HALVES", str(halves))
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    d, k, N, n = P.mlwe_degree, P.mlwe_rank, P.N, P.N // 2
    A = np.random.default_rng(5).uniform(-1, 1, (d // 2, n_ct * k))
    plan = make_slot_to_coeffs_plan(ctx, lazy=lazy, split=BsgsSplit(32, 8) if halves else None)
    b, g = plan.split.baby, plan.split.giant
    keys = slot_to_coeffs_keygen(ctx, sk, plan, seed=13)
    X = encrypt_slots(ctx, sk, A, seed=11)
    Y = slot_to_coeffs(ctx, plan, keys, X)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, np.stack([slots.encode(v, N, plan.input_scale) for v in slot_vectors(P, A)]))
    assert np.array_equal(u32(X.data), ct)
    pt = stc_plaintexts(P, plan.split, 0, n, pt_shift=plan.pt_shift).numpy()
    mods = P.ks_moduli if lazy else P.moduli
    pts = np.stack([np.stack([(pt[t] % q).astype(np.uint32) for q in mods]) for t in range(n)])
    kb = O.rotation_keys(P, 13, s, list(range(1, b)))
    kg = (O.rotation_keys_plain if lazy else O.rotation_keys)(P, 13, s, [j * b for j in range(1, g)])
    for r in range(n_ct):
        want = O.slot_bsgs(P, ct[r], pts, 1, b, g, kb, kg, lazy=lazy)
        assert np.array_equal(u32(Y.data[r, 0]), want), f"ct {r}"
    np.testing.assert_allclose(ctx.decrypt_acts(sk, Y), A, atol=2.0 ** -14)


def test_error_contract():
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    plan = make_slot_to_coeffs_plan(ctx)
    keys = slot_to_coeffs_keygen(ctx, sk, plan, seed=13)
    A = np.zeros((P.mlwe_degree // 2, P.mlwe_rank))
    with pytest.raises(TypeError):
        slot_to_coeffs(ctx, plan, keys, ctx.encrypt_acts(sk, A, seed=1))      # already coefficient-encoded
    X = encrypt_slots(ctx, sk, A, seed=1)
    Y = slot_to_coeffs(ctx, plan, keys, X)
    with pytest.raises(NeedsBootstrapError):
        slot_to_coeffs(ctx, plan, keys, SlotBlocks(Y.data, level=0, n_cols=Y.n_cols))
    # the StC output carries the PCMM's layout tag but no level left on this two-prime chain
    W = np.eye(P.mlwe_rank)
    with pytest.raises(NeedsBootstrapError):
        pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), Y)
    with pytest.raises(ValueError):
        encrypt_slots(ctx, sk, np.zeros((3, P.mlwe_rank)), seed=1)
    with pytest.raises(ValueError):
        slot_to_coeffs(ctx, plan, keys, encrypt_slots(ctx, sk, A, seed=1, scale=P.delta))   # scale mismatch


def test_llama_ring():
    import torch

    P = HeParams()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    d, k = P.mlwe_degree, P.mlwe_rank
    t0 = time.perf_counter()
    plan = make_slot_to_coeffs_plan(ctx)
    keys = slot_to_coeffs_keygen(ctx, sk, plan, seed=13)
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t0
    A = np.random.default_rng(4).uniform(-1, 1, (d // 2, 6 * k))
    X = encrypt_slots(ctx, sk, A, seed=11)
    Y = slot_to_coeffs(ctx, plan, keys, X)                 # warm-up
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(torch.cuda.current_stream())
    reps = 3
    for _ in range(reps):
        Y = slot_to_coeffs(ctx, plan, keys, X)
    ev[1].record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps / X.n_ct
    err = np.abs(ctx.decrypt_acts(sk, Y) - A).max()
    print(f"\nStC N=2^16 ({plan.split.baby}x{plan.split.giant} BSGS): {ms:.2f} ms/ct, plan+keys {t_plan:.1f} s, "
          f"max err {err:.2e} ({-np.log2(err):.1f} bits)")
    assert err < 2.0 ** -12.5
