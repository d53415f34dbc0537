"""The modulus chain on the GPU (he_chain.cu) vs the CPU oracle (he_oracle_chain.c): encryption at level 4,
each factorized-SlotToCoeffs map word for word, and the paper's pipeline -- lower the level, SlotToCoeffs
to level 1, MLWE PCMM, ring packing, ModRaise -- bit-exact at the toy ring
and within the stated precision at N = 2^16."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2601_18511_b200 import (HeContext, HeParams, clear_pcmm, make_mlwe_pcmm_plan, make_ring_pack_plan,
                                   mod_raise, pcmm_mlwe, pcmm_packed, ring_pack_keygen, slots)
from paper_2601_18511_b200.chain import (chain_map, encrypt_slots_at, factorized_stc_keygen, lower_level,
                                         make_factorized_stc_plan, slot_to_coeffs_factorized)
from paper_2601_18511_b200.errors import NeedsBootstrapError
from paper_2601_18511_b200.stc import slot_vectors

pytestmark = pytest.mark.gpu


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _toy(levels=3, seed=0):
    P = HeParams.toy_chain(levels)
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    A = np.random.default_rng(seed).uniform(-1, 1, (P.tokens, 2 * P.mlwe_rank))
    return P, ctx, sk, A


def _oracle_keys(P, m, seed, s):
    return (O.chain_rotation_keys(P, seed, s, m.baby_steps, m.level),
            O.chain_rotation_keys(P, seed, s, m.giant_steps, m.level))


def test_chain_encrypt_matches_oracle():
    P, ctx, sk, A = _toy()
    plan = make_factorized_stc_plan(ctx)
    X = encrypt_slots_at(ctx, sk, A, level=4, seed=13, scale=plan.input_scale)
    s = O.keygen(P, 7)
    z = slot_vectors(P, A)
    pt = np.stack([slots.encode(v, P.N, plan.input_scale) for v in z])
    assert np.array_equal(u32(X.data), O.encrypt(P, 13, s, pt, level=4))


def test_factorized_stc_bit_exact_and_decrypts_to_the_pcmm_layout():
    P, ctx, sk, A = _toy()
    s = O.keygen(P, 7)
    plan = make_factorized_stc_plan(ctx)
    assert [m.level for m in plan.maps] == [4, 3, 2] and plan.output_level == 1
    keys = factorized_stc_keygen(ctx, sk, plan, seed=21)
    X = encrypt_slots_at(ctx, sk, A, level=4, seed=13, scale=plan.input_scale)
    ref = u32(X.data)
    data, level = X.data, 4
    for k, (m, kk) in enumerate(zip(plan.maps, keys)):
        data = chain_map(ctx, m, kk, data, level)
        kb, kg = _oracle_keys(P, m, 21 + 7919 * k, s)
        pts = np.stack([np.stack([(m.pts_int[t] % q).astype(np.uint32) for q in P.moduli[:level + 1]])
                        for t in range(m.b * m.g)])
        ref = np.stack([O.chain_bsgs(P, ref[r], pts, level, m.b, m.g, m.stride, m.T, kb, kg) for r in range(len(ref))])
        assert np.array_equal(u32(data), ref), f"map {k} (level {level}) differs from the oracle"
        level -= 1
    before = ctx.ledger.snapshot()
    Y = slot_to_coeffs_factorized(ctx, plan, keys, X)
    diff = ctx.ledger.diff(before)
    assert Y.level == 1 and np.array_equal(u32(Y.data), ref)
    assert diff["rescales"] == 3 * X.n_ct and diff["ct_rotations"] == plan.rotations * X.n_ct
    got = ctx.decrypt_acts(sk, Y)
    assert np.abs(got - A).max() < 2 ** -14


def test_lower_stc_pcmm_ringpack_modraise_chain_toy():
    """Level 5 -> lower to 4 -> factorized StC -> level-1 PCMM input -> pcmm_mlwe / ring packing (both
    bit-exact vs the oracle run on the StC output) -> ModRaise of the packed level-0 result."""
    P, ctx, sk, A = _toy(levels=4, seed=1)
    s = O.keygen(P, 7)
    W = np.random.default_rng(2).uniform(-1, 1, (2 * P.mlwe_rank, A.shape[1])) / np.sqrt(A.shape[1])
    plan = make_factorized_stc_plan(ctx, input_level=4)
    keys = factorized_stc_keygen(ctx, sk, plan, seed=31)
    X5 = encrypt_slots_at(ctx, sk, A, level=5, seed=17, scale=plan.input_scale)
    with pytest.raises(ValueError, match="lower it first"):
        slot_to_coeffs_factorized(ctx, plan, keys, X5)
    X4 = lower_level(X5, 4)
    assert X4.level == 4 and np.array_equal(u32(X4.data), u32(X5.data)[:, :5])
    Xc = slot_to_coeffs_factorized(ctx, plan, keys, X4)
    assert Xc.level == 1
    ct = u32(Xc.data)
    pplan = make_mlwe_pcmm_plan(ctx, W)
    Y = pcmm_mlwe(ctx, pplan, Xc)
    torch.cuda.synchronize()
    ref = O.pcmm(P, O.encode_weights(P, W), ct)
    d = P.mlwe_degree
    assert np.array_equal(u32(Y.out_a), ref[:, d:])
    assert np.abs(ctx.decrypt_pcmm(sk, Y) - clear_pcmm(W, A)).max() < 2 ** -12
    rk = ring_pack_keygen(ctx, sk, 5)
    Yp = pcmm_packed(ctx, pplan, make_ring_pack_plan(ctx, W.shape[0]), rk, Xc)
    raw = [O.pcmm_limb(P, O.encode_weights(P, W), ct, L) for L in range(2)]
    ref_rp = O.mlwe_to_rlwe(P, *O.raw_device_layout(P, raw), O.mlwe_ks_keys(P, 5, s))
    assert np.array_equal(u32(Yp.data)[:, 0], ref_rp)
    assert np.abs(ctx.decrypt_acts(sk, Yp) - clear_pcmm(W, A)).max() < 2 ** -12
    raised = mod_raise(ctx, Yp, list(P.moduli[2:]))
    assert tuple(raised.shape) == (Yp.data.shape[0], len(P.moduli) - 2, 2, P.N)


def test_chain_errors():
    P, ctx, sk, A = _toy()
    plan = make_factorized_stc_plan(ctx)
    keys = factorized_stc_keygen(ctx, sk, plan, seed=3)
    X = encrypt_slots_at(ctx, sk, A, level=4, seed=4, scale=plan.input_scale)
    with pytest.raises(TypeError):
        slot_to_coeffs_factorized(ctx, plan, keys, X.data)
    with pytest.raises(NeedsBootstrapError):
        slot_to_coeffs_factorized(ctx, plan, keys, lower_level(X, 2))
    with pytest.raises(ValueError, match="scale mismatch"):
        slot_to_coeffs_factorized(ctx, plan, keys, encrypt_slots_at(ctx, sk, A, level=4, seed=4))
    with pytest.raises(ValueError, match="key/plan mismatch"):
        slot_to_coeffs_factorized(ctx, plan, keys[::-1], X)
    with pytest.raises(ValueError):
        make_factorized_stc_plan(HeContext(HeParams.toy(), rng="seeded"))


def test_llama_chain_precision():
    """N = 2^16: level 4 -> factorized StC (54 rotations, 160 plaintexts) -> PCMM -> ring packing, >= 12 bits."""
    P = HeParams.llama_chain()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (P.tokens, 512))
    W = rng.uniform(-1, 1, (512, 512)) / np.sqrt(512)
    plan = make_factorized_stc_plan(ctx)
    assert plan.rotations == 54 and plan.plaintexts == 64 + 64 + 32
    keys = factorized_stc_keygen(ctx, sk, plan, seed=9)
    X = encrypt_slots_at(ctx, sk, A, seed=3, scale=plan.input_scale)
    Xc = slot_to_coeffs_factorized(ctx, plan, keys, X)
    err_stc = np.abs(ctx.decrypt_acts(sk, Xc) - A).max()
    assert err_stc < 2 ** -12, err_stc
    Yp = pcmm_packed(ctx, make_mlwe_pcmm_plan(ctx, W), make_ring_pack_plan(ctx, 512), ring_pack_keygen(ctx, sk, 5), Xc)
    err = np.abs(ctx.decrypt_acts(sk, Yp) - clear_pcmm(W, A)).max()
    assert err < 2 ** -12, err


def test_llama_chain_precision_sweep():
    """Record the StC error against the per-map scale shifts (the default is (10, 10, 10))."""
    P = HeParams.llama_chain()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    A = np.random.default_rng(5).uniform(-1, 1, (P.tokens, 256))
    for shifts in ((3, 3, 3), (6, 6, 6), (10, 10, 10), (12, 12, 12), (8, 10, 12)):
        plan = make_factorized_stc_plan(ctx, shifts=shifts)
        keys = factorized_stc_keygen(ctx, sk, plan, seed=9)
        X = encrypt_slots_at(ctx, sk, A, seed=3, scale=plan.input_scale)
        err = np.abs(ctx.decrypt_acts(sk, slot_to_coeffs_factorized(ctx, plan, keys, X)) - A).max()
        print(f"shifts {shifts}: max err {err:.3e} = 2^{np.log2(err):.1f}")
