"""Error contract of the newer entry points (the reference's matmul.py:139-149 rules: TypeError for a
non-ciphertext operand, ValueError for shape/layout/level misuse, NeedsBootstrapError when no level is
left), raised before any launch, and the C ABI's status codes surfacing as those exceptions."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2601_18511_b200 import (CtBlocks, HeContext, HeParams, make_mlwe_pcmm_plan, make_ring_pack_plan, mod_raise,
                                   native, pcmm_level1, pcmm_packed, ring_pack_keygen)
from paper_2601_18511_b200.errors import NeedsBootstrapError
from paper_2601_18511_b200.rhombus import encrypt_vector, make_rhombus_plan, pcmv_rhombus_shard, rhombus_keygen
from paper_2601_18511_b200.slotpcmm import PackedCt, encrypt_packed, make_rope_plan, slot_linear, slot_linear_keygen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def toy():
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    rng = np.random.default_rng(0)
    W = rng.uniform(-1, 1, (32, 32)) / 8
    X = ctx.encrypt_acts(sk, rng.uniform(-1, 1, (P.tokens, 32)), seed=1)
    return P, ctx, sk, W, X


def test_packed_op_levels_and_types(toy):
    P, ctx, sk, W, X = toy
    plan = make_mlwe_pcmm_plan(ctx, W)
    rp = make_ring_pack_plan(ctx, 32)
    keys = ring_pack_keygen(ctx, sk, 3)
    with pytest.raises(TypeError):
        pcmm_packed(ctx, plan, rp, keys, X.data)
    with pytest.raises(NeedsBootstrapError):
        pcmm_level1(ctx, plan, CtBlocks(X.data, level=0, n_cols=32))
    with pytest.raises(ValueError, match="layout mismatch"):
        pcmm_level1(ctx, plan, CtBlocks(X.data, level=1, n_cols=32, layout="rhombus_h"))
    Y = pcmm_packed(ctx, plan, rp, keys, X)
    with pytest.raises(ValueError):
        mod_raise(ctx, X, [1073707009])          # level 1: ModRaise takes level-0 ciphertexts
    assert tuple(mod_raise(ctx, Y, [1073707009]).shape) == (2, 1, 2, P.N)


def test_rhombus_shard_offsets_checked(toy):
    P, ctx, sk, W, X = toy
    keys = rhombus_keygen(ctx, sk, 9)
    x = encrypt_vector(ctx, sk, np.ones(32) / 4, seed=2)
    plan = make_rhombus_plan(ctx, W)
    with pytest.raises(ValueError, match="exceed"):
        pcmv_rhombus_shard(ctx, plan, keys, x, piece0=P.N // P.rhombus_degree)   # past the last input piece
    part = pcmv_rhombus_shard(ctx, plan, keys, x)
    assert tuple(part.shape) == (2, 2, P.N)


def test_slot_linear_levels(toy):
    P, ctx, sk, W, X = toy
    plan = make_rope_plan(ctx, 16, 16 + np.arange(16), shear_power=2)
    keys = slot_linear_keygen(ctx, sk, plan, 4)
    Xp = encrypt_packed(ctx, sk, np.eye(16) / 4, 2, seed=5)
    with pytest.raises(TypeError):
        slot_linear(ctx, plan, keys, Xp.data)
    with pytest.raises(NeedsBootstrapError):
        slot_linear(ctx, plan, keys, PackedCt(Xp.data, level=0, dim=16, shear_power=2))
    assert slot_linear(ctx, plan, keys, Xp).level == 0


def test_c_abi_status_codes(toy):
    P, ctx, sk, W, X = toy
    h = ctypes.c_void_p()
    with pytest.raises(ValueError):        # n_out not a multiple of k
        native.call("he_ring_pack_plan_create", ctx.handle, 24, 0, ctypes.byref(h))
    with pytest.raises(ValueError):        # unknown packing method
        native.call("he_ring_pack_plan_create", ctx.handle, 32, 7, ctypes.byref(h))
    with pytest.raises(ValueError):        # split does not cover d
        native.call("he_slot_pcmm_plan_create", ctx.handle, X.data.data_ptr(), 16, 3, 5, ctypes.byref(h))
    with pytest.raises(ValueError):        # steps[0] must be 0
        arr = (ctypes.c_int32 * 2)(1, 2)
        native.call("he_slot_lt_plan_create", ctx.handle, X.data.data_ptr(), 2, arr, ctypes.byref(h))
    with pytest.raises(ValueError):        # no primes
        native.call("he_mod_raise", ctx.handle, X.data.data_ptr(), 1, X.data.data_ptr(), 0, X.data.data_ptr(),
                    ctx.stream())
    torch.cuda.synchronize()


def test_slot_bsgs_abi_status_codes(toy):
    """The slot BSGS entry points added for SlotToCoeffs reject bad arguments with HE_EINVAL / ValueError."""
    P, ctx, sk, W, X = toy
    N = P.N
    pts = torch.zeros((16 * 16, 3, N), dtype=torch.int32, device=ctx.device)
    h = ctypes.c_void_p()
    with pytest.raises(ValueError):   # lazy ModDown needs b % 8 == 0
        native.call("he_slot_bsgs_plan_create_ext", ctx.handle, pts.data_ptr(), 4, 64, 1, 1, ctypes.byref(h))
    with pytest.raises(ValueError):   # b g stride > N/2
        native.call("he_slot_bsgs_plan_create_ext", ctx.handle, pts.data_ptr(), 16, 16, 2, 0, ctypes.byref(h))
    pt = torch.zeros((2, N), dtype=torch.int64, device=ctx.device)
    with pytest.raises(ValueError):   # n_mods must be 2 or 3
        native.call("he_slot_pcmm_encode_pts_ext", ctx.handle, pt.data_ptr(), 2, 4, pts.data_ptr(), ctx.stream())
    native.call("he_slot_bsgs_plan_create_ext", ctx.handle, pts.data_ptr(), 16, 16, 1, 3, ctypes.byref(h))
    n = ctypes.c_uint64()
    native.call("he_slot_pcmm_workspace_bytes", h, ctypes.byref(n))
    ws = torch.empty(n.value // 4 + 1, dtype=torch.int32, device=ctx.device)
    ct = torch.zeros((1, 2, 2, N), dtype=torch.int32, device=ctx.device)
    out = torch.zeros((1, 2, N), dtype=torch.int32, device=ctx.device)
    keys = torch.zeros((15, 4, 2, 3, N), dtype=torch.int32, device=ctx.device)
    led = native.HeLedgerC()
    with pytest.raises(ValueError):   # empty batch
        native.call("he_slot_pcmm_run_batch", h, ct.data_ptr(), 0, 1, keys.data_ptr(), keys.data_ptr(), out.data_ptr(),
                    ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    with pytest.raises(NeedsBootstrapError):
        native.call("he_slot_pcmm_run_batch", h, ct.data_ptr(), 1, 0, keys.data_ptr(), keys.data_ptr(), out.data_ptr(),
                    ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    with pytest.raises(ValueError):   # workspace too small
        native.call("he_slot_pcmm_run_batch", h, ct.data_ptr(), 1, 1, keys.data_ptr(), keys.data_ptr(), out.data_ptr(),
                    ws.data_ptr(), 64, ctx.stream(), ctypes.byref(led))
    native.lib().he_slot_pcmm_plan_destroy(h)
    with pytest.raises(ValueError, match="unknown slot plan flags"):
        native.call("he_slot_bsgs_plan_create_ext", ctx.handle, pts.data_ptr(), 16, 16, 1, 8, ctypes.byref(h))
    with pytest.raises(ValueError, match="PLAIN_GIANT needs"):
        native.call("he_slot_bsgs_plan_create_ext", ctx.handle, pts.data_ptr(), 16, 16, 1, 2, ctypes.byref(h))


def test_slot_keys_must_match_the_plan(toy):
    """keys from another plan (other steps, or plain instead of gadget giant keys) are rejected
    before any launch -- the kernels would otherwise read past the key buffers."""
    from paper_2601_18511_b200.slotpcmm import (BsgsSplit, SlotPcmmKeys, make_slot_pcmm_plan, pcmm_slot_bsgs,
                                                slot_pcmm_keygen)
    from paper_2601_18511_b200.stc import (encrypt_slots, make_slot_to_coeffs_plan, slot_to_coeffs,
                                           slot_to_coeffs_keygen)

    P, ctx, sk, W, X = toy
    rng = np.random.default_rng(3)
    p16 = make_slot_pcmm_plan(ctx, rng.uniform(-1, 1, (16, 16)) / 4, shear_power=0)
    p16b = make_slot_pcmm_plan(ctx, rng.uniform(-1, 1, (16, 16)) / 4, shear_power=0, split=BsgsSplit(8, 2))
    k16 = slot_pcmm_keygen(ctx, sk, p16, seed=3)
    B = encrypt_packed(ctx, sk, rng.uniform(-1, 1, (16, 16)) / 4, 1, seed=4)
    with pytest.raises(ValueError, match="key/plan mismatch"):
        pcmm_slot_bsgs(ctx, p16b, k16, B)
    assert pcmm_slot_bsgs(ctx, p16, k16, B).level == 0
    sp = make_slot_to_coeffs_plan(ctx)
    ks = slot_to_coeffs_keygen(ctx, sk, sp, seed=5)
    Xs = encrypt_slots(ctx, sk, rng.uniform(-1, 1, (P.tokens, P.mlwe_rank)), seed=6, scale=sp.input_scale)
    if getattr(sp, "plain_giant", False):   # gadget giant keys where the plan reads plain ones
        bad = SlotPcmmKeys(ks.baby, torch.zeros((ks.giant.shape[0], 4, 2, 3, P.N), dtype=torch.int32,
                                                device=ctx.device), ks.steps)
        with pytest.raises(ValueError, match="giant keys have shape"):
            slot_to_coeffs(ctx, sp, bad, Xs)
    with pytest.raises(ValueError, match="key/plan mismatch"):
        slot_to_coeffs(ctx, sp, k16, Xs)
    assert slot_to_coeffs(ctx, sp, ks, Xs).level == 0


def test_plans_keep_their_context(toy):
    """a plan holds its creating context's device state alive and refuses another context."""
    import gc

    P, ctx, sk, W, X = toy
    other = HeContext(P, rng="seeded")
    plan = make_mlwe_pcmm_plan(other, W)
    del other
    gc.collect()
    with pytest.raises(ValueError, match="another HeContext"):
        from paper_2601_18511_b200 import pcmm_mlwe
        pcmm_mlwe(ctx, plan, X)
    assert plan._ctx_keepalive.handle   # the device context is still alive
