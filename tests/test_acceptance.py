"""Acceptance gate, in the style of the reference's pkg/tests/test_acceptance.py: one criterion
per test, each with a hard wall-clock budget (check_budget, test_acceptance.py:41-43).

  a01  MLWE PCMM consumes exactly one level, one rescale per output block, no rotations
  a02  toy PCMM: every output word bit-exact vs the oracle            (BASELINE config 1)
  a03  Llama 4096x4096x128: decrypted error below 2^-12                (BASELINE config 2)
  a04  metric shape 4096x11008x128: all 4096 x 65 792 words exact via the selection identity
  a05  streamed-to-host output == device output
  a06  Rhombus PCMv toy: every output word bit-exact vs the oracle; one level; n-1 rotations
  a07  App. A index maps equal the reference's bitrev tables           (CPU)
  a08  oracle float semantics equal hesim's clear_pcmm / pcmm_bsgs      (CPU)
  a09  row-sharded gather reassembles the unsharded output exactly     (CPU, gloo)
  a10  slot-domain PCMM at d = 16: BSGS spends 6 rotations, depth-1 15 (reference c03,
       test_acceptance.py:79-90), one level each, both decrypt to clear_pcmm
  a11  ring packing: the packed level-0 output decrypts to A W^T in the input's own layout
"""

import time
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).parent / "golden"


def check_budget(t0: float, budget_s: float) -> None:
    elapsed = time.perf_counter() - t0
    assert elapsed < budget_s, f"took {elapsed:.1f} s > budget {budget_s} s"


@pytest.mark.gpu
def test_a01_one_level_one_rescale_per_block():
    from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe

    t0 = time.perf_counter()
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    rng = np.random.default_rng(0)
    sk = ctx.keygen(1)
    X = ctx.encrypt_acts(sk, rng.uniform(-1, 1, (P.tokens, 64)), seed=2)
    plan = make_mlwe_pcmm_plan(ctx, rng.uniform(-1, 1, (96, 64)) / 8)
    snap = ctx.ledger.snapshot()
    Y = pcmm_mlwe(ctx, plan, X)
    d = ctx.ledger.diff(snap)
    assert X.level - Y.level == 1
    assert d["rescales"] == 96 // P.mlwe_rank and d["ct_rotations"] == 0 and d["bootstraps"] == 0
    check_budget(t0, 30)


@pytest.mark.gpu
def test_a02_toy_bit_exact_config1():
    from test_gpu_pcmm import test_fixture_parity_baseline_config1

    t0 = time.perf_counter()
    test_fixture_parity_baseline_config1()
    check_budget(t0, 30)


@pytest.mark.gpu
def test_a03_llama_qkv_precision():
    import test_gpu_pcmm as G

    from paper_2601_18511_b200 import HeParams, make_mlwe_pcmm_plan, pcmm_mlwe

    t0 = time.perf_counter()
    P = HeParams.llama()
    ctx, sk, A, W, X = G.setup(P, 4096, 4096)
    Y = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), X)
    dec = ctx.decrypt_pcmm(sk, Y, rows=(0, 512))
    err = np.nanmax(np.abs(dec - A @ W.T))
    assert err < 2 ** -12, err
    check_budget(t0, 120)


@pytest.mark.gpu
def test_a04_metric_shape_full_output_exact():
    from test_gpu_pcmm import test_selection_identity_full_output_metric_shape

    t0 = time.perf_counter()
    test_selection_identity_full_output_metric_shape("spectral")
    check_budget(t0, 120)


@pytest.mark.gpu
def test_a05_streamed_equals_device():
    from test_gpu_pcmm import test_streamed_to_host_matches_device_output

    t0 = time.perf_counter()
    test_streamed_to_host_matches_device_output("spectral")
    check_budget(t0, 60)


@pytest.mark.gpu
def test_a06_rhombus_toy_bit_exact():
    from test_gpu_rhombus import test_toy_pcmv_bit_exact

    t0 = time.perf_counter()
    test_toy_pcmv_bit_exact(200, 300, None)
    check_budget(t0, 60)


def test_a07_layout_maps_match_reference():
    import test_layout as T

    t0 = time.perf_counter()
    for k in (3, 7, 8, 11):
        T.test_bit_reverse_matches_reference_table(k)
    T.test_byte_mix_matches_reference()
    T.test_half_reverse_matches_reference()
    T.test_shuffle_matrix_matches_reference()
    T.test_block_conjugation_is_papers_g_shuffle_in_component_order()
    check_budget(t0, 30)


def test_a08_oracle_float_semantics_match_hesim():
    import test_oracle as T

    t0 = time.perf_counter()
    T.test_baseline_config1_matches_hesim()
    check_budget(t0, 30)


def test_a09_row_sharded_gather_exact():
    import test_multirank as T

    t0 = time.perf_counter()
    T.test_row_sharded_pcmm_gathers_exact_output(2, 64)
    check_budget(t0, 120)


@pytest.mark.gpu
def test_a10_slot_pcmm_rotation_counts_like_reference_c03():
    from paper_2601_18511_b200 import HeContext, HeParams
    from paper_2601_18511_b200.slotpcmm import (BsgsSplit, clear_slot_pcmm, decrypt_packed, encrypt_packed,
                                                make_slot_pcmm_plan, pcmm_slot_bsgs, pcmm_slot_depth1,
                                                slot_pcmm_keygen)

    t0 = time.perf_counter()
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(1)
    rng = np.random.default_rng(3)
    d = 16
    W, B = rng.uniform(-1, 1, (d, d)) / 4, rng.uniform(-1, 1, (d, d))
    X = encrypt_packed(ctx, sk, B, 1, seed=2)
    rots = {}
    for name, split, fn in (("bsgs", None, pcmm_slot_bsgs), ("depth1", BsgsSplit(d, 1), pcmm_slot_depth1)):
        plan = make_slot_pcmm_plan(ctx, W, shear_power=0, split=split)
        keys = slot_pcmm_keygen(ctx, sk, plan, 5)
        snap = ctx.ledger.snapshot()
        Y = fn(ctx, plan, keys, X)
        diff = ctx.ledger.diff(snap)
        rots[name] = diff["ct_rotations"]
        assert X.level - Y.level == 1 and diff["rescales"] == 1
        assert np.abs(decrypt_packed(ctx, sk, Y) - clear_slot_pcmm(W, B, 0)).max() < 2 ** -13
    assert rots == {"bsgs": 6, "depth1": 15}
    check_budget(t0, 60)


@pytest.mark.gpu
def test_a11_ring_packed_output_decrypts_in_input_layout():
    from paper_2601_18511_b200 import (HeContext, HeParams, make_mlwe_pcmm_plan, make_ring_pack_plan, pcmm_packed,
                                       ring_pack_keygen)

    t0 = time.perf_counter()
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(1)
    rng = np.random.default_rng(4)
    A, W = rng.uniform(-1, 1, (P.tokens, 48)), rng.uniform(-1, 1, (64, 48)) / 8
    Y = pcmm_packed(ctx, make_mlwe_pcmm_plan(ctx, W), make_ring_pack_plan(ctx, 64), ring_pack_keygen(ctx, sk, 2),
                    ctx.encrypt_acts(sk, A, seed=3))
    assert Y.level == 0 and Y.layout == "app_a_coeff" and Y.n_cols == 64
    assert np.abs(ctx.decrypt_acts(sk, Y) - A @ W.T).max() < 2 ** -14
    check_budget(t0, 60)
