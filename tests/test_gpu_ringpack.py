"""MLWE -> RLWE ring packing on the GPU against the CPU oracle.

Bar: bit-exact on every word -- the level-1 (un-rescaled) PCMM words of both limbs, the Galois
keys, and the packed level-0 RLWE ciphertexts -- at toy size against oracle.pcmm_limb /
oracle.ring_pack_keys / oracle.pcmm_ring_pack; at Llama sizes the level-1 words must rescale to
exactly the words of the (separately tested) level-0 PCMM output, and the packed ciphertexts must
decrypt to A @ W^T within the stated CKKS precision (>= 14 bits; paper target 12)."""

import math

import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200 import (HeParams, make_mlwe_pcmm_plan, make_ring_pack_plan, pcmm_level1, pcmm_mlwe,
                                   pcmm_packed, ring_pack, ring_pack_keygen)

from test_gpu_pcmm import setup, u32

pytestmark = pytest.mark.gpu
ALGOS = ["spectral", "direct"]
METHODS = ["keyswitch", "trace", "keyswitch1"]


def _raw_oracle(P, W, A):
    ct = O.encrypt(P, 11, O.keygen(P, 7), O.encode_acts(P, A))
    Wt = O.encode_weights(P, W)
    return Wt, ct, [O.pcmm_limb(P, Wt, ct, L) for L in range(2)]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("n_out,n_in", [(16, 16), (64, 48), (32, 256)])
def test_toy_level1_words_bit_exact(n_out, n_in, algo):
    P = HeParams.toy()
    ctx, sk, A, W, X = setup(P, n_out, n_in)
    _, _, raw = _raw_oracle(P, W, A)
    d, k = P.mlwe_degree, P.mlwe_rank
    rb, ra = pcmm_level1(ctx, make_mlwe_pcmm_plan(ctx, W, algo=algo), X)
    rb, ra = u32(rb), u32(ra)
    for L in range(2):
        assert np.array_equal(ra[L], raw[L][:, d:]), f"limb {L} a' words"
        for y in range(n_out):
            assert np.array_equal(rb[L, y // k, y % k + k * np.arange(d)], raw[L][y, :d]), f"limb {L} b' row {y}"


@pytest.mark.parametrize("method", METHODS)
def test_toy_keys_match_oracle(method):
    P = HeParams.toy()
    ctx, sk, A, W, X = setup(P, 16, 16)
    keys = ring_pack_keygen(ctx, sk, seed=5, method=method)
    import torch

    if method == "keyswitch1":   # [k, 2, 4, N]: q0, q1, P1 through the context's inverse NTTs (P2 via the output)
        ref = O.mlwe_ks_keys1(P, 5, O.keygen(P, 7))
        g = keys.gal.clone()
        for j in range(3):
            blk = g[:, :, j, :].contiguous().reshape(-1, P.N)
            ctx_ntt_inverse(ctx, blk, j)
            g[:, :, j, :] = blk.reshape(g.shape[0], 2, P.N)
        torch.cuda.synchronize()
        assert np.array_equal(u32(g)[:, :, :3], ref[:, :, :3])
        return
    ref = (O.ring_pack_keys if method == "trace" else O.mlwe_ks_keys)(P, 5, O.keygen(P, 7))
    # device keys are NTT-domain: compare after the inverse transform per modulus
    g = keys.gal.clone()
    lg, N = g.shape[0], P.N
    for j in range(3):
        blk = g[:, :, :, j, :].contiguous().reshape(-1, N)
        ctx_ntt_inverse(ctx, blk, j)
        g[:, :, :, j, :] = blk.reshape(lg, 2, 2, N)
    torch.cuda.synchronize()
    assert np.array_equal(u32(g), ref)


def ctx_ntt_inverse(ctx, data, limb):
    from paper_2601_18511_b200 import native

    native.call("he_ntt_inverse", ctx.handle, data.data_ptr(), ctx.params.N, limb, int(data.shape[0]), ctx.params.N,
                ctx.stream())


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("n_out,n_in", [(16, 16), (64, 48), (48, 128)])
def test_toy_packed_ciphertexts_bit_exact_and_decrypt(n_out, n_in, algo, method):
    P = HeParams.toy()
    ctx, sk, A, W, X = setup(P, n_out, n_in, seed=n_out + n_in)
    Wt, ct, raw = _raw_oracle(P, W, A)
    s = O.keygen(P, 7)
    if method == "trace":
        ref = O.ring_pack(P, O.ring_pack_leaves(P, raw), O.ring_pack_keys(P, 5, s))[1]
    elif method == "keyswitch1":
        ref = O.mlwe_to_rlwe1(P, *O.raw_device_layout(P, raw), O.mlwe_ks_keys1(P, 5, s))
    else:
        ref = O.mlwe_to_rlwe(P, *O.raw_device_layout(P, raw), O.mlwe_ks_keys(P, 5, s))
    keys = ring_pack_keygen(ctx, sk, seed=5, method=method)
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    rp = make_ring_pack_plan(ctx, n_out, method=method)
    before = ctx.ledger.snapshot()
    Y = pcmm_packed(ctx, plan, rp, keys, X)
    diff = ctx.ledger.diff(before)
    k = P.mlwe_rank
    rot = (k - 1) * n_out // k if method == "trace" else 0
    assert diff["ct_rotations"] == rot and diff["rescales"] == n_out // k
    assert Y.level == 0 and Y.n_cols == n_out and tuple(Y.data.shape) == (n_out // k, 1, 2, P.N)
    got = u32(Y.data)[:, 0]
    assert np.array_equal(got, ref), f"{int((got != ref).sum())} words differ"
    dec = ctx.decrypt_acts(sk, Y)
    refm = A @ W.T
    err = np.abs(dec - refm).max()
    assert err < np.abs(refm).max() * 2.0 ** -14


def test_ring_pack_errors():
    P = HeParams.toy()
    ctx, sk, A, W, X = setup(P, 16, 16)
    with pytest.raises(ValueError):
        make_ring_pack_plan(ctx, 24)   # not a multiple of k
    plan = make_mlwe_pcmm_plan(ctx, W)
    with pytest.raises(ValueError):
        pcmm_packed(ctx, plan, make_ring_pack_plan(ctx, 32), ring_pack_keygen(ctx, sk, 5), X)
    with pytest.raises(ValueError):
        make_ring_pack_plan(ctx, 16, method="bogus")
    with pytest.raises(ValueError):   # keys of the other method
        pcmm_packed(ctx, plan, make_ring_pack_plan(ctx, 16), ring_pack_keygen(ctx, sk, 5, method="trace"), X)


def _rescale(P, x0, x1):
    import torch

    q0, q1 = int(P.moduli[0]), int(P.moduli[1])
    x0 = x0.to(torch.int64) & 0xFFFFFFFF
    x1 = x1.to(torch.int64) & 0xFFFFFFFF
    x1c = torch.where(x1 > q1 // 2, x1 - q1, x1)
    t = torch.remainder(x0 - x1c, q0)
    return torch.remainder(t * pow(q1, q0 - 2, q0), q0)


@pytest.mark.parametrize("algo", ALGOS)
def test_llama_level1_words_rescale_to_pcmm_output(algo):
    """Full-output property at a Llama shape: rescale(level-1 words) == the level-0 PCMM words."""
    import torch

    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, 512, 1024, seed=3)
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    Y = pcmm_mlwe(ctx, plan, X)
    rb, ra = pcmm_level1(ctx, plan, X)
    torch.cuda.synchronize()
    assert torch.equal(_rescale(P, ra[0], ra[1]), Y.out_a.to(torch.int64) & 0xFFFFFFFF)
    assert torch.equal(_rescale(P, rb[0], rb[1]), Y.out_b.to(torch.int64) & 0xFFFFFFFF)


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("n_out,n_in", [(512, 1024), (1024, 4096)])
def test_llama_packed_decrypts_to_product(n_out, n_in, method):
    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, n_out, n_in, seed=5)
    keys = ring_pack_keygen(ctx, sk, seed=9, method=method)
    Y = pcmm_packed(ctx, make_mlwe_pcmm_plan(ctx, W), make_ring_pack_plan(ctx, n_out, method=method), keys, X)
    dec = ctx.decrypt_acts(sk, Y)
    ref = A @ W.T
    err = np.abs(dec - ref).max()
    bits = -math.log2(err / np.abs(ref).max())
    assert bits >= 14, f"{bits:.1f} bits"


def test_mod_raise_of_packed_output():
    """ModRaise (the Half-Bootstrap hand-off): the packed level-0 output lifted into two fresh primes
    decrypts, via CRT, to phase_q0 + q0 I(X) with a small integer I -- the form EvalMod expects."""
    from paper_2601_18511_b200 import mod_raise
    from paper_2601_18511_b200.params import ntt_primes

    P = HeParams.toy()
    ctx, sk, A, W, X = setup(P, 32, 48, seed=4)
    Y = pcmm_packed(ctx, make_mlwe_pcmm_plan(ctx, W), make_ring_pack_plan(ctx, 32), ring_pack_keygen(ctx, sk, 5), X)
    primes = [p for p in ntt_primes(2 * P.N, 1 << 30, 4) if p not in P.ks_moduli][:2]
    R = u32(mod_raise(ctx, Y, primes))                                       # [n_ct, 2, 2, N]
    s = sk.s.cpu().numpy()
    q0 = P.moduli[0]
    for b in range(R.shape[0]):
        ph0 = O.decrypt_under(P, u32(Y.data)[b, 0, 0], u32(Y.data)[b, 0, 1], s, q0)
        ph = [O.decrypt_under(P, R[b, i, 0], R[b, i, 1], s, p) for i, p in enumerate(primes)]
        p1, p2 = primes
        # CRT of the two centred residues -> the integer phase (|.| < p1 p2 / 2)
        t = ((ph[1] - ph[0]) % p2) * pow(p1, -1, p2) % p2
        full = ph[0].astype(object) + p1 * t.astype(object)
        full = np.array([v - p1 * p2 if v > p1 * p2 // 2 else v for v in full], dtype=object)
        diff = full - ph0.astype(object)
        assert all(v % q0 == 0 for v in diff)
        I = np.array([v // q0 for v in diff], dtype=np.int64)
        assert np.abs(I).max() <= P.N


@pytest.mark.gpu
def test_llama_fused_digits_cols_equal_unfused(monkeypatch):
    """KEYSWITCH1 at the Llama ring fuses the digit formation with the NTT's cols pass (k_ms1_digits_cols);
    HE_RP_UNFUSED=1 runs the separate kernels every other ring size uses (bit-exact vs the oracle at the toy
    ring).  Both must give the same packed words."""
    import torch

    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, 512, 1024, seed=6)
    keys = ring_pack_keygen(ctx, sk, seed=9, method="keyswitch1")
    plan = make_mlwe_pcmm_plan(ctx, W)
    rp = make_ring_pack_plan(ctx, 512, method="keyswitch1")
    monkeypatch.delenv("HE_RP_UNFUSED", raising=False)
    fused = pcmm_packed(ctx, plan, rp, keys, X).data.clone()
    monkeypatch.setenv("HE_RP_UNFUSED", "1")
    unfused = pcmm_packed(ctx, plan, rp, keys, X).data.clone()
    torch.cuda.synchronize()
    assert torch.equal(fused, unfused)


def test_llama_keyswitch1_block_bit_exact_vs_oracle():
    """Ring packing at the Llama ring (N = 2^16, k = d = 256) word for word against the oracle: one output block
    (256 rows) packed by the GPU (the fused digits + cols path, the rows NTT, the MAC, ModDown + rescale) equals
    oracle.mlwe_to_rlwe1 on the same level-1 words with the oracle's own keys (or_mlwe_ksk1 from the same seed and
    secret; the device keygen equals them at the toy ring)."""
    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, 256, 1024, seed=8)
    keys = ring_pack_keygen(ctx, sk, seed=9, method="keyswitch1")
    plan = make_mlwe_pcmm_plan(ctx, W)
    rp = make_ring_pack_plan(ctx, 256, method="keyswitch1")
    raw_b, raw_a = pcmm_level1(ctx, plan, X, *rp.raw(ctx))
    Y = ring_pack(ctx, rp, keys, raw_b, raw_a)
    got = u32(Y.data)[:, 0]
    s = O.keygen(P, 7)
    assert np.array_equal(s, sk.s.cpu().numpy())
    ref = O.mlwe_to_rlwe1(P, u32(raw_b), u32(raw_a), O.mlwe_ks_keys1(P, 9, s))
    assert np.array_equal(got, ref), f"{int((got != ref).sum())} words differ"
