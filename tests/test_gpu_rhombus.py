"""Rhombus PCMv on the GPU vs the CPU oracle (he_oracle_rhombus.c): every output word
bit-exact at toy size; decrypted W v within the stated precision at Llama shapes."""

import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200 import HeContext, HeParams
from paper_2601_18511_b200.errors import NeedsBootstrapError
from paper_2601_18511_b200.rhombus import (CtVector, clear_pcmv, decrypt_vector, encrypt_vector, make_rhombus_plan,
                                           pcmv_rhombus, rhombus_keygen)

pytestmark = pytest.mark.gpu


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _setup(P, n_out, n_in, seed=0):
    ctx = HeContext(P)
    rng = np.random.default_rng(seed)
    v = rng.uniform(-1, 1, n_in)
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    sk = ctx.keygen(7)
    keys = rhombus_keygen(ctx, sk, 99)
    x = encrypt_vector(ctx, sk, v, seed=5)
    return ctx, sk, keys, x, v, W


@pytest.mark.parametrize("n_out,n_in", [(200, 300), (512, 512), (64, 100)])
def test_toy_pcmv_bit_exact(n_out, n_in):
    P = HeParams.toy()
    ctx, sk, keys, x, v, W = _setup(P, n_out, n_in)
    s = O.keygen(P, 7)
    s_small, s_up, ksk, gal = O.rhombus_keys(P, 99, s)
    assert np.array_equal(keys.s_small.cpu().numpy(), s_small)
    assert np.array_equal(keys.s_up.cpu().numpy(), s_up)
    ct = O.encrypt(P, 5, s, O.encode_vector(P, v))[0]
    assert np.array_equal(u32(x.data), ct)
    plan = make_rhombus_plan(ctx, W)
    before = ctx.ledger.snapshot()
    y = pcmv_rhombus(ctx, plan, keys, x)
    diff = ctx.ledger.diff(before)
    assert diff["rescales"] == 1 and diff["ct_rotations"] == (P.rhombus_degree - 1) * -(-n_out // P.rhombus_degree)
    _, out = O.rhombus_pcmv(P, ct, ksk, gal, O.rhombus_weights(P, W), n_in)
    assert np.array_equal(u32(y.data)[0], out)
    res = decrypt_vector(ctx, keys.s_up_ntt, y)
    err = np.abs(res - clear_pcmv(W, v)).max()
    assert err < 2 ** -14, err


@pytest.mark.parametrize("n_out,n_in", [(1024, 8192), (700, 3000)])
def test_mid_ring_pcmv_bit_exact(n_out, n_in):
    """N = 8192 with the Llama primes, Rhombus degree n = 512: 16 input pieces, 2 output pieces,
    511 Galois key switches per piece -- every output word vs the oracle."""
    P = HeParams(mlwe_degree=32, mlwe_rank=256, rhombus_degree=512, name="mid")
    ctx, sk, keys, x, v, W = _setup(P, n_out, n_in)
    s = O.keygen(P, 7)
    s_small, s_up, ksk, gal = O.rhombus_keys(P, 99, s)
    ct = O.encrypt(P, 5, s, O.encode_vector(P, v))[0]
    assert np.array_equal(u32(x.data), ct)
    y = pcmv_rhombus(ctx, make_rhombus_plan(ctx, W), keys, x)
    _, out = O.rhombus_pcmv(P, ct, ksk, gal, O.rhombus_weights(P, W), n_in)
    assert np.array_equal(u32(y.data)[0], out)
    err = np.abs(decrypt_vector(ctx, keys.s_up_ntt, y) - clear_pcmv(W, v)).max()
    assert err < 2 ** -12, err


def test_pcmv_errors():
    P = HeParams.toy()
    ctx, sk, keys, x, v, W = _setup(P, 32, 40)
    plan = make_rhombus_plan(ctx, W)
    with pytest.raises(TypeError):
        pcmv_rhombus(ctx, plan, keys, np.zeros(3))
    with pytest.raises(ValueError, match="dim mismatch"):
        pcmv_rhombus(ctx, make_rhombus_plan(ctx, np.zeros((32, 41))), keys, x)
    with pytest.raises(NeedsBootstrapError):
        pcmv_rhombus(ctx, plan, keys, CtVector(x.data, 0, x.n_vals))


@pytest.mark.parametrize("n_out,n_in", [(4096, 11008), (14336, 4096)])
def test_llama_pcmv_precision(n_out, n_in):
    """BASELINE config 5 shapes at N' = 4096: decrypted W v vs the float product."""
    P = HeParams.llama()
    ctx, sk, keys, x, v, W = _setup(P, n_out, n_in, seed=3)
    plan = make_rhombus_plan(ctx, W)
    y = pcmv_rhombus(ctx, plan, keys, x)
    res = decrypt_vector(ctx, keys.s_up_ntt, y)
    err = np.abs(res - clear_pcmv(W, v)).max()
    assert err < 2 ** -12, err


@pytest.mark.parametrize("params,n_out,n_in,strategy,world", [
    ("toy", 300, 200, "rows", 3),        # toy pieces are n = 128 elements
    ("toy", 100, 300, "cols", 2),
    ("llama", 8192, 4096, "rows", 2),
    ("llama", 14336, 4096, "rows", 3),
    ("llama", 4096, 11008, "cols", 3),
    ("llama", 4096, 11008, "auto", 8),   # 3 input pieces over 8 ranks: 5 idle ranks add zeros
])
def test_sharded_pcmv_emulated_ranks(params, n_out, n_in, strategy, world):
    """§8e Rhombus sharding, every rank's work run on this one GPU: row shards reproduce the
    one-GPU output words exactly; column shards (a ciphertext sum, different key-switching noise)
    decrypt to the same W v within the stated precision."""
    import torch

    from paper_2601_18511_b200.rhombus import combine_rhombus_parts, pcmv_rhombus_shard
    from paper_2601_18511_b200.sharding import rhombus_shards

    P = HeParams.toy() if params == "toy" else HeParams.llama()
    ctx, sk, keys, x, v, W = _setup(P, n_out, n_in, seed=n_out)
    full = pcmv_rhombus(ctx, make_rhombus_plan(ctx, W), keys, x)
    parts = []
    slices = rhombus_shards(n_out, n_in, P.rhombus_degree, world, strategy)
    for sl in slices:
        (r0, r1), (c0, c1) = sl["rows"], sl["cols"]
        if r1 > r0 and c1 > c0:
            parts.append(pcmv_rhombus_shard(ctx, make_rhombus_plan(ctx, W[r0:r1, c0:c1]), keys, x, sl["piece0"],
                                            sl["opiece0"]))
        else:
            parts.append(torch.zeros((2, 2, P.N), dtype=torch.int32, device=ctx.device))
    y = combine_rhombus_parts(ctx, torch.stack(parts), n_out)
    ref = clear_pcmv(W, v)
    res = decrypt_vector(ctx, keys.s_up_ntt, y)
    if slices[0]["strategy"] == "rows":
        assert torch.equal(y.data, full.data)
    else:
        full_res = decrypt_vector(ctx, keys.s_up_ntt, full)
        assert np.abs(res - full_res).max() < 2 ** -18
    err = np.abs(res - ref).max()
    assert err < np.abs(ref).max() * 2 ** -13, err


def test_graph_replay_same_words():
    """OpGraph: a captured PCMv replays to the same output words as the eager call."""
    import torch

    from paper_2601_18511_b200 import OpGraph

    P = HeParams.llama()
    ctx, sk, keys, x, v, W = _setup(P, 4096, 4096, seed=3)
    plan = make_rhombus_plan(ctx, W)
    ref = pcmv_rhombus(ctx, plan, keys, x).data.clone()
    g = OpGraph(lambda: pcmv_rhombus(ctx, plan, keys, x))
    g.result.data.zero_()
    y = g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y.data, ref)
