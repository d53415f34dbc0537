"""Rhombus PCMv on the GPU vs the CPU oracle (he_oracle_pcmv.c / he_oracle_rhombus.c): every output
word bit-exact at toy size, on a mid ring, and at the BASELINE config-5 shapes (N = 2^16, n = 4096);
both split points (the default input/output-packing split and split 0); both multi-GPU shardings."""

import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200 import HeContext, HeParams
from paper_2601_18511_b200.errors import NeedsBootstrapError
from paper_2601_18511_b200.rhombus import (CtVector, clear_pcmv, decrypt_vector, encrypt_vector, make_rhombus_plan,
                                           pcmv_rhombus, rhombus_keygen, rhombus_window)

pytestmark = pytest.mark.gpu

MID = dict(mlwe_degree=32, mlwe_rank=256, rhombus_degree=512, name="mid")


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _setup(P, n_out, n_in, seed=0, split=None):
    ctx = HeContext(P, rng="seeded")
    rng = np.random.default_rng(seed)
    v = rng.uniform(-1, 1, n_in)
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    sk = ctx.keygen(7)
    keys = rhombus_keygen(ctx, sk, 99)
    x = encrypt_vector(ctx, sk, v, seed=5, split=split)
    return ctx, sk, keys, x, v, W


def _oracle_out(P, x, W, n_in, keys_o, window, piece0=0, level1=False):
    s_small, s_up, ksk, gal = keys_o
    return O.rhombus_pcmv_w(P, u32(x.data), ksk, gal, O.rhombus_weights(P, W), n_in, window, piece0, level1)


@pytest.mark.parametrize("split", [None, 0])
@pytest.mark.parametrize("n_out,n_in", [(200, 300), (512, 512), (64, 100), (130, 40)])
def test_toy_pcmv_bit_exact(n_out, n_in, split):
    P = HeParams.toy()
    ctx, sk, keys, x, v, W = _setup(P, n_out, n_in, split=split)
    s = O.keygen(P, 7)
    keys_o = O.rhombus_keys(P, 99, s)
    assert np.array_equal(keys.s_small.cpu().numpy(), keys_o[0])
    assert np.array_equal(keys.s_up.cpu().numpy(), keys_o[1])
    w = rhombus_window(P, n_in, split)
    assert x.window == w == O.rhombus_window(P, n_in, split)
    ct = O.encrypt(P, 5, s, O.encode_vector(P, v, w))[0]
    assert np.array_equal(u32(x.data), ct)                      # windowed input layout, device encryption
    plan = make_rhombus_plan(ctx, W, split=split)
    before = ctx.ledger.snapshot()
    y = pcmv_rhombus(ctx, plan, keys, x)
    diff = ctx.ledger.diff(before)
    p_out = -(-n_out // P.rhombus_degree)
    assert diff["rescales"] == 1 and diff["ct_rotations"] == (w - 1) * p_out == plan.key_switches()
    assert np.array_equal(u32(y.data)[0], _oracle_out(P, x, W, n_in, keys_o, w))
    if split == 0:  # the s = 0 windowed oracle is the original restatement (schoolbook-checked NTT product)
        _, out0 = O.rhombus_pcmv(P, ct, keys_o[2], keys_o[3], O.rhombus_weights(P, W), n_in)
        assert np.array_equal(u32(y.data)[0], out0)
    res = decrypt_vector(ctx, keys.s_up_ntt, y)
    err = np.abs(res - clear_pcmv(W, v)).max()
    assert err < 2 ** -14, err


@pytest.mark.parametrize("split", [None, 0, 1])
@pytest.mark.parametrize("n_out,n_in", [(1024, 8192), (700, 3000)])
def test_mid_ring_pcmv_bit_exact(n_out, n_in, split):
    """N = 8192 with the Llama primes, Rhombus degree n = 512: every output word vs the oracle."""
    P = HeParams(**MID)
    if split is not None and (P.rhombus_degree >> split) * P.rho < n_in:
        pytest.skip("split point too deep for this input")
    ctx, sk, keys, x, v, W = _setup(P, n_out, n_in, split=split)
    s = O.keygen(P, 7)
    keys_o = O.rhombus_keys(P, 99, s)
    w = rhombus_window(P, n_in, split)
    ct = O.encrypt(P, 5, s, O.encode_vector(P, v, w))[0]
    assert np.array_equal(u32(x.data), ct)
    y = pcmv_rhombus(ctx, make_rhombus_plan(ctx, W, split=split), keys, x)
    assert np.array_equal(u32(y.data)[0], _oracle_out(P, x, W, n_in, keys_o, w))
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
    with pytest.raises(ValueError, match="layout mismatch"):   # split-0 plan, default-window input
        pcmv_rhombus(ctx, make_rhombus_plan(ctx, W, split=0), keys, x)
    with pytest.raises(ValueError, match="dim mismatch"):      # window 16 x 4 pieces cannot hold 100 values
        make_rhombus_plan(ctx, np.zeros((8, 100)), split=3)
    with pytest.raises(NeedsBootstrapError):
        pcmv_rhombus(ctx, plan, keys, CtVector(x.data, 0, x.n_vals, window=x.window))
    with pytest.raises(ValueError, match="another HeContext"):
        pcmv_rhombus(HeContext(P, rng="seeded"), plan, keys, x)


@pytest.mark.parametrize("n_out,n_in,split", [(4096, 11008, None), (14336, 4096, None), (14336, 4096, 0)])
def test_llama_pcmv_bit_exact(n_out, n_in, split):
    """BASELINE config 5 at N' = 4096 (north_star: bit-exact PCMv on every Llama shape): every output
    word vs the oracle (OpenMP, host cores), plus the decrypted W v vs the float product."""
    P = HeParams.llama()
    ctx, sk, keys, x, v, W = _setup(P, n_out, n_in, seed=3, split=split)
    plan = make_rhombus_plan(ctx, W, split=split)
    y = pcmv_rhombus(ctx, plan, keys, x)
    res = decrypt_vector(ctx, keys.s_up_ntt, y)
    err = np.abs(res - clear_pcmv(W, v)).max()
    assert err < 2 ** -12, err
    s = O.keygen(P, 7)
    assert np.array_equal(sk.s.cpu().numpy(), s)
    keys_o = O.rhombus_keys(P, 99, s)
    w = rhombus_window(P, n_in, split)
    assert np.array_equal(u32(y.data)[0], _oracle_out(P, x, W, n_in, keys_o, w))


@pytest.mark.parametrize("params,n_out,n_in,strategy,world", [
    ("toy", 300, 200, "rows", 4),
    ("toy", 100, 300, "cols", 2),
    ("toy", 130, 40, "rows", 8),         # window 16: 2 leaves per rank and output piece
    ("mid", 1024, 3000, "rows", 3),      # 3 ranks: 2 leaf groups, rank 2 idle
    ("llama", 14336, 4096, "auto", 8),   # the paper's column split: 512 input values per rank
    ("llama", 4096, 11008, "auto", 8),   # the paper's row split (broadcast + split the matrix)
    ("llama", 4096, 4096, "auto", 8),
])
def test_sharded_pcmv_emulated_ranks(params, n_out, n_in, strategy, world):
    """§8e Rhombus sharding, every rank's work run on this one GPU: row shards
    (leaf-interleaved packing subtrees + a finish of the top levels) reproduce the one-GPU words
    exactly; column shards (a ciphertext sum) equal the oracle's sum of its column-shard outputs."""
    import torch

    from paper_2601_18511_b200.rhombus import (combine_rhombus_parts, finish_rhombus_subtrees, pcmv_rhombus_shard,
                                               pcmv_rhombus_subtree)
    from paper_2601_18511_b200.sharding import rhombus_shards

    P = {"toy": HeParams.toy, "mid": lambda: HeParams(**MID), "llama": HeParams.llama}[params]()
    ctx, sk, keys, x, v, W = _setup(P, n_out, n_in, seed=n_out)
    full = pcmv_rhombus(ctx, make_rhombus_plan(ctx, W), keys, x)
    slices = rhombus_shards(n_out, n_in, P.rhombus_degree, world, strategy, window=x.window)
    busy = sum(sl["active"] for sl in slices)
    if params == "llama":
        assert busy == world, "every rank gets work at the config-5 shapes"
    if slices[0]["strategy"] == "cols":
        parts = []
        for sl in slices:
            c0, c1 = sl["cols"]
            plan = make_rhombus_plan(ctx, W[:, c0:c1], window=x.window)
            parts.append(pcmv_rhombus_shard(ctx, plan, keys, x, sl["piece0"]))
        y = combine_rhombus_parts(ctx, torch.stack(parts), n_out)
        keys_o = O.rhombus_keys(P, 99, O.keygen(P, 7))
        parts_o = [_oracle_out(P, x, W[:, sl["cols"][0]:sl["cols"][1]], sl["cols"][1] - sl["cols"][0], keys_o,
                               x.window, sl["piece0"], level1=True) for sl in slices]
        for a, b in zip(parts, parts_o):
            assert np.array_equal(u32(a), b)
        assert np.array_equal(u32(y.data)[0], O.rhombus_combine(P, np.stack(parts_o)))
    else:
        G = slices[0]["groups"]
        plans = [make_rhombus_plan(ctx, W, groups=G, group=g) for g in range(G)]
        roots = torch.stack([pcmv_rhombus_subtree(ctx, pl, keys, x) for pl in plans])
        y = finish_rhombus_subtrees(ctx, plans[0], keys, roots)
        assert torch.equal(y.data, full.data)
    ref = clear_pcmv(W, v)
    err = np.abs(decrypt_vector(ctx, keys.s_up_ntt, y) - ref).max()
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
