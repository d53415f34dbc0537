"""Parity of the CUDA path (through the C ABI) with the CPU oracle, on the GPU.

Both a'-column algorithms are covered: "spectral" (K7, the default: blockwise NTT
correlations + per-frequency tcgen05 GEMMs) and "direct" (K1 over all GEMM columns); they
must produce the same words, and each is checked against the oracle.

Bar: bit-exact on every integer ciphertext word (encryption, weight digits, PCMM output)
at toy size (all rows x all columns) and at Llama sizes (sampled rows x columns, plus the
exact selection-matrix identity over the FULL output); decrypted outputs within the
stated CKKS precision of the float product (>= 14 bits here, paper target 12 bits,
PAPER.md:477)."""

from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe
from paper_2601_18511_b200.errors import NeedsBootstrapError

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def gather(P, Y, rows, cols):
    out_a, out_b = u32(Y.out_a), u32(Y.out_b)
    d, k = P.mlwe_degree, P.mlwe_rank
    got = np.zeros((len(rows), len(cols)), np.uint32)
    for i, y in enumerate(rows):
        for j, n in enumerate(cols):
            got[i, j] = out_b[y // k, y % k + k * n] if n < d else out_a[y, n - d]
    return got


def setup(P, n_out, n_in, seed=0, scale=None):
    import torch

    ctx = HeContext(P, rng="seeded")
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / (np.sqrt(n_in) if scale is None else scale)
    sk = ctx.keygen(7)
    X = ctx.encrypt_acts(sk, A, seed=11)
    torch.cuda.synchronize()
    return ctx, sk, A, W, X


def test_fixture_parity_baseline_config1():
    """BASELINE config 1 (16x16x16 on the toy ring) against the committed integer fixture."""
    P = HeParams.toy()
    g = np.load(GOLD / "oracle_toy_int.npz")
    gt = np.load(GOLD / "pcmm_toy_golden.npz")
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    assert np.array_equal(sk.s.cpu().numpy(), g["s"])
    X = ctx.encrypt_acts(sk, gt["M"].T.copy(), seed=11)
    assert np.array_equal(u32(X.data), g["ct"])
    plan = make_mlwe_pcmm_plan(ctx, gt["W"])
    Y = pcmm_mlwe(ctx, plan, X)
    assert np.array_equal(gather(P, Y, range(16), range(P.width)), g["out"])
    dec = ctx.decrypt_pcmm(sk, Y)
    np.testing.assert_allclose(dec.T, gt["hesim_clear"], atol=2 ** -16)
    np.testing.assert_allclose(dec.T, gt["hesim_bsgs"], atol=2 ** -16)


ALGOS = ["spectral", "direct"]


def test_llama_ring_keygen_and_encryption_every_word():
    """N = 2^16: the device secret and every word of a fresh 4-ciphertext encryption (both limbs, a and b)
    equal the oracle's keygen / Ecd_coeff / or_encrypt on the same seeds (the words every Llama-shape PCMM
    check starts from)."""
    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (P.tokens, 4 * P.mlwe_rank))
    sk = ctx.keygen(7)
    s = O.keygen(P, 7)
    assert np.array_equal(sk.s.cpu().numpy(), s)
    X = ctx.encrypt_acts(sk, A, seed=11)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    assert ct.shape == tuple(X.data.shape)
    assert np.array_equal(u32(X.data), ct)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("n_out,n_in", [(16, 16), (48, 32), (256, 384), (128, 1024)])
def test_toy_all_words_bit_exact(n_out, n_in, algo):
    P = HeParams.toy()
    ctx, sk, A, W, X = setup(P, n_out, n_in)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    assert np.array_equal(u32(X.data), ct)
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    Wt = O.encode_weights(P, W)
    dg = plan.digits.cpu().numpy().astype(np.int64)
    assert np.array_equal(sum(dg[i] * 256 ** i for i in range(plan.d_w)), Wt)
    Y = pcmm_mlwe(ctx, plan, X)
    ref = O.pcmm(P, Wt, ct)
    assert np.array_equal(gather(P, Y, range(n_out), range(P.width)), ref)
    dec = ctx.decrypt_pcmm(sk, Y)
    err = np.abs(dec - A @ W.T).max()
    assert err < 2 ** -14, err


@pytest.mark.parametrize("algo", ALGOS)
def test_toy_wide_weights_use_more_digits(algo):
    P = HeParams.toy()
    ctx, sk, A, W, X = setup(P, 64, 64, scale=1.0)      # |W| up to 1 -> 3 weight digits
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    assert plan.d_w == 3
    plan4 = make_mlwe_pcmm_plan(ctx, W, d_w=4, algo=algo)
    ref = O.pcmm(P, O.encode_weights(P, W), u32(X.data))
    for pl in (plan, plan4):
        Y = pcmm_mlwe(ctx, pl, X)
        assert np.array_equal(gather(P, Y, range(64), range(P.width)), ref)


@pytest.mark.parametrize("algo", ALGOS)
def test_wide_params_four_digit_limbs(algo):
    P = HeParams.wide(mlwe_degree=32, mlwe_rank=16, moduli=(1073738753, 1073732609), rhombus_degree=128)
    ctx, sk, A, W, X = setup(P, 32, 48)
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    assert P.ct_digits(1) == 4
    Y = pcmm_mlwe(ctx, plan, X)
    ref = O.pcmm(P, O.encode_weights(P, W), O.encrypt(P, 11, O.keygen(P, 7), O.encode_acts(P, A)))
    assert np.array_equal(gather(P, Y, range(32), range(P.width)), ref)


def _llama_sample(P, n_out):
    rng = np.random.default_rng(5)
    rows = sorted(r for r in set([0, 1, 127, 128, 255, 256, n_out - 1] + list(rng.integers(0, n_out, 5))) if r < n_out)
    cols = sorted(set([0, 1, 255, 256, 257, 511, 512, 4095, P.width - 1] + list(rng.integers(0, P.width, 32))))
    return rows, cols


LLAMA_SHAPES = [(4096, 4096), (4096, 11008), (11008, 4096), (14336, 4096), (4096, 14336)]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("n_out,n_in", LLAMA_SHAPES)
def test_llama_sampled_words_bit_exact_and_precision(n_out, n_in, algo):
    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, n_out, n_in)
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    assert plan.d_w == 2
    Y = pcmm_mlwe(ctx, plan, X)
    rows, cols = _llama_sample(P, n_out)
    # oracle on the same device-made ciphertexts (their words are checked at toy size)
    ref = O.pcmm(P, O.encode_weights(P, W[:0 + n_out]), u32(X.data), rows=rows, cols=cols)
    assert np.array_equal(gather(P, Y, rows, cols), ref)
    dec = ctx.decrypt_pcmm(sk, Y, rows=(0, 256))
    err = np.nanmax(np.abs(dec - A @ W.T))
    assert err < 2 ** -12, err          # paper target 12 bits; measured ~14.5 bits


@pytest.mark.parametrize("n_out,n_in", LLAMA_SHAPES)
def test_llama_last_row_block_every_word(n_out, n_in):
    """Every word of the LAST 256-row output block (all 65 792 columns, b' and a') of each Llama-2-7B /
    Llama-3-8B projection shape on the default (spectral) path equals the oracle's exact BCHPS24 Alg. 2 on the
    same ciphertexts (the bench checks the FIRST block of the metric shape the same way)."""
    import torch

    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, n_out, n_in, seed=7)
    Y = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), X)
    torch.cuda.synchronize()
    k, d = P.mlwe_rank, P.mlwe_degree
    y0 = n_out - k
    ref = O.pcmm(P, O.encode_weights(P, W), u32(X.data), rows=list(range(y0, n_out)))
    got_a = u32(Y.out_a[y0:n_out])
    got_b = u32(Y.out_b[y0 // k])
    assert np.array_equal(got_a, ref[:, d:]), f"{int((got_a != ref[:, d:]).sum())} a' words differ"
    for t in range(k):
        assert np.array_equal(got_b[t + k * np.arange(d)], ref[t, :d]), f"b' row {y0 + t}"


@pytest.mark.parametrize("n_out,n_in", LLAMA_SHAPES)
def test_llama_full_output_every_word_vs_cpu_spectral_oracle(n_out, n_in):
    """EVERY word of the full output (all n_out rows x 65 792 columns, b' and a') of each Llama-2-7B / Llama-3-8B
    projection shape equals the CPU restatement oracle/he_oracle_spectral.c on the same ciphertexts -- itself
    pinned word for word to the direct BCHPS24 Alg. 2 oracle (tests/test_oracle.py, toy and Llama ring)."""
    import torch

    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, n_out, n_in, seed=5)
    Y = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), X)
    torch.cuda.synchronize()
    k, d = P.mlwe_rank, P.mlwe_degree
    ref = O.pcmm_spectral(P, O.encode_weights(P, W), u32(X.data))
    got_a = u32(Y.out_a)
    assert np.array_equal(got_a, ref[:, d:]), f"{int((got_a != ref[:, d:]).sum())} a' words differ"
    got_b = u32(Y.out_b).reshape(-1, P.N)
    ref_b = ref[:, :d].reshape(-1, k, d).transpose(0, 2, 1).reshape(-1, P.N)   # b'_(Y k + t)[m] at t + k m
    assert np.array_equal(got_b, ref_b), f"{int((got_b != ref_b).sum())} b' words differ"


@pytest.mark.parametrize("n_out,n_in", LLAMA_SHAPES)
def test_spectral_equals_direct_every_word(n_out, n_in):
    """The two a'-column algorithms agree on ALL n_out x 65 792 output words (random weights);
    the direct K1 words are themselves oracle-pinned on samples and by the selection identity."""
    import torch

    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, n_out, n_in, seed=3)
    ys = {}
    for algo in ALGOS:
        plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
        Y = pcmm_mlwe(ctx, plan, X)
        ys[algo] = (Y.out_a.clone(), Y.out_b.clone())
        del plan, Y
        torch.cuda.empty_cache()
    assert torch.equal(ys["spectral"][0], ys["direct"][0])
    assert torch.equal(ys["spectral"][1], ys["direct"][1])


def _selection_identity(n_out, n_in, seed=9, algo="spectral"):
    """W a 0/1 selection matrix (W~ = q1 at (y, pi(y))): the rescaled output row y equals, word
    for word, the limb-0 MLWE decomposition of input row pi(y) -- checked over ALL n_out x 65 792
    output words, a size-independent exact property."""
    import torch

    from paper_2601_18511_b200.layout import block_permutation

    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    sk = ctx.keygen(3)
    X = ctx.encrypt_acts(sk, A, seed=4)
    pi = rng.integers(0, n_in, n_out)
    # GEMM row y = k r' + t' reads W[k r' + sigma(t')]; GEMM col x reads W[:, k r + sigma(t)]
    prow = block_permutation(n_out, P.mlwe_rank)
    pcol = block_permutation(n_in, P.mlwe_rank)
    W = np.zeros((n_out, n_in))
    W[prow, pcol[pi]] = 1.0                   # GEMM-order W~[y][pi(y)] = q1
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    Y = pcmm_mlwe(ctx, plan, X)
    torch.cuda.synchronize()
    ct = X.data
    d, k, N, q0 = P.mlwe_degree, P.mlwe_rank, P.N, P.moduli[0]
    a0 = ct[:, 0, 0].to(torch.int64)                       # [n_ct, N]
    b0 = ct[:, 0, 1].to(torch.int64)
    j = torch.arange(k, device=ct.device).view(1, k, 1)
    m = torch.arange(d, device=ct.device).view(1, 1, d)
    for y0 in range(0, n_out, 2048):                       # expected a'[y][j][m] = a_r[t - j + k m] (negacyclic)
        y1 = min(n_out, y0 + 2048)
        x = torch.as_tensor(pi[y0:y1], device=ct.device)
        r, t = x // k, x % k
        c = t.view(-1, 1, 1) - j + k * m
        neg = c < 0
        av = a0[r.view(-1, 1, 1), torch.where(neg, c + N, c)]
        exp_a = torch.where(neg & (av != 0), q0 - av, av).view(y1 - y0, k * d)
        assert torch.equal(Y.out_a[y0:y1].to(torch.int64) & 0xFFFFFFFF, exp_a)
        del c, neg, av, exp_a
    x = torch.as_tensor(pi, device=ct.device)
    r, t = x // k, x % k
    mm = torch.arange(d, device=ct.device).view(1, d)
    bb = b0[r.view(-1, 1), t.view(-1, 1) + k * mm]        # [n_out, d]
    y = torch.arange(n_out, device=ct.device)
    got_b = (Y.out_b.to(torch.int64) & 0xFFFFFFFF)[(y // k).view(-1, 1), (y % k).view(-1, 1) + k * mm]
    assert torch.equal(got_b, bb)


@pytest.mark.parametrize("algo", ALGOS)
def test_selection_identity_full_output_metric_shape(algo):
    _selection_identity(4096, 11008, algo=algo)


@pytest.mark.parametrize("n_out,n_in", [s for s in LLAMA_SHAPES if s != (4096, 11008)])
def test_selection_identity_full_output_all_llama_shapes(n_out, n_in):
    _selection_identity(n_out, n_in)


@pytest.mark.parametrize("algo", ALGOS)
def test_wide_weights_at_llama_size_use_32_column_tiles(algo):
    """|W| up to 1 -> d_w = 3 at q1 ~ 2^20: the 256x32 CTA-pair instance, sampled parity."""
    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, 1024, 4096, scale=1.0)
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    assert plan.d_w == 3
    Y = pcmm_mlwe(ctx, plan, X)
    rows, cols = _llama_sample(P, 1024)
    ref = O.pcmm(P, O.encode_weights(P, W), u32(X.data), rows=rows, cols=cols)
    assert np.array_equal(gather(P, Y, rows, cols), ref)


def test_errors_and_ledger_on_device():
    P = HeParams.toy()
    ctx, sk, A, W, X = setup(P, 32, 32)
    plan = make_mlwe_pcmm_plan(ctx, W)
    before = ctx.ledger.snapshot()
    Y = pcmm_mlwe(ctx, plan, X)
    diff = ctx.ledger.diff(before)
    assert diff["rescales"] == 2 and diff["ct_rotations"] == 0 and diff["pc_mults"] == 4
    assert Y.level == X.level - 1 == 0
    from paper_2601_18511_b200.context import CtBlocks

    with pytest.raises(NeedsBootstrapError):
        pcmm_mlwe(ctx, plan, CtBlocks(X.data, 0, X.n_cols))
    with pytest.raises(TypeError):
        pcmm_mlwe(ctx, plan, Y)
    plan2 = make_mlwe_pcmm_plan(ctx, np.zeros((32, 48)))
    with pytest.raises(ValueError, match="dim mismatch"):
        pcmm_mlwe(ctx, plan2, X)
    # inputs are never mutated
    snap = X.data.clone()
    pcmm_mlwe(ctx, plan, X)
    assert bool((snap == X.data).all())


def test_ntt_roundtrip_and_product():
    import torch

    from paper_2601_18511_b200 import native

    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    rng = np.random.default_rng(1)
    for n in (P.N, P.rhombus_degree):
        for limb, q in enumerate(P.moduli):
            a = rng.integers(0, q, (3, n)).astype(np.uint32)
            t = torch.from_numpy(a.view(np.int32)).cuda()
            native.call("he_ntt_forward", ctx.handle, t.data_ptr(), n, limb, 3, n, ctx.stream())
            native.call("he_ntt_inverse", ctx.handle, t.data_ptr(), n, limb, 3, n, ctx.stream())
            assert np.array_equal(u32(t), a)


@pytest.mark.parametrize("algo", ALGOS)
def test_streamed_to_host_matches_device_output(algo):
    """pcmm_mlwe_to_host (row chunks streamed to pinned host memory) == pcmm_mlwe."""
    import torch

    from paper_2601_18511_b200 import pcmm_mlwe_to_host

    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, 1280, 512)
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    Y = pcmm_mlwe(ctx, plan, X)
    hb = torch.empty(tuple(Y.out_b.shape), dtype=torch.int32, pin_memory=True)
    ha = torch.empty(tuple(Y.out_a.shape), dtype=torch.int32, pin_memory=True)
    x_host = X.data.cpu().pin_memory()
    before = ctx.ledger.snapshot()
    pcmm_mlwe_to_host(ctx, plan, X, hb, ha, x_host=x_host, chunk_rows=512)
    torch.cuda.synchronize()
    assert ctx.ledger.diff(before)["rescales"] == 5
    assert torch.equal(ha, Y.out_a.cpu()) and torch.equal(hb, Y.out_b.cpu())


def test_spectral_transform_length_512_subprocess():
    """The L = 2k = 512 spectral variant (HE_SPEC_L=512, read once per process) produces the same
    words as the direct K1 path at a Llama shape -- run in a child process."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, torch, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import test_gpu_pcmm as G; from paper_2601_18511_b200 import HeParams, make_mlwe_pcmm_plan, pcmm_mlwe;"
        "P = HeParams.llama(); ctx, sk, A, W, X = G.setup(P, 1024, 4096, seed=4);"
        "ps = make_mlwe_pcmm_plan(ctx, W); assert ps.spectral_info()['L'] == 512;"
        "Y1 = pcmm_mlwe(ctx, ps, X); a1, b1 = Y1.out_a.clone(), Y1.out_b.clone();"
        "Y2 = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W, algo='direct'), X);"
        "assert torch.equal(a1, Y2.out_a) and torch.equal(b1, Y2.out_b); print('ok')"
    )
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, HE_SPEC_L="512")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("env", [{"HE_S4_RUNTIME_Q": "1"}, {"HE_S4_STRICT": "1"}])
def test_s4_variants_subprocess(env):
    """The S4 instantiations the Llama parameters do not select by default -- moduli as kernel parameters
    (HE_S4_RUNTIME_Q) and corrected q1 butterflies (HE_S4_STRICT) -- produce the default path's words, in both
    the rescaled and the level-1 output modes (read once per process: child process)."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, torch, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import test_gpu_pcmm as G; from paper_2601_18511_b200 import HeParams, make_mlwe_pcmm_plan, pcmm_mlwe;"
        "P = HeParams.llama(); ctx, sk, A, W, X = G.setup(P, 512, 2048, seed=6);"
        "Y1 = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), X);"
        "Y2 = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W, algo='direct'), X);"
        "assert torch.equal(Y1.out_a, Y2.out_a) and torch.equal(Y1.out_b, Y2.out_b);"
        "from paper_2601_18511_b200 import pcmm_level1;"
        "rb, ra = pcmm_level1(ctx, make_mlwe_pcmm_plan(ctx, W), X);"
        "rb2, ra2 = pcmm_level1(ctx, make_mlwe_pcmm_plan(ctx, W, algo='direct'), X);"
        "assert torch.equal(ra, ra2) and torch.equal(rb, rb2); print('ok')"
    )
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("algo", ALGOS)
def test_fused_peer_output_writes_every_destination(algo):
    """he_pcmm_gemm_rows_peers (the fused output all-gather): the shard's words land, identical to
    pcmm_mlwe's, in every one of several full-size destination buffers at rows dst_row0 + y; rows
    outside the shard are untouched.  (Two local buffers stand in for two ranks' peer memory.)"""
    import torch

    from paper_2601_18511_b200 import pcmm_mlwe_into_peers

    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, 512, 1024, seed=6)
    plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
    ref = pcmm_mlwe(ctx, plan, X)
    ref_a, ref_b = ref.out_a.clone(), ref.out_b.clone()
    n_full, row0, k = 1536, 768, P.mlwe_rank
    dst = [(torch.full((n_full // k, P.N), -7, dtype=torch.int32, device="cuda"),
            torch.full((n_full, P.N), -7, dtype=torch.int32, device="cuda")) for _ in range(2)]
    pcmm_mlwe_into_peers(ctx, plan, X, [b.data_ptr() for b, _ in dst], [a.data_ptr() for _, a in dst], row0)
    torch.cuda.synchronize()
    for b, a in dst:
        assert torch.equal(a[row0:row0 + 512], ref_a) and torch.equal(b[row0 // k:(row0 + 512) // k], ref_b)
        assert bool((a[:row0] == -7).all()) and bool((a[row0 + 512:] == -7).all())
        assert bool((b[:row0 // k] == -7).all()) and bool((b[(row0 + 512) // k:] == -7).all())


def test_fused_sharded_symmetric_memory_single_rank():
    """The symmetric-memory fused path degrades to None at world size 1 (plain local output)."""
    from paper_2601_18511_b200.sharding import symmetric_outputs

    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    assert symmetric_outputs(ctx, 512) is None


def test_plan_files_round_trip(tmp_path):
    """On-disk plan format (§8f 4): saved digit planes reload to a plan with the same output words;
    files made for other parameters or other formats are refused."""
    import torch

    from paper_2601_18511_b200 import load_mlwe_pcmm_plan, load_plan_bundle, save_mlwe_pcmm_plan, save_plan_bundle

    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, 512, 1024, seed=8)
    plan = make_mlwe_pcmm_plan(ctx, W)
    ref = pcmm_mlwe(ctx, plan, X)
    ra, rb = ref.out_a.clone(), ref.out_b.clone()
    save_mlwe_pcmm_plan(ctx, plan, tmp_path / "p.npz")
    for algo in (None, "direct"):
        p2 = load_mlwe_pcmm_plan(ctx, tmp_path / "p.npz", algo=algo)
        assert p2.algo == (algo or "spectral") and p2.shape == plan.shape and p2.d_w == plan.d_w
        Y = pcmm_mlwe(ctx, p2, X)
        torch.cuda.synchronize()
        assert torch.equal(Y.out_a, ra) and torch.equal(Y.out_b, rb)
    save_plan_bundle(ctx, {"layer0.down": plan}, tmp_path / "bundle")
    b = load_plan_bundle(ctx, tmp_path / "bundle")
    assert list(b) == ["layer0.down"] and torch.equal(pcmm_mlwe(ctx, b["layer0.down"], X).out_a, ra)
    with pytest.raises(ValueError):
        load_mlwe_pcmm_plan(HeContext(HeParams.toy(), rng="seeded"), tmp_path / "p.npz")


@pytest.mark.parametrize("algo", ALGOS)
def test_llama_minimal_and_zero_operands(algo):
    """Edge shapes at the Llama ring: one output block x one input ciphertext (n_out = n_in = k) checked
    word for word against the oracle; an all-zero weight matrix gives outputs that decrypt to 0 and a
    zero activation block decrypts to 0 (noise only)."""
    P = HeParams.llama()
    k = P.mlwe_rank
    ctx, sk, A, W, X = setup(P, k, k, seed=12)
    Y = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W, algo=algo), X)
    rows, cols = _llama_sample(P, k)
    rows = [r for r in rows if r < k]
    ref = O.pcmm(P, O.encode_weights(P, W), u32(X.data), rows=rows, cols=cols)
    assert np.array_equal(gather(P, Y, rows, cols), ref)
    Z = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, np.zeros_like(W), algo=algo), X)
    assert np.abs(ctx.decrypt_pcmm(sk, Z)).max() < 2 ** -20
    X0 = ctx.encrypt_acts(sk, np.zeros_like(A), seed=13)
    assert np.abs(ctx.decrypt_pcmm(sk, pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W, algo=algo), X0))).max() < 2 ** -14


@pytest.mark.parametrize("params", ["toy", "llama"])
def test_mlwe_decryption_matches_oracle_and_direct_kernel(params):
    """he_decrypt_mlwe (one NTT product per row through the RLWE view) gives the oracle's centred phases
    (or_decrypt_mlwe, the O(k d^2) definition) on every row checked."""
    import torch

    from paper_2601_18511_b200 import native

    P = HeParams.toy() if params == "toy" else HeParams.llama()
    n_out, n_in = (64, 48) if params == "toy" else (512, 1024)
    ctx, sk, A, W, X = setup(P, n_out, n_in, seed=21)
    Y = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), X)
    rows = list(range(n_out)) if params == "toy" else [0, 1, 255, 256, 300, 511]
    ph = torch.empty((n_out, P.mlwe_degree), dtype=torch.int64, device=ctx.device)
    native.call("he_decrypt_mlwe", ctx.handle, sk.s.data_ptr(), Y.out_b.data_ptr(), Y.out_a.data_ptr(), n_out, 0, n_out,
                ph.data_ptr(), ctx.stream())
    got = ph.cpu().numpy()
    d, k = P.mlwe_degree, P.mlwe_rank
    ob, oa = u32(Y.out_b), u32(Y.out_a)
    full = np.zeros((len(rows), P.width), np.uint32)
    for i, y in enumerate(rows):
        full[i, :d] = ob[y // k, y % k + k * np.arange(d)]
        full[i, d:] = oa[y]
    ref = O.decrypt_mlwe(P, sk.s.cpu().numpy(), full)
    assert np.array_equal(got[rows], ref)


@pytest.mark.parametrize("n_out,n_in", [(4096, 4096), (4096, 11008)])
def test_llama_headroom_log_delta_24(n_out, n_in):
    """Dynamic-range option: at the default Delta = 2^26 a level-0 output must stay below q0 / (2 Delta) = 8 in
    magnitude; HeParams.llama(log_delta=24) raises that bound to 32 (activations / outputs with outliers) at
    2 bits less precision.  Outputs up to |y| ~ 20 here: sampled words bit-exact vs the oracle and the decrypted
    product within 2^-10 relative to its range."""
    P = HeParams.llama(log_delta=24)
    ctx, sk, A, W, X = setup(P, n_out, n_in, scale=np.sqrt(n_in) / 10.0)   # 10x the default weights: |y| up to ~14
    plan = make_mlwe_pcmm_plan(ctx, W)
    Y = pcmm_mlwe(ctx, plan, X)
    rows, cols = _llama_sample(P, n_out)
    ref = O.pcmm(P, O.encode_weights(P, W), u32(X.data), rows=rows, cols=cols)
    assert np.array_equal(gather(P, Y, rows, cols), ref)
    dec = ctx.decrypt_pcmm(sk, Y, rows=(0, 256))
    exact = A @ W.T
    top = np.abs(exact[:, :256]).max()
    assert 8 < top < 32, top                         # beyond the default preset's range, inside this one's
    err = np.nanmax(np.abs(dec - exact))
    assert err / top < 2 ** -10, (err, top)


def test_llama_wide_input_two_k_blocks():
    """n_in = 72 x 256 (R = 72 > 64 input cts): the spectral GEMM's K spans two 64-byte blocks (G^ rows at the full
    128-byte padding, two TMA boxes per digit), sampled words bit-exact vs the oracle, spectral == direct."""
    P = HeParams.llama()
    ctx, sk, A, W, X = setup(P, 512, 72 * 256, seed=9)
    plan = make_mlwe_pcmm_plan(ctx, W)
    Y = pcmm_mlwe(ctx, plan, X)
    rows, cols = _llama_sample(P, 512)
    ref = O.pcmm(P, O.encode_weights(P, W), u32(X.data), rows=rows, cols=cols)
    assert np.array_equal(gather(P, Y, rows, cols), ref)
    Yd = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W, algo="direct"), X)
    assert np.array_equal(u32(Y.out_a), u32(Yd.out_a)) and np.array_equal(u32(Y.out_b), u32(Yd.out_b))
