"""The MLWE PCMM at the reference's plug-in point: hesim's chunked prefill with every
projection of the private chunk computed by the GPU PCMM on ciphertexts (toy ring: 16-row activation
blocks, k = 16) matches the reference's own float prefill (golden file from hesim)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2601_18511_b200 import HeContext, HeParams
from paper_2601_18511_b200.prefill import ToyConfig, chunked_prefill, make_projection_plans, make_weights

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).parent / "golden" / "prefill_golden.npz")


@pytest.mark.parametrize("algo", ["spectral", "direct"])
@pytest.mark.parametrize("name", ["toy", "toy2"])
def test_encrypted_projection_prefill_matches_hesim(name, algo):
    d_model, d_head, n_heads, d_ff, n_layers, seed, ptok = (int(v) for v in G[name + "_cfg"])
    cfg = ToyConfig(d_model, d_head, n_heads, d_ff, n_layers, seed)
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(5)
    layers, _ = make_weights(cfg)
    proj = make_projection_plans(ctx, layers, algo=algo)
    before = ctx.ledger.snapshot()
    logits, cache = chunked_prefill(G[name + "_tokens"], ptok, cfg, ctx, sk, proj)
    assert proj.calls == 7 * n_layers
    assert ctx.ledger.diff(before)["rescales"] > 0
    ref = G[name + "_logits"]
    assert np.abs(logits - ref).max() < 1e-3 * max(1.0, np.abs(ref).max())
    for li in range(n_layers):
        assert np.abs(cache.k[li] - G[f"{name}_k{li}"]).max() < 1e-3
        assert np.abs(cache.v[li] - G[f"{name}_v{li}"]).max() < 1e-3


@pytest.mark.parametrize("name", ["toy", "toy2"])
def test_encrypted_decode_step_rhombus_matches_hesim(name):
    """Generation: the new token's seven projections through the GPU Rhombus PCMv (encrypted vector ->
    PCMv -> decrypt under s'(X^rho)), against hesim's decode_step after its chunked prefill."""
    from paper_2601_18511_b200.prefill import decode_step, make_vector_projection_plans

    d_model, d_head, n_heads, d_ff, n_layers, seed, ptok = (int(v) for v in G[name + "_cfg"])
    cfg = ToyConfig(d_model, d_head, n_heads, d_ff, n_layers, seed)
    _, cache = chunked_prefill(G[name + "_tokens"], ptok, cfg)
    P = HeParams.toy()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(5)
    layers, _ = make_weights(cfg)
    proj = make_vector_projection_plans(ctx, sk, layers)
    logits, _ = decode_step(cache, G[name + "_next"], cfg, ctx, sk, proj)
    assert proj.calls == 7 * n_layers
    ref = G[name + "_decode_logits"]
    assert np.abs(logits - ref).max() < 1e-3 * max(1.0, np.abs(ref).max())
