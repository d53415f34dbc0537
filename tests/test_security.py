"""Sampling security: contexts default to ChaCha20 sampling under a fresh 256-bit key with
fresh nonces; the seeded splitmix path is an explicit test mode.  The ChaCha20 block function the
device sampler uses is checked against RFC 8439's known answer and the `cryptography` package."""
import ctypes

import numpy as np
import pytest

from paper_2601_18511_b200 import HeContext, HeParams, native


def _block(key: bytes, counter: int, nonce: bytes) -> bytes:
    out = ctypes.create_string_buffer(64)
    native.call("he_chacha20_block", key, counter, nonce, out)
    return out.raw


def test_chacha20_block_rfc8439_vector():
    """RFC 8439 §2.3.2: key 00..1f, counter 1, nonce 00 00 00 09 00 00 00 4a 00 00 00 00."""
    key = bytes(range(32))
    nonce = bytes.fromhex("000000090000004a00000000")
    want = bytes.fromhex(
        "10f1e7e4d13b5915500fdd1fa32071c4c7d1f4c733c068030422aa9ac3d46c4e"
        "d2826446079faa0914c2d705d98b02a2b5129cd1de164eb9cbd083e8a2503c4e")
    assert _block(key, 1, nonce) == want


def test_chacha20_block_matches_cryptography():
    cryptography = pytest.importorskip("cryptography.hazmat.primitives.ciphers")
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms

    rng = np.random.default_rng(1)
    for counter in (0, 7, 0xFFFFFFFF):
        key = rng.bytes(32)
        nonce = rng.bytes(12)
        enc = Cipher(algorithms.ChaCha20(key, counter.to_bytes(4, "little") + nonce), mode=None).encryptor()
        assert _block(key, counter, nonce) == enc.update(bytes(64))


def test_rng_modes_are_explicit():
    with pytest.raises(ValueError):
        HeContext(HeParams.toy(), rng="fast")
    ctx = HeContext(HeParams.toy(), rng="seeded")
    with pytest.raises(ValueError, match="explicit seeds"):
        ctx.nonce(None)
    sec = HeContext(HeParams.toy())
    assert sec.rng == "secure"
    a, b = sec.nonce(None), sec.nonce(None)
    assert a != b and sec.nonce(5) == 5


@pytest.mark.gpu
def test_secure_context_round_trips_and_never_repeats_masks():
    from paper_2601_18511_b200 import (clear_pcmm, clear_pcmv, decrypt_vector, encrypt_vector, make_mlwe_pcmm_plan,
                                       make_rhombus_plan, pcmm_mlwe, pcmv_rhombus, rhombus_keygen)

    P = HeParams.toy()
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (P.tokens, 32))
    W = rng.uniform(-1, 1, (32, 32)) / 8
    sec = HeContext(P)
    det = HeContext(P, rng="seeded")
    sk_s, sk_d = sec.keygen(7), det.keygen(7)
    assert not np.array_equal(sk_s.s.cpu().numpy(), sk_d.s.cpu().numpy())   # same seed, keyed ChaCha20 differs
    s = sk_s.s.cpu().numpy()
    assert set(np.unique(s)) <= {-1, 0, 1} and 0.45 < np.mean(s == 0) < 0.55   # ternary, P(0) = 1/2
    X1, X2 = sec.encrypt_acts(sk_s, A), sec.encrypt_acts(sk_s, A)            # fresh nonces
    assert not np.array_equal(X1.data.cpu().numpy(), X2.data.cpu().numpy())
    Y = pcmm_mlwe(sec, make_mlwe_pcmm_plan(sec, W), X1)
    assert np.abs(sec.decrypt_pcmm(sk_s, Y) - clear_pcmm(W, A)).max() < 2 ** -14
    v = rng.uniform(-1, 1, 100)
    Wv = rng.uniform(-1, 1, (64, 100)) / 10
    keys = rhombus_keygen(sec, sk_s)
    y = pcmv_rhombus(sec, make_rhombus_plan(sec, Wv), keys, encrypt_vector(sec, sk_s, v))
    assert np.abs(decrypt_vector(sec, keys.s_up_ntt, y) - clear_pcmv(Wv, v)).max() < 2 ** -13
