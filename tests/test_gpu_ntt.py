"""K2 NTT / INTT against a numpy restatement of the merged-twiddle Cooley-Tukey / Gentleman-Sande pair
(the order oracle/he_oracle.c ntt_fwd / ntt_inv produce: natural -> bit-reversed, and back scaled by
n^-1), on every ring degree the path uses -- including the single-launch 2^16 kernels."""
import numpy as np
import pytest
import torch

from paper_2601_18511_b200 import HeContext, HeParams, native

pytestmark = pytest.mark.gpu


def _psi(q, n):
    for g in range(2, q):
        c = pow(g, (q - 1) // (2 * n), q)
        if pow(c, n, q) == q - 1:
            return c
    raise ValueError


def _tables(q, n):
    psi = _psi(q, n)
    lg = n.bit_length() - 1
    br = np.array([int(format(i, f"0{lg}b")[::-1], 2) for i in range(n)]) if lg else np.zeros(1, int)
    pw = np.array([pow(psi, int(e), q) for e in range(n)], dtype=object)
    pwi = np.array([pow(pow(psi, q - 2, q), int(e), q) for e in range(n)], dtype=object)
    return pw[br].astype(np.int64), pwi[br].astype(np.int64)


def ntt_ref(x, q, fw):
    a = x.astype(np.int64).copy()
    n = a.shape[-1]
    t, m = n, 1
    while m < n:
        t //= 2
        a = a.reshape(*a.shape[:-1], m, 2, t)
        w = fw[m:2 * m].reshape(m, 1)
        u, v = a[..., 0, :], a[..., 1, :] * w % q
        a = np.stack([(u + v) % q, (u - v) % q], axis=-2).reshape(*x.shape)
        m *= 2
    return a


@pytest.mark.parametrize("n,count", [(65536, 3), (4096, 5), (8192, 2)])
@pytest.mark.parametrize("limb", [0, 1])
def test_ntt_matches_restatement(n, count, limb):
    P = HeParams.llama() if n in (65536, 4096) else HeParams(mlwe_degree=32, mlwe_rank=256, rhombus_degree=512)
    ctx = HeContext(P, rng="seeded")
    q = P.moduli[limb]
    rng = np.random.default_rng(n + limb)
    x = rng.integers(0, q, (count, n), dtype=np.int64)
    dev = torch.from_numpy(x.astype(np.int32)).cuda()
    st = ctx.stream()
    native.call("he_ntt_forward", ctx.handle, dev.data_ptr(), n, limb, count, n, st)
    fw, _ = _tables(q, n)
    got = dev.cpu().numpy().astype(np.int64) & 0xFFFFFFFF
    assert np.array_equal(got, ntt_ref(x, q, fw))
    native.call("he_ntt_inverse", ctx.handle, dev.data_ptr(), n, limb, count, n, st)
    assert np.array_equal(dev.cpu().numpy().astype(np.int64) & 0xFFFFFFFF, x)


def test_ntt_strided_batch():
    """Polys spaced `stride` words apart (ciphertext slots), the layout the encryptor and key switches use."""
    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    q, n = P.moduli[0], P.N
    rng = np.random.default_rng(9)
    buf = rng.integers(0, q, (3, 2, n), dtype=np.int64)
    dev = torch.from_numpy(buf.astype(np.int32)).cuda()
    native.call("he_ntt_forward", ctx.handle, dev.data_ptr(), n, 0, 3, 2 * n, ctx.stream())
    got = dev.cpu().numpy().astype(np.int64) & 0xFFFFFFFF
    fw, _ = _tables(q, n)
    assert np.array_equal(got[:, 0], ntt_ref(buf[:, 0], q, fw))
    assert np.array_equal(got[:, 1], buf[:, 1])   # untouched
