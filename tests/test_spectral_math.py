"""CPU check of the K7 spectral formulation (he_spectral.cu) against the oracle's direct PCMM.

The a' columns of the MLWE PCMM are, per input ct r, length-k correlations of the weight segment
g_{y,r}[t] = W~[y][k r + t] with a_r, sampled at c = k m - j.  This test restates
the blockwise overlap-save evaluation in exact integer numpy (cyclic NTTs of length L over Z_q, blocks
of ob = L - k outputs) for both transform lengths the library uses (L = 2k and L = 4k) and checks
every a' word against oracle/ (the GEMM restatement) on the toy ring.  Test infrastructure only.
"""

import numpy as np
import pytest

import oracle as O
from paper_2601_18511_b200.params import HeParams


def _root(q, L):
    for g in range(2, q):
        w = pow(g, (q - 1) // L, q)
        if pow(w, L // 2, q) != 1:
            return w
    raise ValueError


def _dft(x, w, q):
    L = len(x)
    idx = np.arange(L)
    mat = np.array([[pow(w, int(f * i % L), q) for i in idx] for f in idx], dtype=object)
    return (mat.dot(np.asarray(x, dtype=object))) % q


@pytest.mark.parametrize("mult", [2, 4])
def test_blockwise_ntt_correlation_equals_oracle_pcmm(mult):
    P = HeParams.toy()
    d, k, N = P.mlwe_degree, P.mlwe_rank, P.N
    L, ob = mult * k, mult * k - k
    nblk = -(-N // ob)
    rng = np.random.default_rng(mult)
    n_out, n_in = 16, 32
    R = n_in // k
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    ct = O.encrypt(P, 11, O.keygen(P, 7), O.encode_acts(P, A))
    Wt = O.encode_weights(P, W)
    ref = O.pcmm(P, Wt, ct)[:, d:]                     # rescaled a' words, [n_out][k d]
    limbs = []
    for limb in range(2):
        q = P.moduli[limb]
        w = _root(q, L)
        wi = pow(w, q - 2, q)
        Linv = pow(L, q - 2, q)
        a = [ct[r, limb, 0].astype(object) for r in range(R)]

        def aread(r, i):
            if i < 0:
                return (-a[r][i + N]) % q
            if i >= N:
                return (-a[r][i - N]) % q
            return a[r][i]

        Ahat = [[_dft([aread(r, ob * b - k + 1 + u) for u in range(L)], w, q) for b in range(nblk)]
                for r in range(R)]
        out = np.zeros((n_out, N), dtype=object)
        for y in range(n_out):
            Ghat = []
            for r in range(R):
                g = [0] * L
                for t in range(k):
                    g[(-t) % L] = int(Wt[y, k * r + t]) % q
                Ghat.append(_dft(g, w, q))
            for b in range(nblk):
                C = sum(Ghat[r] * Ahat[r][b] for r in range(R)) % q
                c = _dft(C, wi, q) * Linv % q
                for u in range(ob):
                    cp = ob * b + u                    # c' = k m + (k - 1 - j)
                    if cp >= N:
                        break
                    m, j = cp // k, k - 1 - cp % k
                    out[y, d * j + m] = c[u]
        limbs.append(out)
    got = np.array([[O.rescale(P, int(limbs[0][y, n]), int(limbs[1][y, n])) for n in range(N)]
                    for y in range(n_out)], dtype=np.uint32)
    assert np.array_equal(got, ref)
