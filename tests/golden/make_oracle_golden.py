"""Seeded integer fixtures of the CPU oracle (the integer pin of the path; parity with the
paper's HEaaN2 implementation is unpinned -- see DESIGN.md §3).

    python tests/golden/make_oracle_golden.py
Records, for the toy ring (N = 512, MLWE (32, 16)) and BASELINE config 1's 16 x 16 x 16
PCMM: the secret, the level-1 ciphertexts, the encoded weights W~ and the level-0 output
words of every row and column.  Tests compare both the oracle (regression) and the GPU
path (parity) against these words.
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import oracle as O
from paper_2601_18511_b200.params import HeParams


def main():
    P = HeParams.toy()
    g = np.load(HERE / "pcmm_toy_golden.npz")
    W, M = g["W"], g["M"]
    A = M.T.copy()                       # tokens x n_in (App. A orientation)
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    Wt = O.encode_weights(P, W)
    out = O.pcmm(P, Wt, ct)
    np.savez_compressed(HERE / "oracle_toy_int.npz", s=s, ct=ct, Wt=Wt, out=out,
                        moduli=np.array(P.moduli, dtype=np.int64))
    print("wrote oracle_toy_int.npz", out.shape)


if __name__ == "__main__":
    main()
