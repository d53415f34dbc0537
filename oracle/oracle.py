"""ctypes front end of the C oracle (he_oracle.c) plus a pure-Python restatement
for the toy ring.  Test infrastructure only -- see package docstring."""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from pathlib import Path

import numpy as np

__all__ = [
    "lib", "build", "keygen", "encode_acts", "decode_acts", "encrypt", "decrypt_rlwe",
    "encode_weights", "pcmm", "pcmm_spectral", "pcmm_limb", "decrypt_mlwe", "decode_mlwe_rows", "rescale",
    "negacyclic_mul", "negacyclic_mul_schoolbook", "sigma_table", "clear_pcmm", "mlwe_column",
    "py_mlwe_components", "py_pcmm_rows", "num_threads", "time_pcmm_sample", "rng",
    "stream_a", "stream_e", "STREAM_SECRET", "half_reverse", "rhombus_keys", "keyswitch", "encode_vector",
    "decode_vector", "rhombus_pcmv", "rhombus_pcmv_w", "rhombus_combine", "rhombus_window", "rhombus_weights", "decrypt_under", "ring_pack_keys", "ring_pack_leaves",
    "ring_pack", "pcmm_ring_pack", "mlwe_ks_keys", "raw_device_layout", "mlwe_to_rlwe", "mlwe_ks_keys1",
    "mlwe_to_rlwe1", "ring_pack_special2", "rotation_keys", "slot_pcmm",
    "slot_bsgs", "rotation_keys_plain", "chain_rotation_keys", "chain_bsgs", "chain_key_id",
]

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "_build" / "libhe_oracle.so"
_lib = None

STREAM_SECRET = 0x5EC0000000000000


def stream_a(r: int, limb: int) -> int:
    return 0xA000000000000000 | (r << 8) | limb


def stream_e(r: int) -> int:
    return 0xE000000000000000 | (r << 8)


def build(force: bool = False) -> Path:
    srcs = [_HERE / "he_oracle.c", _HERE / "he_oracle_rhombus.c", _HERE / "he_oracle_pcmv.c", _HERE / "he_oracle_chain.c",
            _HERE / "he_oracle_spectral.c"]
    if force or not _SO.exists() or any(_SO.stat().st_mtime < s.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        L = ctypes.CDLL(str(_SO))
        u32p = ctypes.POINTER(ctypes.c_uint32)
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        f64p = ctypes.POINTER(ctypes.c_double)
        u32, u64, i64 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64
        sig = {
            "or_rng": (u64, [u64, u64, u64]),
            "or_keygen": (None, [u64, u32, i32p]),
            "or_encode_acts": (None, [f64p, u32, u32, u32, ctypes.c_double, i64p]),
            "or_decode_acts": (None, [i64p, u32, u32, u32, ctypes.c_double, f64p]),
            "or_encrypt": (ctypes.c_int, [u64, u32, u32, u32p, i32p, i64p, u32, u32, u32p]),
            "or_decrypt_rlwe": (ctypes.c_int, [u32p, u32p, i32p, u32, u32, i64p]),
            "or_encode_weights": (None, [f64p, u32, u32, u32, ctypes.c_double, i64p]),
            "or_pcmm": (ctypes.c_int, [u32, u32, u32p, i64p, u32, u32, u32p, i32p, u32, i32p, u32, u32p]),
            "or_pcmm_limb": (ctypes.c_int, [u32, u32, u32, u32, u32, i64p, u32, u32, u32p, i32p, u32, i32p, u32, u32p]),
            "or_decrypt_mlwe": (None, [u32, u32, u32, i32p, u32p, u32, i64p]),
            "or_rescale": (u32, [u32, u32, u32, u32]),
            "or_negacyclic_mul": (ctypes.c_int, [u32p, i32p, u32, u32, u32p]),
            "or_negacyclic_mul_schoolbook": (None, [u32p, i32p, u32, u32, u32p]),
            "or_sigma": (u32, [u32, u32]),
            "or_mlwe_column": (None, [u32p, u32, u32, u32, u32, u32, u32, u32, u32p]),
            "or_num_threads": (ctypes.c_int, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _u32(a):
    return _p(a, ctypes.c_uint32)


def _i32(a):
    return _p(a, ctypes.c_int32)


def _i64(a):
    return _p(a, ctypes.c_int64)


def _f64(a):
    return _p(a, ctypes.c_double)


def _moduli(params) -> np.ndarray:
    return np.ascontiguousarray(np.array(params.moduli, dtype=np.uint32))


def num_threads() -> int:
    return int(lib().or_num_threads())


def rng(seed: int, stream: int, idx: int) -> int:
    return int(lib().or_rng(seed, stream, idx))


def sigma_table(k: int) -> np.ndarray:
    return np.array([lib().or_sigma(t, k) for t in range(k)], dtype=np.int64)


def keygen(params, seed: int) -> np.ndarray:
    s = np.zeros(params.N, dtype=np.int32)
    lib().or_keygen(seed, params.N, _i32(s))
    return s


def encode_acts(params, A: np.ndarray) -> np.ndarray:
    """A: tokens x n_in (tokens = d/2) -> integer plaintext polys [n_in/k, N]."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    tokens, n_in = A.shape
    if tokens != params.tokens or n_in % params.mlwe_rank:
        raise ValueError("activation block shape mismatch")
    pt = np.zeros((n_in // params.mlwe_rank, params.N), dtype=np.int64)
    lib().or_encode_acts(_f64(A), n_in, params.mlwe_degree, params.mlwe_rank, params.delta, _i64(pt))
    return pt


def decode_acts(params, phase: np.ndarray, n_cols: int) -> np.ndarray:
    phase = np.ascontiguousarray(phase, dtype=np.int64)
    A = np.zeros((params.tokens, n_cols), dtype=np.float64)
    lib().or_decode_acts(_i64(phase), n_cols, params.mlwe_degree, params.mlwe_rank, params.delta, _f64(A))
    return A


def encrypt(params, seed: int, s: np.ndarray, pt: np.ndarray, r0: int = 0, level: int = 1) -> np.ndarray:
    """-> uint32 [n_ct, limbs = level + 1, 2 (a, b), N]"""
    pt = np.ascontiguousarray(pt, dtype=np.int64)
    n_ct = pt.shape[0]
    ct = np.zeros((n_ct, level + 1, 2, params.N), dtype=np.uint32)
    rc = lib().or_encrypt(seed, params.N, level + 1, _u32(_moduli(params)), _i32(np.ascontiguousarray(s)),
                          _i64(pt), n_ct, r0, _u32(ct))
    if rc:
        raise RuntimeError("oracle encrypt failed")
    return ct


def decrypt_rlwe(params, ct: np.ndarray, s: np.ndarray, limb: int = 0) -> np.ndarray:
    ct = np.ascontiguousarray(ct)
    out = np.zeros((ct.shape[0], params.N), dtype=np.int64)
    s = np.ascontiguousarray(s, dtype=np.int32)
    for r in range(ct.shape[0]):
        a = np.ascontiguousarray(ct[r, limb, 0])
        b = np.ascontiguousarray(ct[r, limb, 1])
        row = np.zeros(params.N, dtype=np.int64)
        lib().or_decrypt_rlwe(_u32(a), _u32(b), _i32(s), params.N, params.moduli[limb], _i64(row))
        out[r] = row
    return out


def encode_weights(params, W: np.ndarray) -> np.ndarray:
    W = np.ascontiguousarray(W, dtype=np.float64)
    n_out, n_in = W.shape
    Wt = np.zeros((n_out, n_in), dtype=np.int64)
    lib().or_encode_weights(_f64(W), n_out, n_in, params.mlwe_rank, float(params.delta_w), _i64(Wt))
    return Wt


def _sel(idx):
    if idx is None:
        return None, 0
    a = np.ascontiguousarray(np.asarray(idx, dtype=np.int32))
    return a, len(a)


def pcmm(params, Wt: np.ndarray, ct: np.ndarray, rows=None, cols=None) -> np.ndarray:
    """Rescaled level-0 output words (limb q0) for selected rows x GEMM columns."""
    Wt = np.ascontiguousarray(Wt, dtype=np.int64)
    ct = np.ascontiguousarray(ct, dtype=np.uint32)
    n_out, n_in = Wt.shape
    r, nr = _sel(rows)
    c, nc = _sel(cols)
    nr = nr if r is not None else n_out
    nc = nc if c is not None else params.width
    out = np.zeros((nr, nc), dtype=np.uint32)
    lib().or_pcmm(params.mlwe_degree, params.mlwe_rank, _u32(_moduli(params)), _i64(Wt), n_out, n_in,
                  _u32(ct), _i32(r) if r is not None else None, nr, _i32(c) if c is not None else None, nc,
                  _u32(out))
    return out


def pcmm_spectral(params, Wt: np.ndarray, ct: np.ndarray, row0: int = 0, n_rows=None, L=None) -> np.ndarray:
    """Rescaled level-0 output rows [row0, row0 + n_rows) x all columns (the `pcmm` layout), computed by the
    spectral restatement (he_oracle_spectral.c: overlap-save correlations, L = 4k by default) -- the same words
    as `pcmm`, fast enough for every row of a Llama shape."""
    Wt = np.ascontiguousarray(Wt, dtype=np.int64)
    ct = np.ascontiguousarray(ct, dtype=np.uint32)
    n_out, n_in = Wt.shape
    n_rows = n_out - row0 if n_rows is None else n_rows
    L = 4 * params.mlwe_rank if L is None else L
    out = np.zeros((n_rows, params.width), dtype=np.uint32)
    L_ = lib()
    if not getattr(L_, "_sp_bound", False):
        u32p, i64p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int64)
        u32 = ctypes.c_uint32
        L_.or_pcmm_spectral.restype = ctypes.c_int
        L_.or_pcmm_spectral.argtypes = [u32, u32, u32p, i64p, u32, u32, u32p, u32, u32, u32, u32p]
        L_._sp_bound = True
    rc = L_.or_pcmm_spectral(params.mlwe_degree, params.mlwe_rank, _u32(_moduli(params)), _i64(Wt), n_out, n_in,
                             _u32(ct), row0, n_rows, L, _u32(out))
    if rc != 0:
        raise ValueError("or_pcmm_spectral: unsupported parameters")
    return out


def pcmm_limb(params, Wt, ct, limb: int, rows=None, cols=None) -> np.ndarray:
    Wt = np.ascontiguousarray(Wt, dtype=np.int64)
    ct = np.ascontiguousarray(ct, dtype=np.uint32)
    n_out, n_in = Wt.shape
    r, nr = _sel(rows)
    c, nc = _sel(cols)
    nr = nr if r is not None else n_out
    nc = nc if c is not None else params.width
    out = np.zeros((nr, nc), dtype=np.uint32)
    lib().or_pcmm_limb(params.mlwe_degree, params.mlwe_rank, params.moduli[limb], ct.shape[1], limb,
                       _i64(Wt), n_out, n_in, _u32(ct), _i32(r) if r is not None else None, nr,
                       _i32(c) if c is not None else None, nc, _u32(out))
    return out


def mlwe_column(params, ct, limb: int, n: int) -> np.ndarray:
    ct = np.ascontiguousarray(ct, dtype=np.uint32)
    col = np.zeros(ct.shape[0] * params.mlwe_rank, dtype=np.uint32)
    lib().or_mlwe_column(_u32(ct), ct.shape[0], ct.shape[1], limb, params.mlwe_degree, params.mlwe_rank,
                         params.moduli[limb], n, _u32(col))
    return col


def decrypt_mlwe(params, s: np.ndarray, rows_out: np.ndarray) -> np.ndarray:
    """rows_out: n_rows x width (b' first).  -> centred phases n_rows x d."""
    rows_out = np.ascontiguousarray(rows_out, dtype=np.uint32)
    ph = np.zeros((rows_out.shape[0], params.mlwe_degree), dtype=np.int64)
    lib().or_decrypt_mlwe(params.mlwe_degree, params.mlwe_rank, params.moduli[0],
                          _i32(np.ascontiguousarray(s, dtype=np.int32)), _u32(rows_out), rows_out.shape[0],
                          _i64(ph))
    return ph


def decode_mlwe_rows(params, phase: np.ndarray, rows) -> dict:
    """Map MLWE output rows y (component t' of block r') to (token, out_col) values:
    phase_y[m] = Delta * Out[bitReverse(m)][k r' + sigma(t')] (App. A layout)."""
    d, k = params.mlwe_degree, params.mlwe_rank
    half = d // 2
    sig = sigma_table(k)
    lh = half.bit_length() - 1
    br = np.array([int(format(m, f"0{lh}b")[::-1], 2) if lh else 0 for m in range(half)])
    vals = {}
    for i, y in enumerate(rows):
        col = (y // k) * k + int(sig[y % k])
        vals[col] = (br, phase[i, :half] / params.delta)
    return vals


def rescale(params, x0: int, x1: int) -> int:
    return int(lib().or_rescale(x0, x1, params.moduli[0], params.moduli[1]))


def negacyclic_mul(a: np.ndarray, s: np.ndarray, q: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    out = np.zeros(len(a), dtype=np.uint32)
    if lib().or_negacyclic_mul(_u32(a), _i32(s), len(a), q, _u32(out)):
        raise ValueError("q is not NTT-friendly for this N")
    return out


def negacyclic_mul_schoolbook(a, s, q) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    out = np.zeros(len(a), dtype=np.uint32)
    lib().or_negacyclic_mul_schoolbook(_u32(a), _i32(s), len(a), q, _u32(out))
    return out


def clear_pcmm(W: np.ndarray, A: np.ndarray) -> np.ndarray:
    """Float oracle in the activation orientation: A (tokens x n_in) -> A @ W^T
    (tokens x n_out), i.e. (W @ M)^T with M = A^T -- hesim.clear_pcmm(W, M, 0)^T
    (matmul.py:179-181 with shear power 0)."""
    return np.asarray(A, float) @ np.asarray(W, float).T


# ---------------------------------------------------------------- pure-Python restatement (toy)

def py_mlwe_components(params, a: list[int], q: int):
    """Explicit RLWE->MLWE a-part from SURVEY.md App. B.2, written in the branchy
    form (j <= t: a_{t-j};  j > t: Y * a_{t-j+k}) -- independent of the C oracle's
    unified negacyclic index.  Returns at[t][j] = list of d coefficients."""
    d, k = params.mlwe_degree, params.mlwe_rank
    comp = [[a[t + k * m] for m in range(d)] for t in range(k)]  # a_t(Y)
    at = []
    for t in range(k):
        row = []
        for j in range(k):
            if j <= t:
                row.append(list(comp[t - j]))
            else:
                p = comp[t - j + k]
                row.append([(-p[d - 1]) % q] + p[: d - 1])  # Y * p in Z_q[Y]/(Y^d+1)
        at.append(row)
    return at


def py_pcmm_rows(params, Wt, ct, rows):
    """Pure-Python MLWE PCMM for a few rows (toy sizes): returns rows x width words."""
    d, k, N = params.mlwe_degree, params.mlwe_rank, params.N
    q0, q1 = params.moduli[:2]
    n_ct = ct.shape[0]
    per_limb = []
    for limb, q in enumerate((q0, q1)):
        cols = []  # MLWE ciphertexts x = (r, t): [b (d) | a (k*d)]
        for r in range(n_ct):
            a = [int(v) for v in ct[r, limb, 0]]
            b = [int(v) for v in ct[r, limb, 1]]
            at = py_mlwe_components(params, a, q)
            for t in range(k):
                vec = [b[t + k * m] for m in range(d)]
                for j in range(k):
                    vec.extend(at[t][j])
                cols.append(vec)
        res = []
        for y in rows:
            w = [int(v) for v in Wt[y]]
            res.append([sum(w[x] * cols[x][n] for x in range(len(cols))) % q for n in range(params.width)])
        per_limb.append(res)
    inv = pow(q1, q0 - 2, q0)
    out = []
    for i in range(len(rows)):
        row = []
        for n in range(params.width):
            x0, x1 = per_limb[0][i][n], per_limb[1][i][n]
            x1c = x1 - q1 if x1 > q1 // 2 else x1
            row.append((x0 - x1c) % q0 * inv % q0)
        out.append(row)
    return np.array(out, dtype=np.uint32)


# ---------------------------------------------------------------- CPU baseline timing

def time_pcmm_sample(params, Wt, ct, n_rows: int) -> dict:
    """Time the oracle PCMM on the first n_rows output rows x all columns x full K,
    both limbs + rescale (the sample the cpu_baseline is extrapolated from)."""
    rows = list(range(n_rows))
    t0 = time.perf_counter()
    out = pcmm(params, Wt, ct, rows=rows)
    dt = time.perf_counter() - t0
    return {"seconds": dt, "rows": n_rows, "threads": num_threads(), "words": out}


# ---------------------------------------------------------------- Rhombus PCMv (he_oracle_rhombus.c)
def _rh_lib():
    L = lib()
    if not getattr(L, "_rh_bound", False):
        u32p, i32p, i64p, f64p = (ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32),
                                  ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double))
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        sig = {
            "or_half_reverse": (u32, [u32, u32]),
            "or_automorphism": (None, [u32p, u32, u32, u32, u32p]),
            "or_ksk_gen": (None, [u64, u32, i32p, i32p, u32, u32p, u32p]),
            "or_keyswitch": (None, [u32p, u32p, u32, u32p, u32p, u32p]),
            "or_rhombus_secret": (None, [u64, u32, u32, i32p, i32p]),
            "or_galois_ksk": (None, [u64, u32, i32p, u32, u32p, u32p]),
            "or_rhombus_pcmv": (ctypes.c_int, [u32, u32, u32p, u32p, u32p, u32p, i64p, u32, u32, u32p, u32p]),
            "or_encode_vector": (None, [f64p, u32, u32, u32, ctypes.c_double, i64p]),
            "or_decode_vector": (None, [i64p, u32, u32, u32, ctypes.c_double, f64p]),
            "or_encode_vector_w": (None, [f64p, u32, u32, u32, u32, ctypes.c_double, i64p]),
            "or_window_reverse": (u32, [u32, u32]),
            "or_rhombus_pcmv_w": (ctypes.c_int, [u32, u32, u32, u32p, u32p, u32p, u32p, i64p, u32, u32, u32,
                                                 ctypes.c_int, u32p]),
            "or_rhombus_combine": (None, [u32p, u32, u32, u32p, u32p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        L._rh_bound = True
    return L


def half_reverse(x: int, n: int) -> int:
    return int(_rh_lib().or_half_reverse(x, n))


def rhombus_keys(params, seed: int, s: np.ndarray):
    """(s_small [n], s_up [N], ksk_dec [2,2,3,N], gal [log n, 2,2,3,n]) -- see he_oracle_rhombus.c."""
    L = _rh_lib()
    N, n = params.N, params.rhombus_degree
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    s_small = np.zeros(n, np.int32)
    s_up = np.zeros(N, np.int32)
    L.or_rhombus_secret(seed, n, N, _i32(s_small), _i32(s_up))
    ksk = np.zeros((2, 2, 3, N), np.uint32)
    L.or_ksk_gen(seed, 0, _i32(np.ascontiguousarray(s, dtype=np.int32)), _i32(s_up), N, _u32(m), _u32(ksk))
    lg = n.bit_length() - 1
    gal = np.zeros((lg, 2, 2, 3, n), np.uint32)
    for lv in range(1, lg + 1):
        g = np.zeros((2, 2, 3, n), np.uint32)
        L.or_galois_ksk(seed, lv, _i32(s_small), n, _u32(m), _u32(g))
        gal[lv - 1] = g
    return s_small, s_up, ksk, gal


def keyswitch(params, c: np.ndarray, ksk: np.ndarray, n: int):
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    c = np.ascontiguousarray(c, dtype=np.uint32)
    u = np.zeros((2, n), np.uint32)
    w = np.zeros((2, n), np.uint32)
    _rh_lib().or_keyswitch(_u32(c), _u32(np.ascontiguousarray(ksk)), n, _u32(m), _u32(u), _u32(w))
    return u, w


def rhombus_window(params, n_in: int, split=None) -> int:
    """Input window w = n >> split of the Rhombus PCMv (he_oracle_pcmv.c).  Default: the largest split
    point whose pieces still hold n_in values (w = the smallest power of two >= n_in / rho)."""
    n, rho = params.rhombus_degree, params.N // params.rhombus_degree
    if split is None:
        w = 1
        while w * rho < n_in:
            w *= 2
        return min(w, n)
    w = n >> int(split)
    if w < 1 or w * rho < n_in:
        raise ValueError(f"split {split}: window {w} x {rho} pieces cannot hold {n_in} values")
    return w


def encode_vector(params, v: np.ndarray, window=None) -> np.ndarray:
    """Input layout: element e at (e / w) + rho h_w(e mod w); window None = the old h layout (w = n)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    pt = np.zeros((1, params.N), np.int64)
    w = params.rhombus_degree if window is None else int(window)
    _rh_lib().or_encode_vector_w(_f64(v), len(v), params.N, params.rhombus_degree, w, params.delta, _i64(pt))
    return pt


def decode_vector(params, phase: np.ndarray, n_vals: int) -> np.ndarray:
    v = np.zeros(n_vals)
    _rh_lib().or_decode_vector(_i64(np.ascontiguousarray(phase, dtype=np.int64)), n_vals, params.N,
                               params.rhombus_degree, params.delta, _f64(v))
    return v


def rhombus_pcmv(params, ct_in: np.ndarray, ksk: np.ndarray, gal: np.ndarray, Wt: np.ndarray, n_in: int):
    """ct_in [2 limbs][2][N] level 1 -> (packed level-1 pieces [p_out][2][2][n], out [2][N] level 0)."""
    N, n = params.N, params.rhombus_degree
    Wt = np.ascontiguousarray(Wt, dtype=np.int64)
    n_out = Wt.shape[0]
    p_out = -(-n_out // n)
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    pieces = np.zeros((p_out, 2, 2, n), np.uint32)
    out = np.zeros((2, N), np.uint32)
    _rh_lib().or_rhombus_pcmv(N, n, _u32(m), _u32(np.ascontiguousarray(ct_in, dtype=np.uint32)),
                              _u32(np.ascontiguousarray(ksk)), _u32(np.ascontiguousarray(gal)), _i64(Wt), n_out, n_in,
                              _u32(pieces), _u32(out))
    return pieces, out


def rhombus_pcmv_w(params, ct_in: np.ndarray, ksk: np.ndarray, gal: np.ndarray, Wt: np.ndarray, n_in: int,
                   window: int, piece0: int = 0, level1: bool = False) -> np.ndarray:
    """Windowed (split-point) PCMv, he_oracle_pcmv.c or_rhombus_pcmv_w: level1=False -> [2 (a, b)][N]
    level 0; level1=True -> the column shard's level-1 composed output [2 limbs][2][N]."""
    N, n = params.N, params.rhombus_degree
    Wt = np.ascontiguousarray(Wt, dtype=np.int64)
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    out = np.zeros((2, 2, N) if level1 else (2, N), np.uint32)
    rc = _rh_lib().or_rhombus_pcmv_w(N, n, int(window), _u32(m), _u32(np.ascontiguousarray(ct_in, dtype=np.uint32)),
                                     _u32(np.ascontiguousarray(ksk, dtype=np.uint32)),
                                     _u32(np.ascontiguousarray(gal, dtype=np.uint32)), _i64(Wt), Wt.shape[0], n_in,
                                     int(piece0), int(level1), _u32(out))
    if rc:
        raise ValueError("or_rhombus_pcmv_w: bad shape / window")
    return out


def rhombus_combine(params, parts: np.ndarray) -> np.ndarray:
    """Sum column-shard level-1 outputs [count][2][2][N] mod q_i, rescale by q1 -> [2][N]."""
    parts = np.ascontiguousarray(parts, dtype=np.uint32)
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    out = np.zeros((2, params.N), np.uint32)
    _rh_lib().or_rhombus_combine(_u32(parts), parts.shape[0], params.N, _u32(m), _u32(out))
    return out


def rhombus_weights(params, W: np.ndarray) -> np.ndarray:
    """W~ = round_half_even(q1 W) (the h shuffle is applied inside the PCMv)."""
    return np.rint(np.asarray(W, np.float64) * params.delta_w).astype(np.int64)


def decrypt_under(params, a: np.ndarray, b: np.ndarray, s: np.ndarray, q: int) -> np.ndarray:
    """centred b + a s mod q (degree len(a))."""
    n = len(a)
    prod = negacyclic_mul(np.ascontiguousarray(a, dtype=np.uint32), np.ascontiguousarray(s, dtype=np.int32), q)
    v = (prod.astype(np.int64) + b.astype(np.int64)) % q
    return np.where(v > q // 2, v - q, v)


# ---------------------------------------------------------------- MLWE -> RLWE ring packing (§8f1)
def _rp_lib():
    L = _rh_lib()
    if not getattr(L, "_rp_bound", False):
        u32p, i32p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32)
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        L.or_ring_galois_ksk.restype = None
        L.or_ring_galois_ksk.argtypes = [u64, u32, i32p, u32, u32, u32p, u32p]
        L.or_ring_pack.restype = ctypes.c_int
        L.or_ring_pack.argtypes = [u32, u32, u32, u32p, u32p, u32, u32p, u32p, u32p]
        L._rp_bound = True
    return L


def ring_pack_keys(params, seed: int, s: np.ndarray) -> np.ndarray:
    """Galois keys sigma_{1 + 2^l d}: sigma(s) -> s at degree N, l = 1 .. log2 k -> [log k, 2, 2, 3, N]."""
    N, d, k = params.N, params.mlwe_degree, params.mlwe_rank
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    lg = k.bit_length() - 1
    gal = np.zeros((lg, 2, 2, 3, N), np.uint32)
    for lv in range(1, lg + 1):
        g = np.zeros((2, 2, 3, N), np.uint32)
        _rp_lib().or_ring_galois_ksk(seed, lv, _i32(np.ascontiguousarray(s, dtype=np.int32)), N, d, _u32(m), _u32(g))
        gal[lv - 1] = g
    return gal


def ring_pack_leaves(params, raw: list) -> np.ndarray:
    """Leaf ciphertexts C_y [n_out, 2 limbs, 2, N] (scaled by k^-1) from the un-rescaled MLWE words
    raw[limb] = [n_out, d + d k] (pcmm_limb):  A_y[k m - j] = a'_y[j][m] (negacyclic), B_y[k m] = b'_y[m]."""
    N, d, k = params.N, params.mlwe_degree, params.mlwe_rank
    n_out = raw[0].shape[0]
    j = np.arange(k)[:, None]
    mm = np.arange(d)[None, :]
    c = (k * mm - j).ravel()                 # position of a'[j][m] (flattened j-major like the words)
    neg = c < 0
    c = np.where(neg, c + N, c)
    leaves = np.zeros((n_out, 2, 2, N), np.uint32)
    for L in range(2):
        q = int(params.moduli[L])
        kinv = pow(k, q - 2, q)
        v = raw[L].astype(np.int64)
        a = v[:, d:]
        a = np.where(neg[None, :], (q - a) % q, a)
        leaves[:, L, 0, c] = (a * kinv % q).astype(np.uint32)
        leaves[:, L, 1, k * np.arange(d)] = (v[:, :d] * kinv % q).astype(np.uint32)
    return leaves


def ring_pack(params, leaves: np.ndarray, gal: np.ndarray):
    """-> (packed level-1 [blocks, 2, 2, N], out level-0 [blocks, 2 (a, b), N]); see he_oracle_rhombus.c."""
    N, d, k = params.N, params.mlwe_degree, params.mlwe_rank
    cnt = leaves.shape[0]
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    packed = np.zeros((cnt // k, 2, 2, N), np.uint32)
    out = np.zeros((cnt // k, 2, N), np.uint32)
    rc = _rp_lib().or_ring_pack(N, d, k, _u32(m), _u32(np.ascontiguousarray(leaves, dtype=np.uint32)), cnt,
                                _u32(np.ascontiguousarray(gal, dtype=np.uint32)), _u32(packed), _u32(out))
    if rc:
        raise ValueError("ring pack: bad shape")
    return packed, out


def pcmm_ring_pack(params, Wt, ct, gal):
    """Reference MLWE PCMM followed by ring packing: level-0 RLWE output blocks [n_out / k, 2, N]."""
    raw = [pcmm_limb(params, Wt, ct, L) for L in range(2)]
    return ring_pack(params, ring_pack_leaves(params, raw), gal)[1]


def _ms_bind():
    L = _rp_lib()
    if not getattr(L, "_ms_bound", False):
        u32p, i32p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32)
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        L.or_mlwe_ksk.restype = None
        L.or_mlwe_ksk.argtypes = [u64, u32, i32p, u32, u32, u32p, u32p]
        L.or_mlwe_to_rlwe.restype = ctypes.c_int
        L.or_mlwe_to_rlwe.argtypes = [u32, u32, u32p, u32p, u32p, u32, u32p, u32p]
        L._ms_bound = True
    return L


def mlwe_ks_keys(params, seed: int, s: np.ndarray) -> np.ndarray:
    """MLWE -> RLWE key-switching keys s_j(X^k) -> s, j = 0 .. k-1 -> [k, 2, 2, 3, N] (coefficient form)."""
    N, k = params.N, params.mlwe_rank
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    out = np.zeros((k, 2, 2, 3, N), np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    for j in range(k):
        g = np.zeros((2, 2, 3, N), np.uint32)
        _ms_bind().or_mlwe_ksk(seed, j, _i32(s), N, k, _u32(m), _u32(g))
        out[j] = g
    return out


def ring_pack_special2(params) -> int:
    """The second special prime of ring packing KEYSWITCH1 (he_ring_pack_special2): the largest prime < 2^30,
    1 mod 2N, other than q0, q1 and P."""
    from paper_2601_18511_b200.params import ntt_primes

    for p in ntt_primes(2 * params.N, 1 << 30, 8):
        if p not in (params.moduli[0], params.moduli[1], params.special_prime):
            return p
    raise ValueError("no second special prime")


def _ms1_bind():
    L = _rp_lib()
    if not getattr(L, "_ms1_bound", False):
        u32p, i32p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32)
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        L.or_mlwe_ksk1.restype = None
        L.or_mlwe_ksk1.argtypes = [u64, u32, i32p, u32, u32, u32p, u32p]
        L.or_mlwe_ksk1_all.restype = None
        L.or_mlwe_ksk1_all.argtypes = [u64, i32p, u32, u32, u32p, u32p]
        L.or_mlwe_to_rlwe1.restype = ctypes.c_int
        L.or_mlwe_to_rlwe1.argtypes = [u32, u32, u32p, u32p, u32p, u32, u32p, u32p]
        L._ms1_bound = True
    return L


def _m4(params):
    return np.ascontiguousarray(np.array([params.moduli[0], params.moduli[1], params.special_prime,
                                          ring_pack_special2(params)], dtype=np.uint32))


def mlwe_ks_keys1(params, seed: int, s: np.ndarray) -> np.ndarray:
    """One-digit MLWE -> RLWE keys s_j(X^k) -> s mod (q0, q1, P1, P2): [k, 2, 4, N] (coefficient form)."""
    N, k = params.N, params.mlwe_rank
    m = _m4(params)
    out = np.zeros((k, 2, 4, N), np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    _ms1_bind().or_mlwe_ksk1_all(seed, _i32(s), N, k, _u32(m), _u32(out))
    return out


def mlwe_to_rlwe1(params, raw_b: np.ndarray, raw_a: np.ndarray, ksk: np.ndarray) -> np.ndarray:
    """One-digit MLWE -> RLWE key-switch packing (or_mlwe_to_rlwe1) -> [n_out/k, 2, N] level 0."""
    d, k, N = params.mlwe_degree, params.mlwe_rank, params.N
    n_out = raw_a.shape[1]
    out = np.zeros((n_out // k, 2, N), np.uint32)
    rc = _ms1_bind().or_mlwe_to_rlwe1(d, k, _u32(_m4(params)), _u32(np.ascontiguousarray(raw_b, dtype=np.uint32)),
                                      _u32(np.ascontiguousarray(raw_a, dtype=np.uint32)), n_out,
                                      _u32(np.ascontiguousarray(ksk, dtype=np.uint32)), _u32(out))
    if rc:
        raise ValueError("mlwe_to_rlwe1: bad shape")
    return out


def raw_device_layout(params, raw: list):
    """pcmm_limb words [limb] -> (raw_b [2, n_out/k, N] RLWE order, raw_a [2, n_out, k d]) as
    he_pcmm_run_level1 writes them."""
    N, d, k = params.N, params.mlwe_degree, params.mlwe_rank
    n_out = raw[0].shape[0]
    raw_b = np.zeros((2, n_out // k, N), np.uint32)
    raw_a = np.zeros((2, n_out, N), np.uint32)
    for L in range(2):
        raw_a[L] = raw[L][:, d:]
        for y in range(n_out):
            raw_b[L, y // k, y % k + k * np.arange(d)] = raw[L][y, :d]
    return raw_b, raw_a


def mlwe_to_rlwe(params, raw_b: np.ndarray, raw_a: np.ndarray, ksk: np.ndarray) -> np.ndarray:
    """MLWE -> RLWE key-switch packing (he_oracle_rhombus.c or_mlwe_to_rlwe) -> [n_out/k, 2, N] level 0."""
    d, k, N = params.mlwe_degree, params.mlwe_rank, params.N
    n_out = raw_a.shape[1]
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    out = np.zeros((n_out // k, 2, N), np.uint32)
    rc = _ms_bind().or_mlwe_to_rlwe(d, k, _u32(m), _u32(np.ascontiguousarray(raw_b, dtype=np.uint32)),
                                    _u32(np.ascontiguousarray(raw_a, dtype=np.uint32)), n_out,
                                    _u32(np.ascontiguousarray(ksk, dtype=np.uint32)), _u32(out))
    if rc:
        raise ValueError("mlwe_to_rlwe: bad shape")
    return out


# ---------------------------------------------------------------- slot-domain BSGS PCMM (§8f3)
def _sd_bind():
    L = _rh_lib()
    if not getattr(L, "_sd_bound", False):
        u32p, i32p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32)
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        L.or_rotation_ksk.restype = None
        L.or_rotation_ksk.argtypes = [u64, u32, i32p, u32, u32p, u32p]
        L.or_slot_pcmm.restype = ctypes.c_int
        L.or_slot_pcmm.argtypes = [u32, u32p, u32, u32, u32, u32p, u32p, u32p, u32p, u32p]
        L.or_slot_bsgs.restype = ctypes.c_int
        L.or_slot_bsgs.argtypes = [u32, u32p, u32, u32, u32, u32p, u32p, u32p, u32p, u32p]
        L.or_slot_bsgs_lazy.restype = ctypes.c_int
        L.or_slot_bsgs_lazy.argtypes = [u32, u32p, u32, u32, u32, u32p, u32p, u32p, u32p, ctypes.c_int, u32p]
        L.or_rotation_ksk_plain.restype = None
        L.or_rotation_ksk_plain.argtypes = [ctypes.c_uint64, u32, i32p, u32, u32p, u32p]
        L._sd_bound = True
    return L


def rotation_keys(params, seed: int, s: np.ndarray, steps) -> np.ndarray:
    """Gadget keys sigma_{5^r}(s) -> s for each step r -> [len(steps), 4, 2, 3, N] (coefficient form)."""
    N = params.N
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    out = np.zeros((len(steps), 4, 2, 3, N), np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    for t, r in enumerate(steps):
        g = np.zeros((4, 2, 3, N), np.uint32)
        _sd_bind().or_rotation_ksk(seed, int(r) % (N // 2), _i32(s), N, _u32(m), _u32(g))
        out[t] = g
    return out


def slot_pcmm(params, ct_in: np.ndarray, pts: np.ndarray, d: int, b: int, g: int, keys_baby, keys_giant) -> np.ndarray:
    """or_slot_pcmm: ct_in [2, 2, N] level 1, pts [d, 2, N] residues (coefficient form) -> [2, N] level 0."""
    N = params.N
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    out = np.zeros((2, N), np.uint32)
    kb = np.ascontiguousarray(keys_baby if len(keys_baby) else np.zeros((1, 4, 2, 3, N), np.uint32), dtype=np.uint32)
    kg = np.ascontiguousarray(keys_giant if len(keys_giant) else np.zeros((1, 4, 2, 3, N), np.uint32), dtype=np.uint32)
    rc = _sd_bind().or_slot_pcmm(N, _u32(m), d, b, g, _u32(np.ascontiguousarray(ct_in, dtype=np.uint32)),
                                 _u32(np.ascontiguousarray(pts, dtype=np.uint32)), _u32(kb), _u32(kg), _u32(out))
    if rc:
        raise ValueError("slot_pcmm: split does not cover d")
    return out


def rotation_keys_plain(params, seed: int, s: np.ndarray, steps) -> np.ndarray:
    """Plain dnum-2 keys sigma_{5^r}(s) -> s for each step r -> [len(steps), 2, 2, 3, N] (coefficient form)."""
    N = params.N
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    out = np.zeros((len(steps), 2, 2, 3, N), np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    for t, r in enumerate(steps):
        g = np.zeros((2, 2, 3, N), np.uint32)
        _sd_bind().or_rotation_ksk_plain(seed, int(r) % (N // 2), _i32(s), N, _u32(m), _u32(g))
        out[t] = g
    return out


def slot_bsgs(params, ct_in: np.ndarray, pts: np.ndarray, stride: int, b: int, g: int, keys_baby,
              keys_giant, lazy: bool = False) -> np.ndarray:
    """or_slot_bsgs: the general BSGS slot map (baby steps i stride, giant steps j b stride) -- SlotToCoeffs
    with stride 1.  pts [b g, 2, N] residues (coefficient form) -> [2, N] level 0.  lazy: or_slot_bsgs_lazy
    (baby rotations kept mod PQ, one ModDown per group), pts [b g, 3, N] (q0, q1, P); giant keys of
    rotation_keys_plain's shape [.., 2, 2, 3, N] select plain dnum-2 giant rotations."""
    N = params.N
    m = np.ascontiguousarray(np.array(params.ks_moduli, dtype=np.uint32))
    out = np.zeros((2, N), np.uint32)
    kb = np.ascontiguousarray(keys_baby if len(keys_baby) else np.zeros((1, 4, 2, 3, N), np.uint32), dtype=np.uint32)
    kg = np.ascontiguousarray(keys_giant if len(keys_giant) else np.zeros((1, 4, 2, 3, N), np.uint32), dtype=np.uint32)
    args = [N, _u32(m), stride, b, g, _u32(np.ascontiguousarray(ct_in, dtype=np.uint32)),
            _u32(np.ascontiguousarray(pts, dtype=np.uint32)), _u32(kb), _u32(kg)]
    if lazy:
        plain = kg.ndim == 5 and kg.shape[1] == 2 and len(keys_giant)
        rc = _sd_bind().or_slot_bsgs_lazy(*args, 1 if plain else 0, _u32(out))
    else:
        rc = _sd_bind().or_slot_bsgs(*args, _u32(out))
    if rc:
        raise ValueError("slot_bsgs: split x stride exceeds the slots")
    return out


# ---------------------------------------------------------------- modulus chain (he_oracle_chain.c)
def _ch_bind():
    L = lib()
    if not getattr(L, "_ch_bound", False):
        u32p, i32p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32)
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        L.or_chain_key_id.restype = u32
        L.or_chain_key_id.argtypes = [u32, u32]
        L.or_chain_rotation_ksk.restype = None
        L.or_chain_rotation_ksk.argtypes = [u64, u32, i32p, u32, u32p, u32, u32p]
        L.or_chain_bsgs.restype = ctypes.c_int
        L.or_chain_bsgs.argtypes = [u32, u32p, u32, u32, u32, u32, u32, u32p, u32p, u32p, u32p, u32p]
        L._ch_bound = True
    return L


def _chain_mods(params, level: int) -> np.ndarray:
    return np.ascontiguousarray(np.array(list(params.moduli[: level + 1]) + [params.special_prime], dtype=np.uint32))


def chain_key_id(level: int, step: int) -> int:
    return int(_ch_bind().or_chain_key_id(level, step))


def chain_rotation_keys(params, seed: int, s: np.ndarray, steps, level: int) -> np.ndarray:
    """[len(steps), l+1, 2, l+2, N] coefficient-form rotation keys at `level` (he_oracle_chain.c)."""
    L = _ch_bind()
    N, nq = params.N, level + 1
    m = _chain_mods(params, level)
    out = np.zeros((max(len(steps), 1), nq, 2, nq + 1, N), np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    for t, r in enumerate(steps):
        k = np.zeros((nq, 2, nq + 1, N), np.uint32)
        L.or_chain_rotation_ksk(seed, int(r) % (N // 2), _i32(s), N, _u32(m), nq, _u32(k))
        out[t] = k
    return out


def chain_bsgs(params, ct_in: np.ndarray, pts: np.ndarray, level: int, b: int, g: int, stride: int, T: int,
               keys_baby: np.ndarray, keys_giant: np.ndarray) -> np.ndarray:
    """One BSGS map at `level` (he_oracle_chain.c or_chain_bsgs): ct [l+1, 2, N] -> [l, 2, N]."""
    L = _ch_bind()
    N, nq = params.N, level + 1
    m = _chain_mods(params, level)
    out = np.zeros((nq - 1, 2, N), np.uint32)
    rc = L.or_chain_bsgs(N, _u32(m), nq, b, g, stride, T, _u32(np.ascontiguousarray(ct_in, dtype=np.uint32)),
                         _u32(np.ascontiguousarray(pts, dtype=np.uint32)),
                         _u32(np.ascontiguousarray(keys_baby, dtype=np.uint32)),
                         _u32(np.ascontiguousarray(keys_giant, dtype=np.uint32)), _u32(out))
    if rc:
        raise ValueError("or_chain_bsgs: bad level")
    return out
