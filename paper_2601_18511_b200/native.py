"""ctypes binding of the in-tree C ABI (include/he_b200.h -> _lib/libhe_b200.so).

There is no fallback: if the library is missing or was built for another
architecture, every op raises.  Status codes map onto the reference's exceptions
(matmul.py:139-149, slotsim.py:27-28).
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import NeedsBootstrapError

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libhe_b200.so"
_lock = threading.Lock()
_lib = None

HE_OK, HE_EINVAL, HE_ETYPE, HE_ENEEDS_BOOTSTRAP, HE_ECUDA, HE_ENOMEM = range(6)

# every symbol include/he_b200.h declares (tests/test_boundary.py checks the header agrees)
EXPORTS = (
    "he_last_error", "he_version", "he_context_create", "he_context_destroy", "he_keygen",
    "he_encrypt_acts", "he_decrypt_rlwe", "he_decrypt_mlwe", "he_ntt_forward", "he_ntt_inverse",
    "he_pcmm_weight_maxabs", "he_pcmm_encode_weights", "he_pcmm_plan_create", "he_pcmm_plan_destroy",
    "he_pcmm_workspace_bytes", "he_pcmm_run", "he_pcmm_decompose", "he_pcmm_gemm",
    "he_encrypt_vector", "he_rhombus_keygen", "he_rhombus_weight_bytes", "he_rhombus_encode_weights",
    "he_rhombus_plan_create", "he_rhombus_plan_destroy", "he_rhombus_workspace_bytes", "he_rhombus_run",
    "he_pcmm_gemm_rows", "he_pcmm_spectral_weight_bytes", "he_pcmm_spectral_prepare", "he_pcmm_algo",
    "he_pcmm_profile", "he_pcmm_profile_read", "he_pcmm_spectral_info", "he_pcmm_gemm_rows_peers",
    "he_pcmm_run_level1", "he_ring_pack_key_bytes", "he_ring_pack_keygen", "he_ring_pack_plan_create", "he_ring_pack_plan_destroy",
    "he_ring_pack_workspace_bytes", "he_ring_pack_run", "he_rhombus_run_shard", "he_rhombus_combine",
    "he_encrypt_poly", "he_slot_rotation_keygen", "he_slot_pcmm_encode_pts", "he_slot_pcmm_plan_create",
    "he_slot_pcmm_plan_destroy", "he_slot_pcmm_workspace_bytes", "he_slot_pcmm_run", "he_slot_pcmm_run_batch", "he_mod_raise",
    "he_slot_lt_plan_create", "he_slot_bsgs_plan_create", "he_slot_bsgs_plan_create_ext", "he_slot_pcmm_encode_pts_ext", "he_slot_rotation_keygen_plain",
    "he_encrypt_vector_w", "he_rhombus_weight_bytes_w", "he_rhombus_encode_weights_w", "he_rhombus_plan_create_w",
    "he_rhombus_plan_info", "he_rhombus_run_subtree", "he_rhombus_finish", "he_context_set_rng_key",
    "he_chacha20_block", "he_chain_create", "he_chain_destroy", "he_chain_encrypt", "he_chain_key_id",
    "he_chain_key_words", "he_chain_rotation_keygen", "he_chain_encode_pts", "he_chain_map_create",
    "he_chain_map_destroy", "he_chain_map_workspace_bytes", "he_chain_map_run", "he_chain_decrypt",
    "he_ring_pack_special2",
)


class HeParamsC(ctypes.Structure):
    _fields_ = [("mlwe_degree", ctypes.c_uint32), ("mlwe_rank", ctypes.c_uint32),
                ("moduli", ctypes.c_uint32 * 2), ("log_delta", ctypes.c_uint32),
                ("rhombus_degree", ctypes.c_uint32), ("special_prime", ctypes.c_uint32)]


class HeLedgerC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("ct_rotations", "cc_mults", "pc_mults", "pt_rotations",
                                               "pt_mults", "rescales", "bootstraps")]


def library_path() -> Path:
    return _LIB_PATH


def lib():
    """Load the CUDA library (no fallback: raises if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists():
            raise RuntimeError(
                f"CUDA library {_LIB_PATH} is missing; run __graft_entry__.build() "
                "(python -m paper_2601_18511_b200.build). There is no CPU fallback.")
        L = ctypes.CDLL(str(_LIB_PATH))
        vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        st = ctypes.c_int
        sig = {
            "he_last_error": (ctypes.c_char_p, []),
            "he_version": (i32, []),
            "he_context_create": (st, [ctypes.POINTER(HeParamsC), ctypes.POINTER(vp)]),
            "he_context_destroy": (st, [vp]),
            "he_keygen": (st, [vp, u64, vp, vp, vp]),
            "he_encrypt_acts": (st, [vp, vp, vp, u32, u64, u32, vp, vp]),
            "he_decrypt_rlwe": (st, [vp, vp, vp, u32, u32, u32, vp, vp]),
            "he_decrypt_mlwe": (st, [vp, vp, vp, vp, u32, u32, u32, vp, vp]),
            "he_ntt_forward": (st, [vp, vp, u32, u32, u32, u64, vp]),
            "he_ntt_inverse": (st, [vp, vp, u32, u32, u32, u64, vp]),
            "he_pcmm_weight_maxabs": (st, [vp, vp, u32, u32, ctypes.POINTER(u64), vp]),
            "he_pcmm_encode_weights": (st, [vp, vp, u32, u32, u32, vp, vp]),
            "he_pcmm_plan_create": (st, [vp, vp, u32, u32, u32, ctypes.POINTER(vp)]),
            "he_pcmm_plan_destroy": (st, [vp]),
            "he_pcmm_workspace_bytes": (st, [vp, ctypes.POINTER(u64)]),
            "he_pcmm_run": (st, [vp, vp, u32, vp, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
            "he_pcmm_decompose": (st, [vp, vp, vp, u64, vp]),
            "he_pcmm_gemm": (st, [vp, vp, vp, vp, vp]),
            "he_pcmm_gemm_rows": (st, [vp, vp, u32, u32, vp, vp, vp]),
            "he_pcmm_gemm_rows_peers": (st, [vp, vp, u32, u32, ctypes.POINTER(vp), ctypes.POINTER(vp), u32, u32, vp]),
            "he_pcmm_spectral_weight_bytes": (st, [vp, ctypes.POINTER(u64)]),
            "he_pcmm_spectral_prepare": (st, [vp, vp, vp]),
            "he_pcmm_algo": (st, [vp, ctypes.POINTER(ctypes.c_int)]),
            "he_pcmm_profile": (st, [vp, i32]),
            "he_pcmm_spectral_info": (st, [vp, ctypes.POINTER(u32)]),
            "he_pcmm_profile_read": (st, [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u32), u32]),
            "he_encrypt_vector": (st, [vp, vp, vp, u32, u64, u32, vp, vp]),
            "he_rhombus_keygen": (st, [vp, u64, vp, vp, vp, vp, vp, vp, vp]),
            "he_rhombus_weight_bytes": (st, [vp, u32, u32, ctypes.POINTER(u64)]),
            "he_rhombus_encode_weights": (st, [vp, vp, u32, u32, vp, vp]),
            "he_rhombus_plan_create": (st, [vp, vp, u32, u32, ctypes.POINTER(vp)]),
            "he_rhombus_plan_destroy": (st, [vp]),
            "he_rhombus_workspace_bytes": (st, [vp, ctypes.POINTER(u64)]),
            "he_rhombus_run": (st, [vp, vp, u32, vp, vp, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
            "he_pcmm_run_level1": (st, [vp, vp, u32, vp, vp, vp, u64, vp]),
            "he_rhombus_run_shard": (st, [vp, vp, u32, vp, vp, u32, u32, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
            "he_rhombus_combine": (st, [vp, vp, u32, vp, vp, ctypes.POINTER(HeLedgerC)]),
            "he_encrypt_poly": (st, [vp, vp, vp, u32, u64, u32, vp, vp]),
            "he_mod_raise": (st, [vp, vp, u32, vp, u32, vp, vp]),
            "he_slot_lt_plan_create": (st, [vp, vp, u32, vp, ctypes.POINTER(vp)]),
            "he_slot_bsgs_plan_create": (st, [vp, vp, u32, u32, u32, ctypes.POINTER(vp)]),
            "he_slot_rotation_keygen_plain": (st, [vp, u64, vp, vp, u32, vp, vp]),
            "he_slot_bsgs_plan_create_ext": (st, [vp, vp, u32, u32, u32, u32, ctypes.POINTER(vp)]),
            "he_slot_pcmm_encode_pts_ext": (st, [vp, vp, u32, u32, vp, vp]),
            "he_slot_rotation_keygen": (st, [vp, u64, vp, vp, u32, vp, vp]),
            "he_slot_pcmm_encode_pts": (st, [vp, vp, u32, vp, vp]),
            "he_slot_pcmm_plan_create": (st, [vp, vp, u32, u32, u32, ctypes.POINTER(vp)]),
            "he_slot_pcmm_plan_destroy": (st, [vp]),
            "he_slot_pcmm_workspace_bytes": (st, [vp, ctypes.POINTER(u64)]),
            "he_slot_pcmm_run": (st, [vp, vp, u32, vp, vp, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
            "he_slot_pcmm_run_batch": (st, [vp, vp, u32, u32, vp, vp, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
            "he_context_set_rng_key": (st, [vp, ctypes.c_char_p]),
            "he_chacha20_block": (st, [ctypes.c_char_p, u32, ctypes.c_char_p, ctypes.c_char_p]),
            "he_chain_create": (st, [vp, vp, u32, ctypes.POINTER(vp)]),
            "he_chain_destroy": (st, [vp]),
            "he_chain_encrypt": (st, [vp, vp, vp, u32, u32, u64, u32, vp, vp]),
            "he_chain_decrypt": (st, [vp, vp, vp, u32, u32, u32, vp, vp]),
            "he_ring_pack_special2": (st, [vp, ctypes.POINTER(u32)]),
            "he_chain_key_id": (u32, [u32, u32]),
            "he_chain_key_words": (st, [vp, u32, ctypes.POINTER(u64)]),
            "he_chain_rotation_keygen": (st, [vp, u64, vp, u32, vp, u32, vp, vp]),
            "he_chain_encode_pts": (st, [vp, vp, u32, u32, vp, vp]),
            "he_chain_map_create": (st, [vp, vp, u32, u32, u32, u32, u32, ctypes.POINTER(vp)]),
            "he_chain_map_destroy": (st, [vp]),
            "he_chain_map_workspace_bytes": (st, [vp, ctypes.POINTER(u64)]),
            "he_chain_map_run": (st, [vp, vp, u32, u32, vp, vp, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
            "he_encrypt_vector_w": (st, [vp, vp, vp, u32, u32, u64, u32, vp, vp]),
            "he_rhombus_weight_bytes_w": (st, [vp, u32, u32, u32, u32, ctypes.POINTER(u64)]),
            "he_rhombus_encode_weights_w": (st, [vp, vp, u32, u32, u32, u32, u32, vp, vp]),
            "he_rhombus_plan_create_w": (st, [vp, vp, u32, u32, u32, u32, u32, ctypes.POINTER(vp)]),
            "he_rhombus_plan_info": (st, [vp, ctypes.POINTER(u32)]),
            "he_rhombus_run_subtree": (st, [vp, vp, u32, vp, vp, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
            "he_rhombus_finish": (st, [vp, vp, vp, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
            "he_ring_pack_key_bytes": (st, [vp, i32, ctypes.POINTER(u64)]),
            "he_ring_pack_keygen": (st, [vp, i32, u64, vp, vp, vp]),
            "he_ring_pack_plan_create": (st, [vp, u32, i32, ctypes.POINTER(vp)]),
            "he_ring_pack_plan_destroy": (st, [vp]),
            "he_ring_pack_workspace_bytes": (st, [vp, ctypes.POINTER(u64)]),
            "he_ring_pack_run": (st, [vp, vp, vp, vp, vp, vp, u64, vp, ctypes.POINTER(HeLedgerC)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == HE_OK:
        return
    msg = (lib().he_last_error() or b"").decode(errors="replace")
    if status == HE_EINVAL:
        raise ValueError(msg)
    if status == HE_ETYPE:
        raise TypeError(msg)
    if status == HE_ENEEDS_BOOTSTRAP:
        raise NeedsBootstrapError(msg)
    raise RuntimeError(msg or f"he status {status}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
