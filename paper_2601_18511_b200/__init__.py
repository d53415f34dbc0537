"""B200-native MLWE-format PCMM / Rhombus PCMv for CKKS-encrypted Llama inference.

Host mirror of the reference's operator API (hesim/__init__.py:3-19 exports) for
the encrypted-projection path; every computation runs in hand-written sm_100a CUDA
behind the C ABI of include/he_b200.h.  There is no CPU fallback.
"""

from .errors import NeedsBootstrapError
from .params import HeParams
from .context import CostLedger, CtBlocks, HeContext, MlweBlocks, SecretKey, LEDGER_COUNTERS
from .layout import bit_reverse, byte_mix, half_reverse, rotate_bits_down, shuffle_matrix, sigma_table
from .pcmm import (MlwePcmmPlan, clear_pcmm, load_mlwe_pcmm_plan, load_plan_bundle, make_mlwe_pcmm_plan, pcmm_mlwe,
                   pcmm_mlwe_into_peers, pcmm_mlwe_to_host, save_mlwe_pcmm_plan, save_plan_bundle)
from .rhombus import (CtVector, RhombusKeys, RhombusPlan, clear_pcmv, decrypt_vector, encrypt_vector,
                      make_rhombus_plan, pcmv_rhombus, rhombus_keygen)
from .slotpcmm import (BsgsSplit, PackedCt, SlotPcmmKeys, SlotPcmmPlan, clear_slot_pcmm, decrypt_packed,
                       encrypt_packed, make_slot_pcmm_plan, pcmm_slot_bsgs, pcmm_slot_depth1, slot_pcmm_keygen)
from .graphs import OpGraph
from .ringpack import (RingPackKeys, RingPackPlan, make_ring_pack_plan, mod_raise, pcmm_level1, pcmm_packed, ring_pack,
                       ring_pack_keygen)
from .stc import SlotBlocks, encrypt_slots, make_slot_to_coeffs_plan, slot_to_coeffs, slot_to_coeffs_keygen

__all__ = [
    "NeedsBootstrapError", "HeParams", "CostLedger", "CtBlocks", "HeContext", "MlweBlocks", "SecretKey",
    "LEDGER_COUNTERS", "bit_reverse", "byte_mix", "half_reverse", "rotate_bits_down", "shuffle_matrix",
    "sigma_table", "MlwePcmmPlan", "clear_pcmm", "make_mlwe_pcmm_plan", "pcmm_mlwe", "pcmm_mlwe_to_host",
    "pcmm_mlwe_into_peers", "save_mlwe_pcmm_plan", "load_mlwe_pcmm_plan", "save_plan_bundle", "load_plan_bundle",
    "CtVector", "RhombusKeys", "RhombusPlan", "clear_pcmv", "decrypt_vector", "encrypt_vector",
    "make_rhombus_plan", "pcmv_rhombus", "rhombus_keygen",
    "RingPackKeys", "RingPackPlan", "make_ring_pack_plan", "pcmm_level1", "pcmm_packed", "ring_pack",
    "ring_pack_keygen", "mod_raise",
    "BsgsSplit", "PackedCt", "SlotPcmmKeys", "SlotPcmmPlan", "clear_slot_pcmm", "decrypt_packed", "encrypt_packed",
    "make_slot_pcmm_plan", "pcmm_slot_bsgs", "pcmm_slot_depth1", "slot_pcmm_keygen", "OpGraph",
    "SlotBlocks", "encrypt_slots", "make_slot_to_coeffs_plan", "slot_to_coeffs", "slot_to_coeffs_keygen",
]

__version__ = "0.1.0"
