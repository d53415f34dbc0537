"""Exceptions of the reference's error contract (slotsim.py:27-28, matmul.py:139-149)."""


class NeedsBootstrapError(RuntimeError):
    """Multiplicative depth is exhausted; the ciphertext needs a bootstrap."""
