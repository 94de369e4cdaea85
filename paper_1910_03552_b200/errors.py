"""Exception classes mirroring the reference's (same names, same bases).

SchemaError    rollout.py:15   shape / range / dtype violations of the learner input
DimensionError model.py:17     model / array shape inconsistencies
NonFiniteError model.py:21     NaN / inf where training must halt
"""
from __future__ import annotations

import torch


class SchemaError(ValueError):
    """A rollout or batch violates the learner input schema (rollout.py:15)."""


class DimensionError(ValueError):
    """Array shapes inconsistent with the model or with each other (model.py:17)."""


class NonFiniteError(ValueError):
    """A NaN/inf showed up where training must halt (model.py:21)."""


class NativeError(RuntimeError):
    """The CUDA library is missing, or a launch / argument error from the C ABI."""


# device status-word bits (include/beast_b200.h)
ACTION_RANGE = 1
NONFINITE_IN = 2
NEG_DISCOUNT = 4
NONFINITE_LOSS = 8
NONFINITE_GRAD = 16
BATCH_NONFINITE = 32


class StatusWord:
    """A device uint32 the kernels OR violation bits into.

    `check()` synchronises (reads 4 bytes), raises the reference's exception
    class for the first violation found, and clears the word.  In the learner
    loop it is checked lazily (once per step after the result is read back).
    """

    def __init__(self, device=None):
        self.word = torch.zeros(1, dtype=torch.int32, device=device or "cuda")

    def ptr(self) -> int:
        return self.word.data_ptr()

    def clear(self) -> None:
        self.word.zero_()

    def bits(self) -> int:
        return int(self.word.item())

    def check(self, context: str = "") -> None:
        bits = self.bits()
        if not bits:
            return
        self.word.zero_()
        raise_for_bits(bits, context)


def raise_for_bits(bits: int, context: str = "", learner: bool = False) -> None:
    """Raise the reference's exception for a status word.  learner=True maps a non-finite
    batch field to SchemaError as the learner step's validate_batch does (rollout.py:189-192);
    otherwise to NonFiniteError as _check_vtrace_inputs does (vtrace.py:83-91)."""
    where = f"{context}: " if context else ""
    if bits & ACTION_RANGE:
        raise SchemaError(f"{where}actions outside [0, num_actions)")
    if bits & NEG_DISCOUNT:
        raise SchemaError(f"{where}discounts must be non-negative")
    if bits & BATCH_NONFINITE:
        if learner:
            raise SchemaError(f"{where}reward / policy_logits contain non-finite values")
        raise NonFiniteError(f"{where}input contains non-finite values")
    if bits & NONFINITE_IN:
        raise NonFiniteError(f"{where}input contains non-finite values")
    if bits & NONFINITE_LOSS:
        raise NonFiniteError(f"{where}non-finite loss")
    if bits & NONFINITE_GRAD:
        raise NonFiniteError(f"{where}non-finite gradient")
