"""Device buffers that only ever grow (the reference's GrowBuffer policy on HBM).

Same reallocation rule as /root/reference/pkg/src/mpmbench/memory.py:18-22 -- grow to four
times the request once a request exceeds half the capacity, never shrink -- so that
steady-state frames allocate nothing (tests/test_acceptance.py:287-307 of the
reference).  torch only provides the device allocation; the kernels see raw pointers.
"""
from __future__ import annotations

import torch

from .errors import RejectedInputError, ResourceError

GROWTH_FACTOR = 4


def grown_capacity(capacity: int, requested: int) -> int:
    """Capacity after a request: 4x the request once the buffer is half-filled."""
    if requested > capacity // 2:
        return GROWTH_FACTOR * requested
    return capacity


class DeviceBuffer:
    """Typed device array, `data[:len]` live; contents up to len survive a reallocation."""

    generation = 0      # bumped by every (re)allocation of any buffer of the process: "has a pointer moved?" in O(1)

    def __init__(self, dtype, element_shape=(), device="cuda", capacity: int = 0):
        self.dtype = dtype
        self.element_shape = tuple(element_shape)
        self.device = torch.device(device)
        self.capacity = int(capacity)
        self.len = 0
        self.realloc_count = 0
        self.data = torch.zeros((self.capacity, *self.element_shape), dtype=dtype, device=self.device)

    def ensure_capacity(self, requested: int, keep: bool = True) -> "DeviceBuffer":
        if requested < 0:
            raise RejectedInputError(f"requested capacity must be >= 0, got {requested}")
        new_cap = grown_capacity(self.capacity, requested)
        if new_cap != self.capacity:
            try:
                fresh = torch.zeros((new_cap, *self.element_shape), dtype=self.dtype,
                                    device=self.device)
            except RuntimeError as exc:   # torch.cuda.OutOfMemoryError is a RuntimeError
                raise ResourceError(
                    f"device allocation of {new_cap} x {self.element_shape} {self.dtype} "
                    f"elements failed (requested {requested})") from exc
            if keep and self.len:
                fresh[:self.len] = self.data[:self.len]
            self.data = fresh
            self.capacity = new_cap
            self.realloc_count += 1
            DeviceBuffer.generation += 1
        return self

    def resize(self, new_len: int, keep: bool = True) -> torch.Tensor:
        self.ensure_capacity(new_len, keep=keep)
        self.len = new_len
        return self.data[:new_len]

    @property
    def ptr(self) -> int:
        return self.data.data_ptr()

    def live(self) -> torch.Tensor:
        return self.data[:self.len]
