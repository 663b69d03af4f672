"""Geometry record types shared by the host-side modules (tree.py:37-53)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True, eq=False)
class BoundingBox:
    lo: np.ndarray
    hi: np.ndarray

    @property
    def extents(self) -> np.ndarray:
        return self.hi - self.lo

    @property
    def center(self) -> np.ndarray:
        return 0.5 * (self.lo + self.hi)

    @property
    def radius(self) -> float:
        """Half the box diagonal."""
        return 0.5 * float(np.sqrt(np.sum((self.hi - self.lo) ** 2)))
