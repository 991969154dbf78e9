"""Kernel families and the bandwidth spec (mirror of reference kernels.py:22-62).

The family determines the metric the fused GPU kernels evaluate: squared L2
for gaussian, L2 for exponential, L1 for laplacian (kernels.py:34-39).  The
kernel values themselves are computed inside the CUDA kernels (tile epilogue,
gather kernel); these types only carry the parameters across the boundary.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

__all__ = ["KernelFamily", "KernelSpec"]


class KernelFamily(str, enum.Enum):
    """Kernel families, named as in the reference CLI/configs (kernels.py:22-31)."""

    EXPONENTIAL = "exponential"
    GAUSSIAN = "gaussian"
    LAPLACIAN = "laplacian"

    @property
    def metric(self) -> str:
        return _METRIC[self]


_METRIC = {
    KernelFamily.EXPONENTIAL: "l2",
    KernelFamily.GAUSSIAN: "sql2",
    KernelFamily.LAPLACIAN: "l1",
}


@dataclass(frozen=True)
class KernelSpec:
    """Family + bandwidth h > 0 (ValueError otherwise, kernels.py:53-58)."""

    family: KernelFamily
    bandwidth: float

    def __post_init__(self):
        object.__setattr__(self, "family", KernelFamily(getattr(self.family, "value", self.family)))
        h = float(self.bandwidth)
        if not math.isfinite(h) or h <= 0.0:
            raise ValueError(f"bandwidth must be positive and finite, got {self.bandwidth!r}")
        object.__setattr__(self, "bandwidth", h)

    @property
    def metric(self) -> str:
        return self.family.metric


def as_spec(kernel) -> KernelSpec:
    """Accept this package's KernelSpec or any duck-typed (family, bandwidth) object,
    e.g. the reference's deann.KernelSpec."""
    if isinstance(kernel, KernelSpec):
        return kernel
    return KernelSpec(getattr(kernel.family, "value", kernel.family), kernel.bandwidth)
