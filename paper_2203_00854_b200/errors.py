"""Exception hierarchy of the Evoformer hot path.

Same class names and meaning as the reference's ``evoplan.errors``
(/root/reference/pkg/src/evoplan/errors.py:1-57) so callers that catch
``DimensionError`` / ``DomainError`` / ``ShardError`` / ``MeshError`` keep
working.  Status codes returned by the C-ABI (include/evo.h) map onto these.
"""

from __future__ import annotations


class EvoplanError(Exception):
    """Base class of every error raised by this package."""


class DimensionError(EvoplanError):
    """Shapes, axes or config extents do not conform (errors.py:8-9)."""


class DomainError(EvoplanError):
    """Numerically invalid input, e.g. non-finite softmax input (errors.py:12-13)."""


class ShardError(EvoplanError):
    """A tensor extent is not divisible by the device count (errors.py:37-38)."""


class MeshError(EvoplanError):
    """Device mesh is invalid or incompatible (errors.py:41-42)."""


class KernelError(EvoplanError):
    """A CUDA kernel launch or the native library failed (no reference twin)."""


class NativeLibraryMissing(KernelError):
    """libevo.so is not built / not loadable.  There is no CPU fallback."""


class HeadLimitError(EvoplanError):
    """Head-sharded (tensor) parallelism cannot use more devices than attention heads
    (errors.py:44-53); raised by the closed-form volume model."""

    def __init__(self, n_devices: int, n_heads: int):
        self.n_devices = n_devices
        self.n_heads = n_heads
        super().__init__(f"tensor parallelism over {n_devices} devices exceeds the head-count limit of {n_heads}")
