"""Dynamic Axial Parallelism (DAP) over torch.distributed / NCCL.

Reference: dap_block.py:46-152 (the sharded schedule), sharding.py:26-212
(mesh, ledger, collective semantics) and commcost.py:126-158 (the byte-exact
ledger prediction).  The reference simulates devices as a Python loop; here
one process drives one GPU and the collectives are real:

  reference (simulated)                 here
  all_to_all_switch_axis (sharding:130)  dist.all_to_all_single (pack-free on one side)
  all_gather (sharding:162)              dist.all_gather_into_tensor, rank-major output
                                         addressed in place by the GEMMs (no unpack)
  (no backward in the reference)         all-gather^T = reduce_scatter_tensor, a2a^T = a2a

Canonical shards (dap_block.py:58-59, 150-151): m on the sequence axis,
z on the row axis; blocks chain on shards.  Per block forward: 6 all-to-all,
3 projection all-gathers, 1 bias all-gather (ledger categories as the
reference's CommLedger).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import torch

from .config import EvoConfig
from .errors import DomainError, MeshError, ShardError

REPORTING_ELEMENT_SIZE = 2


# ----------------------------------------------------------------------------- mesh + ledger
@dataclass(frozen=True)
class DeviceMesh:
    """1-D mesh (sharding.py:26-44).  On the GPU path device d is torch.distributed rank d;
    device_order only permutes host-side iteration and never changes results."""

    n_devices: int
    device_order: tuple = ()

    def __post_init__(self):
        if self.n_devices < 1:
            raise MeshError(f"need at least one device, got {self.n_devices}")
        order = self.device_order or tuple(range(self.n_devices))
        if sorted(order) != list(range(self.n_devices)):
            raise MeshError(f"device_order {order} is not a permutation of range({self.n_devices})")
        object.__setattr__(self, "device_order", tuple(order))


class CommLedger:
    """Per-device, per-category collective traffic (sharding.py:47-92), same JSON schema
    ``evoplan-ledger-v1``.  Bytes are logical sends under the reporting element size."""

    def __init__(self, n_devices: int, element_size: int = REPORTING_ELEMENT_SIZE):
        self.n_devices = n_devices
        self.element_size = element_size
        self.counts: dict[str, int] = {}
        self.bytes: dict[str, list[int]] = {}

    def record(self, category: str, per_device_elements) -> None:
        if len(per_device_elements) != self.n_devices:
            raise MeshError("ledger entry must cover every device")
        self.counts[category] = self.counts.get(category, 0) + 1
        row = self.bytes.setdefault(category, [0] * self.n_devices)
        for d, e in enumerate(per_device_elements):
            row[d] += int(e) * self.element_size

    def total_bytes(self, category: str | None = None) -> int:
        if category is not None:
            return sum(self.bytes.get(category, []))
        return sum(sum(v) for v in self.bytes.values())

    def device_bytes(self, device: int) -> int:
        return sum(v[device] for v in self.bytes.values())

    def summary(self) -> dict:
        return {cat: {"count": self.counts[cat], "bytes": sum(self.bytes[cat])} for cat in self.counts}

    def to_json(self) -> str:
        per_device = [{cat: {"count": self.counts[cat], "bytes": self.bytes[cat][d]} for cat in sorted(self.counts)}
                      for d in range(self.n_devices)]
        totals = {cat: {"count": self.counts[cat], "bytes": sum(self.bytes[cat])} for cat in sorted(self.counts)}
        return json.dumps({"schema": "evoplan-ledger-v1", "n_devices": self.n_devices,
                           "element_size": self.element_size, "per_device": per_device, "totals": totals},
                          sort_keys=True)


def predict_block_ledger(cfg: EvoConfig, n_devices: int, element_size: int = 2) -> dict:
    """Expected forward ledger of one sharded block (commcost.py:126-158): count and total
    bytes summed over devices for all_to_all / all_gather / bias_gather."""
    if n_devices < 1:
        raise DomainError(f"device count must be positive, got {n_devices}")
    if n_devices == 1:
        return {}
    es, n = element_size, n_devices
    m_bytes = cfg.n_seq * cfg.n_res * cfg.h_msa * es
    z_bytes = cfg.n_res * cfg.n_res * cfg.h_pair * es
    opm_factor = cfg.n_seq * cfg.n_res * cfg.hidden_proj * es
    tri_factor = cfg.n_res * cfg.n_res * cfg.hidden_proj * es
    bias_bytes = cfg.n_res * cfg.n_res * cfg.n_head_msa * es
    return {
        "all_to_all": {"count": 6, "bytes": round((2 * m_bytes + 4 * z_bytes) * (n - 1) / n)},
        "all_gather": {"count": 3, "bytes": round((opm_factor + 2 * tri_factor) * (n - 1))},
        "bias_gather": {"count": 1, "bytes": round(bias_bytes * (n - 1))},
    }
