"""Closed-form per-device communication volume of one Evoformer block, forward + backward,
for head-sharded ("tensor") parallelism versus Dynamic Axial Parallelism, in units of K =
the byte size of the sharded activation (the model of commcost.py:50-123, paper §3.2):

  tensor parallel : 12 ring all-reduces per block, both passes     -> 24 K (N-1)/N
  axial  parallel : OPM factor gather + two triangle factor gathers ->  3 K (N-1)/N
                    + 6 axis switches (all-to-all) each way          -> 12 K (N-1)/N^2

Head sharding cannot use more devices than heads (HeadLimitError).  The byte-exact
ledger of a single block's forward is ``dap.predict_block_ledger``; this module is the
asymptotic comparison the `commvolume` CLI command reports.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

from .errors import DomainError, HeadLimitError


@dataclass(frozen=True)
class VolumeReport:
    k: float
    n_devices: int
    tp_volume: float
    dap_volume: float
    dap_breakdown: dict = field(default_factory=dict)

    @property
    def ratio(self) -> float:
        return self.tp_volume / self.dap_volume if self.dap_volume else float("inf")

    def as_dict(self) -> dict:
        return {"dap_breakdown": dict(self.dap_breakdown), "dap_volume": self.dap_volume, "k": self.k,
                "n_devices": self.n_devices, "ratio": self.ratio, "schema": "evoplan-commvolume-v1",
                "tp_volume": self.tp_volume}

    def to_json(self) -> str:
        return json.dumps(self.as_dict(), sort_keys=True)


@dataclass(frozen=True)
class CommModel:
    n_heads: int = 4
    all_reduces_per_block: int = 12
    axis_switches_per_block: int = 6

    @staticmethod
    def _validate(k: float, n: int) -> None:
        if k < 0:
            raise DomainError(f"volume parameter k must be non-negative, got {k}")
        if n < 1:
            raise DomainError(f"device count must be positive, got {n}")

    def tp_volume(self, k: float, n: int) -> float:
        self._validate(k, n)
        if n > self.n_heads:
            raise HeadLimitError(n, self.n_heads)
        frac = (n - 1) / n
        return 2.0 * self.all_reduces_per_block * k * frac

    def dap_breakdown(self, k: float, n: int) -> dict:
        self._validate(k, n)
        frac = (n - 1) / n
        return {"axis_switch": 2.0 * self.axis_switches_per_block * k * frac / n,
                "opm_gather": k * frac,
                "triangle_gather": 2.0 * k * frac}

    def dap_volume(self, k: float, n: int) -> float:
        return sum(self.dap_breakdown(k, n).values())

    def compare(self, k: float, n: int) -> VolumeReport:
        return VolumeReport(k=k, n_devices=n, tp_volume=self.tp_volume(k, n), dap_volume=self.dap_volume(k, n),
                            dap_breakdown=self.dap_breakdown(k, n))
