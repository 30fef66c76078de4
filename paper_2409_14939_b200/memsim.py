"""IO accounting types of ``minigl.memsim`` as reported by the B200 trainer.

The reference *simulates* the host-to-device feature traffic of an epoch
(memsim.py:129-186) and prices the aggregation fetches with an analytic model
(memsim.py:83-107).  On the GPU path the traffic is not simulated: the Match
loader (loader.cu ``fgl_gather_rows_cached``) counts, per batch, the rows it
read from the feature store and the rows the static HBM cache served, and
``trainer.train`` turns those counts into the same report.  The analytic
fetch model is kept because ``EpochStats.modeled_fetch_seconds`` is defined
by it (trainer.py:230-242); its inputs -- the per-layer row-length histograms
of the block CSRs -- come from the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import ValidationError

__all__ = ["CostParams", "BatchTraffic", "TrafficReport", "t_naive", "t_memory_aware"]


@dataclass
class CostParams:
    """Modeled bandwidths (bytes/s) and capacities (memsim.py:28-47)."""

    shared_bw: float = 12e12
    global_bw: float = 938e9
    host_link_bw: float = 32e9
    device_capacity: int = 24 * 2**30
    bytes_per_elem: int = 4

    def validate(self):
        if min(self.shared_bw, self.global_bw, self.host_link_bw) <= 0:
            raise ValidationError("bandwidths must be positive")
        if self.device_capacity <= 0 or self.bytes_per_elem <= 0:
            raise ValidationError("capacities must be positive")


@dataclass
class BatchTraffic:
    """One executed batch (memsim.py:50-58): rows over the host link, and the
    bytes the static cache and the Match reuse served instead."""

    position: int
    loaded_nodes: int
    bytes_h2d: int
    bytes_cache: int
    bytes_match: int


@dataclass
class TrafficReport:
    """Epoch totals and the per-batch rows they sum from (memsim.py:61-79)."""

    bytes_host_to_device: int
    bytes_served_by_cache: int
    bytes_served_by_match: int
    modeled_io_seconds: float
    per_batch: list = field(default_factory=list)

    def to_dict(self) -> dict:
        out = {k: getattr(self, k) for k in ("bytes_host_to_device", "bytes_served_by_cache",
                                             "bytes_served_by_match", "modeled_io_seconds")}
        out["per_batch"] = [vars(b) for b in self.per_batch]
        return out

    def __getitem__(self, key):  # dict-style access used by older callers
        return getattr(self, key)

    @classmethod
    def from_batches(cls, per_batch, params: CostParams) -> "TrafficReport":
        h2d = sum(b.bytes_h2d for b in per_batch)
        return cls(bytes_host_to_device=h2d, bytes_served_by_cache=sum(b.bytes_cache for b in per_batch),
                   bytes_served_by_match=sum(b.bytes_match for b in per_batch),
                   modeled_io_seconds=h2d / params.host_link_bw, per_batch=list(per_batch))


def _check(fanout, dim, params):
    if fanout < 1 or dim < 1:
        raise ValidationError("fanout and dim must be >= 1")
    params.validate()


def t_naive(fanout: int, dim: int, params: CostParams) -> float:
    """All operands from global memory (memsim.py:83-93, Eq. 3): partial sums
    (fanout-1)*dim, one weight per element, one feature element each."""
    _check(fanout, dim, params)
    return 4 * dim * ((fanout - 1) + 2 * fanout) / params.global_bw


def t_memory_aware(fanout: int, dim: int, params: CostParams) -> float:
    """Partial sums and weights staged in the scratch tier (memsim.py:96-107,
    Eq. 4); features and one read per weight stay in global memory."""
    _check(fanout, dim, params)
    fast = 4 * ((fanout - 1) * dim + fanout * (dim - 1))
    slow = 4 * fanout * (dim + 1)
    return fast / params.shared_bw + slow / params.global_bw
