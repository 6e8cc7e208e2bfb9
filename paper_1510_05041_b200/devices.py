"""Devices, topology, trace records and run metrics.

The reference describes a *simulated* fabric (/root/reference/pkg/src/tileblas/devices.py:
39-88) with speeds and link bandwidths; on B200 the topology is discovered: every visible
GPU is an accelerator, and all GPUs with mutual CUDA peer access (NVLink 5 / NVSwitch:
all 8) form one peer group, so any holder can serve an L2 hit.  ``DeviceDesc`` keeps the
reference fields (speed is informational; arena_capacity = 0 means "size it for the
call").  Metrics keep the reference JSON schema (devices.py:190-242, cli.py:83-84) with
*measured* seconds from CUDA events.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple, Optional

from .errors import ConfigError

ACCELERATOR = "accelerator"
HOST_COMPUTE = "host_compute"
N_STREAMS = 4


@dataclass(frozen=True)
class DeviceDesc:
    device_id: int                 # CUDA ordinal
    kind: str = ACCELERATOR
    speed: float = 37.1e12         # measured FP64 DMMA peak (informational)
    arena_capacity: int = 0        # bytes; 0 = auto
    peer_group: object = None
    cuda_ordinal: Optional[int] = None   # GPU backing this device (default: device_id)


@dataclass
class Topology:
    devices: list

    def __post_init__(self):
        if not self.devices:
            raise ConfigError("topology has no devices")
        ids = [d.device_id for d in self.devices]
        if len(set(ids)) != len(ids):
            raise ConfigError("duplicate device_id in topology")
        for d in self.devices:
            if d.kind != ACCELERATOR:
                # the host-compute worker of the reference (scheduler.py:508-539) is out of
                # scope: this library has no CPU fallback
                raise ConfigError(f"device {d.device_id}: only accelerators are supported")
            if d.arena_capacity < 0:
                raise ConfigError(f"device {d.device_id}: arena_capacity must be >= 0")

    def accelerators(self) -> list:
        return list(self.devices)

    def peer_group_of(self, desc: DeviceDesc):
        return ("standalone", desc.device_id) if desc.peer_group is None else desc.peer_group


def discover_topology(n_gpus: Optional[int] = None, arena_capacity: int = 0) -> Topology:
    """All visible GPUs (or the first ``n_gpus``), one NVLink peer group."""
    from . import _native
    count = _native.device_count()
    if count < 1:
        raise _native.NativeUnavailable("no CUDA device visible; this library has no CPU fallback")
    n = count if n_gpus is None else n_gpus
    if not 1 <= n <= count:
        raise ConfigError(f"requested {n} GPUs, {count} visible")
    return Topology([DeviceDesc(d, arena_capacity=arena_capacity, peer_group="nvlink")
                     for d in range(n)])


class TraceEvent(NamedTuple):
    time_start: float
    time_end: float
    device: int
    stream: int          # -1 when not tied to a stream; H2D/D2H/P2P use lanes -1/-2/-3
    event: str           # H2D | D2H | D2D | KERNEL | SYNC
    bytes_or_flops: int
    task_id: int
    k: int


def exposed_comm_time(transfers, kernels) -> float:
    """Transfer time not covered by any kernel interval on the same device."""
    if not transfers:
        return 0.0
    ks = sorted(kernels)
    merged = []
    for s, e in ks:
        if merged and s <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], e)
        else:
            merged.append([s, e])
    exposed = 0.0
    for ts, te in sorted(transfers):
        covered = 0.0
        for s, e in merged:
            if e <= ts:
                continue
            if s >= te:
                break
            covered += min(te, e) - max(ts, s)
        exposed += (te - ts) - covered
    return exposed


@dataclass
class DeviceMetrics:
    compt_seconds: float = 0.0
    comm_unoverlapped_seconds: float = 0.0
    other_seconds: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    d2d_in_bytes: int = 0
    d2d_out_bytes: int = 0
    tasks: int = 0
    kernel_launches: int = 0

    def elapsed_seconds(self) -> float:
        return self.compt_seconds + self.comm_unoverlapped_seconds + self.other_seconds

    def busy_seconds(self) -> float:
        return self.compt_seconds + self.comm_unoverlapped_seconds


@dataclass
class Metrics:
    makespan_seconds: float = 0.0
    l1_hits: int = 0
    l2_hits: int = 0
    host_fetches: int = 0
    devices: dict = field(default_factory=dict)
    total_flops: int = 0
    wall_seconds: float = 0.0
    phases: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        return {
            "makespan_seconds": self.makespan_seconds,
            "cache": {"l1_hits": self.l1_hits, "l2_hits": self.l2_hits,
                      "host_fetches": self.host_fetches},
            "devices": {
                str(d): {"compt_seconds": m.compt_seconds,
                         "comm_unoverlapped_seconds": m.comm_unoverlapped_seconds,
                         "other_seconds": m.other_seconds,
                         "h2d_bytes": m.h2d_bytes, "d2h_bytes": m.d2h_bytes,
                         "d2d_in_bytes": m.d2d_in_bytes, "d2d_out_bytes": m.d2d_out_bytes}
                for d, m in sorted(self.devices.items())},
        }

    def total_h2d_bytes(self) -> int:
        return sum(m.h2d_bytes for m in self.devices.values())

    def total_d2h_bytes(self) -> int:
        return sum(m.d2h_bytes for m in self.devices.values())

    def total_d2d_bytes(self) -> int:
        return sum(m.d2d_in_bytes for m in self.devices.values())

    def tflops(self) -> float:
        return self.total_flops / self.makespan_seconds / 1e12 if self.makespan_seconds else 0.0
