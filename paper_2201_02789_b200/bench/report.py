"""Run report: the reference's SimReport (sim/report.py:12-50) measured on
the device, plus timing and traffic fields.

Counter semantics follow the simulator (sim/machine.py:165-247, 330-331):
``num_launches`` counts device-initiated launches with a non-empty
configuration, ``host_launches`` host-initiated ones, ``blocks_scheduled`` the
blocks of every launched grid.  ``makespan`` is the measured device time of
the run in nanoseconds; ``max_pending_depth`` is the deepest device launch
queue seen (launches issued whose first child block had not started);
``instructions`` is not observable on hardware and reads 0; the per-phase
times (``phase_time``, warp-ns) are filled by the ``-DDP_PROFILE=1`` build
(libdynpar_prof.so) and read 0 in the default build.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

PHASES = ("parent", "launch", "agg", "disagg", "child")


def _fmt_array(a: np.ndarray) -> str:
    a = a.ravel()
    if a.dtype.kind == "f":
        return " ".join(repr(float(v)) for v in a.tolist())
    return " ".join(map(str, a.tolist()))


def memory_digest(arrays: dict, kinds: dict) -> str:
    """sha256 over ``name:kind:v v v\\n`` in name order (sim/report.py:59-68):
    byte-identical buffers give the reference's digest."""
    h = hashlib.sha256()
    for name in sorted(arrays):
        h.update(name.encode())
        h.update(b":")
        h.update(kinds[name].encode())
        h.update(b":")
        h.update(_fmt_array(np.asarray(arrays[name])).encode())
        h.update(b"\n")
    return h.hexdigest()


@dataclass
class Report:
    num_launches: int
    host_launches: int
    blocks_scheduled: int
    instructions: int
    makespan: int
    max_pending_depth: int
    phase_time: dict
    arrays: dict            # output name -> numpy array (device results)
    kinds: dict             # output name -> element kind ("int", "long", ...)
    iterations: int = 0
    ns_device: float = 0.0
    ns_host: float = 0.0
    work_units: int = 0
    bytes_alg: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernel_launches: int = 0
    launch_lat_ns: float = 0.0  # mean device-launch latency (%globaltimer)
    unpublished_reads: int = 0  # publication-checker builds only
    poisoned_reads: int = 0     # publication-checker builds only
    extra: dict = field(default_factory=dict)
    _digest: str | None = field(default=None, repr=False)
    _lists: dict | None = field(default=None, repr=False)

    @property
    def buffers(self) -> dict:
        """Outputs as Python lists, like SimReport.buffers."""
        if self._lists is None:
            self._lists = {k: np.asarray(v).tolist()
                           for k, v in self.arrays.items()}
        return self._lists

    @property
    def memory_digest(self) -> str:
        if self._digest is None:
            self._digest = memory_digest(self.arrays, self.kinds)
        return self._digest

    @property
    def busy_time(self) -> int:
        return sum(self.phase_time.values())

    def to_text(self, include_buffers: bool = False) -> str:
        lines = [
            f"num_launches={self.num_launches}",
            f"host_launches={self.host_launches}",
            f"blocks_scheduled={self.blocks_scheduled}",
            f"instructions={self.instructions}",
            f"makespan={self.makespan}",
            f"max_pending_depth={self.max_pending_depth}",
        ]
        lines += [f"t_{ph}={self.phase_time.get(ph, 0)}" for ph in PHASES]
        lines.append(f"memory_digest={self.memory_digest}")
        if include_buffers:
            for name in sorted(self.arrays):
                lines.append(f"buffer {name} = "
                             f"{_fmt_array(np.asarray(self.arrays[name]))}")
        return "\n".join(lines) + "\n"

    @classmethod
    def from_stats(cls, st: dict, arrays: dict, kinds: dict,
                   **extra) -> "Report":
        phase = {ph: int(t) for ph, t in zip(PHASES, st["ns_phase"])}
        return cls(num_launches=int(st["num_launches"]),
                   host_launches=int(st["host_launches"]),
                   blocks_scheduled=int(st["blocks_scheduled"]),
                   instructions=0,
                   makespan=int(round(st["ns_device"])),
                   max_pending_depth=int(st["max_pending_depth"]),
                   phase_time=phase, arrays=arrays, kinds=kinds,
                   iterations=int(st["iterations"]),
                   ns_device=float(st["ns_device"]),
                   ns_host=float(st["ns_host"]),
                   work_units=int(st["work_units"]),
                   bytes_alg=int(st["bytes_alg"]),
                   h2d_bytes=int(st["h2d_bytes"]),
                   d2h_bytes=int(st["d2h_bytes"]),
                   kernel_launches=int(st["kernel_launches"]),
                   launch_lat_ns=float(st.get("launch_lat_ns_mean", 0.0)),
                   unpublished_reads=int(st.get("unpublished_reads", 0)),
                   poisoned_reads=int(st.get("poisoned_reads", 0)),
                   extra=dict(extra))
