"""Device-timed measurement helpers shared by bench.py, tune.py and the selector.

Every number is CUDA-event time on the launching stream around CUDA-graph
replays of back-to-back calls; multi-GPU numbers take the max over ranks per
replay (the reference's makespan convention, bench.hpp:116-118).
"""
from __future__ import annotations

import ctypes
import statistics
import subprocess
import threading
from typing import Callable, List, Optional

import torch
import torch.distributed as dist

from . import dist as D

L2_BYTES = 126 << 20
ROTATE_BYTES = 160 << 20  # rotating input+output footprint per GPU (> L2)


def calls_for(msg_bytes: int, ranks_on_gpu: int = 1) -> int:
    """Back-to-back calls per graph so that distinct buffers exceed the L2."""
    per_call = 2 * msg_bytes * ranks_on_gpu
    return int(min(1000, max(50, -(-ROTATE_BYTES // per_call))))


def graph_of(fn: Callable[[int], None], calls: int, stream: torch.cuda.Stream):
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        for i in range(min(calls, 4)):
            fn(i)
    torch.cuda.current_stream().wait_stream(stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(calls):
            fn(i)
    torch.cuda.synchronize()
    return g


def time_replays(replay: Callable[[], None], steps: int, warmup: int,
                 barrier: Callable[[], None], stream: torch.cuda.Stream) -> List[float]:
    """Device ms of each of `steps` replays (after `warmup`), events on `stream`."""
    for _ in range(warmup):
        with torch.cuda.stream(stream):
            replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for a, b in ev:
            a.record(stream)
            replay()
            b.record(stream)
    torch.cuda.synchronize()
    barrier()
    return [a.elapsed_time(b) for a, b in ev]


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING a timed region: NVML every
    millisecond (the GPU found by its PCI bus id), else nvidia-smi every 0.2 s."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: List[tuple] = []  # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t: Optional[threading.Thread] = None
        self._nvml = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            import torch
            pr = torch.cuda.get_device_properties(index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self._h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            self._bits = {
                "hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
            }
            self._nvml = nv
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        self.rows.append((float(sm), float(mx), {k for k, b in self._bits.items() if bits & b}))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                              "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        if out:
            r = [c.strip() for c in out.split(",")]
            num = (lambda v: float(v) if v.replace(".", "").isdigit() else None)
            self.rows.append((num(r[1]), num(r[2]),
                              {self.NAMES[i] for i in range(4)
                               if len(r) > 3 + i and r[3 + i].lower() == "active"}))

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.001 if self._nvml is not None else 0.2)

    def _sample(self):
        try:
            if self._nvml is not None:
                self._sample_nvml()
            else:
                self._sample_smi()
        except Exception:
            pass

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        # a last sample at the end of the region (a short region may otherwise
        # see only the thread's first sample)
        if self._nvml is not None:
            self._sample()
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"],
                    "samples": 0}
        sm = [r[0] for r in self.rows if r[0] is not None]
        mx = [r[1] for r in self.rows if r[1] is not None]
        reasons = sorted(set().union(*(r[2] for r in self.rows)))
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self._nvml else "nvidia-smi"}


def alpha_signal_us(comm, rank: int, world: int, iters: int = 200, reps: int = 5,
                    group=None) -> Optional[float]:
    """One-way NVLink flag latency rank 0 <-> rank 1 (device ping-pong), p50 µs."""
    if world < 2:
        return None
    vals = []
    for _ in range(reps):
        dist.barrier(group)
        ns = ctypes.c_uint64()
        rc = 0
        if rank == 0:
            rc = comm._lib.nvrar_pingpong(comm._h, 1, iters, 1, None, ctypes.byref(ns))
        elif rank == 1:
            rc = comm._lib.nvrar_pingpong(comm._h, 0, iters, 0, None, ctypes.byref(ns))
        if rc:
            raise RuntimeError(comm.last_error())
        vals.append(ns.value / iters / 2 / 1e3 if rank == 0 else 0.0)
    out = D.max_over_ranks([statistics.median(vals)], group)
    return out[0]
