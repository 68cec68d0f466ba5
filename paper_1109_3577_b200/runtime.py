"""Execution strategies and run statistics (mirror of patchyhjb.runtime,
runtime.py:1-173).

The reference's Method 1 (batch-parallel Gauss-Seidel over threads) becomes
the CUDA grid of one cooperative launch; Method 2 (a task pool of patches)
becomes "all patches in one launch" on one GPU and an LPT split of patches
over ranks when ``torch.distributed`` is initialised (``dist.py``).
``ExecutionStrategy`` is kept for API compatibility; ``workers`` is ignored.
Phase timers use CUDA events on the current stream (device time).
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass, field

import torch

from .grid import ConfigurationError

import os

#: PHJ_SYNC_PHASES=1 times phases by host wall clock around device syncs
_SYNC_PHASES = os.environ.get("PHJ_SYNC_PHASES", "0") == "1"

SERIAL = "serial"
METHOD1 = "method1"
METHOD2 = "method2"
_KINDS = (SERIAL, METHOD1, METHOD2)


@dataclass(frozen=True)
class ExecutionStrategy:
    """How work is scheduled (runtime.py:39-60); accepted and validated."""

    kind: str = SERIAL
    workers: int = 1

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ConfigurationError(f"unknown strategy {self.kind!r}")
        if self.workers < 1:
            raise ConfigurationError("workers must be >= 1")
        if self.kind == SERIAL and self.workers != 1:
            raise ConfigurationError("serial strategy implies workers=1")

    @property
    def batch_parallel(self) -> bool:
        return self.kind == METHOD1 and self.workers > 1

    @property
    def task_parallel(self) -> bool:
        return self.kind == METHOD2 and self.workers > 1


@dataclass
class RunStats:
    """Work counters and per-phase device times for one run (runtime.py:63-93).

    ``phases`` holds seconds (like the reference) measured with CUDA events;
    call ``finalize()`` (done by run_patchy) to resolve pending events.
    ``performed_evals`` counts candidate evaluations the device really did."""

    node_relaxations: int = 0
    candidate_evals: int = 0
    transport_updates: int = 0
    sweeps: int = 0
    phases: dict = field(default_factory=dict)
    warnings: list = field(default_factory=list)
    speedup_vs_serial: float = None
    performed_evals: int = 0
    kernels: dict = field(default_factory=dict)
    _pending: list = field(default_factory=list, repr=False)

    @contextmanager
    def phase(self, name: str):
        if _SYNC_PHASES and torch.cuda.is_available():
            import time

            torch.cuda.synchronize()
            t0 = time.perf_counter()
            try:
                yield
            finally:
                torch.cuda.synchronize()
                self.phases[name] = self.phases.get(name, 0.0) + time.perf_counter() - t0
        elif torch.cuda.is_available():
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            try:
                yield
            finally:
                b.record()
                self._pending.append((name, a, b))
        else:
            import time

            t0 = time.perf_counter()
            try:
                yield
            finally:
                self.phases[name] = self.phases.get(name, 0.0) + time.perf_counter() - t0

    def finalize(self) -> "RunStats":
        if self._pending:
            torch.cuda.synchronize()
            for name, a, b in self._pending:
                self.phases[name] = self.phases.get(name, 0.0) + a.elapsed_time(b) / 1000.0
            self._pending.clear()
        return self

    def merge_counts(self, other):
        self.node_relaxations += getattr(other, "node_relaxations", 0)
        self.candidate_evals += getattr(other, "candidate_evals", 0)
        self.transport_updates += getattr(other, "transport_updates", 0)
        self.sweeps += getattr(other, "sweeps", 0)
        self.performed_evals += getattr(other, "performed_evals", 0)
        self.warnings.extend(getattr(other, "warnings", ()))

    def phases_ms(self) -> dict:
        self.finalize()
        return {k: 1000.0 * v for k, v in self.phases.items()}
