"""Execution configuration and the fixed-shape reductions of the integrate API.

Mirror of the reference's engine layer (reference: pkg/src/parcube/engine.py).  The thread
pool itself is what the GPU replaces: `ExecConfig.workers/chunk` are accepted and ignored
(they never change results in the reference either, engine.py:36-41); the reductions run
on the device with the reference's tree shape (engine.py:69-86).
"""

from __future__ import annotations

import os

import numpy as np

from . import _native
from .domain import _Frozen

WORKERS_ENV_VAR = "PARCUBE_WORKERS"
DETERMINISTIC_TREE = "deterministic-tree"
UNORDERED = "unordered"


class GroupTaskError(RuntimeError):
    """A work item failed; carries the lowest failing group id (engine.py:25-31)."""

    def __init__(self, group_id: int, cause: BaseException):
        self.group_id = group_id
        self.cause = cause
        super().__init__(f"task for group {group_id} failed: {cause!r}")


class ExecConfig(_Frozen):
    """workers (0 = auto), determinism flag, chunk (engine.py:34-66).

    `device` (extension) selects the CUDA ordinal; default LOCAL_RANK or 0.
    """

    __slots__ = ("workers", "deterministic", "chunk", "device")

    def __init__(self, workers: int = 0, deterministic: bool = True, chunk: int = 0, device=None):
        if workers < 0:
            raise ValueError("workers must be >= 0")
        self._put("workers", int(workers))
        self._put("deterministic", bool(deterministic))
        self._put("chunk", int(chunk))
        self._put("device", device)

    def resolve_workers(self) -> int:
        if self.workers > 0:
            return self.workers
        env = os.environ.get(WORKERS_ENV_VAR)
        if env:
            try:
                n = int(env)
            except ValueError:
                raise ValueError(f"{WORKERS_ENV_VAR} must be an integer, got {env!r}")
            if n > 0:
                return n
        return os.cpu_count() or 1

    @property
    def reduction_mode(self) -> str:
        return DETERMINISTIC_TREE if self.deterministic else UNORDERED


def tree_sum(values, axis: int = -1):
    """Adjacent-pair tree sum along `axis`, odd levels zero-padded (engine.py:69-86); on the device."""
    a = np.asarray(values, dtype=np.float64)
    if a.ndim == 1:
        return 0.0 if a.size == 0 else _native.tree_sum_1d(a)
    moved = np.moveaxis(a, axis, -1)
    flat = moved.reshape(-1, moved.shape[-1])
    out = np.array([_native.tree_sum_1d(row) for row in flat])
    return out.reshape(moved.shape[:-1])


def reduce(values, mode: str = DETERMINISTIC_TREE) -> float:
    """Sum of a list of reals, 0 for empty input (engine.py:89-103).  Both modes use the
    device tree: `unordered` promises no order, so the fixed tree is a valid instance."""
    if mode not in (DETERMINISTIC_TREE, UNORDERED):
        raise ValueError(f"unknown reduction mode {mode!r}")
    a = np.asarray(values, dtype=np.float64).ravel()
    return tree_sum(a) if a.size else 0.0


class _Accumulator:
    """Indexed accumulation handle of the reference's engine (engine.py:181-253): `add(index, value, stream)`,
    `add_array(values, stream)`, `snapshot()`.  The integrators do not use it -- their accumulation is the
    V-Sample kernel's shared-memory table -- but host callers of the reference API do.  Deterministic mode keeps
    one partial buffer per logical stream and merges them in ascending stream order with the device pair tree
    (`tree_sum`, engine.py:217-220); unordered mode is one shared buffer."""

    def __init__(self, size, per_stream: bool):
        import threading
        self._shape = (int(size),) if np.isscalar(size) else tuple(int(v) for v in size)
        self._per_stream = per_stream
        self._bufs: dict = {}
        self._lock = threading.Lock()

    def _buf(self, stream):
        key = stream if self._per_stream else 0
        with self._lock:
            return self._bufs.setdefault(key, np.zeros(self._shape))

    def add(self, index, value, stream=0):
        buf = self._buf(stream)
        with self._lock:
            buf[index] += value

    def add_array(self, values, stream=0):
        values = np.asarray(values, dtype=float)
        if values.shape != self._shape:
            raise IndexError(f"expected shape {self._shape}, got {values.shape}")
        buf = self._buf(stream)
        with self._lock:
            buf += values

    def snapshot(self) -> np.ndarray:
        with self._lock:
            parts = [self._bufs[k].copy() for k in sorted(self._bufs)]
        if not parts:
            return np.zeros(self._shape)
        return tree_sum(np.stack(parts, axis=0), axis=0) if len(parts) > 1 else parts[0]


class DeterministicAccumulator(_Accumulator):
    def __init__(self, size):
        super().__init__(size, per_stream=True)


class UnorderedAccumulator(_Accumulator):
    def __init__(self, size):
        super().__init__(size, per_stream=False)


def accumulator(size, mode: str = DETERMINISTIC_TREE):
    """Shared accumulation handle for an index space (engine.py:247-253)."""
    if mode == DETERMINISTIC_TREE:
        return DeterministicAccumulator(size)
    if mode == UNORDERED:
        return UnorderedAccumulator(size)
    raise ValueError(f"unknown accumulation mode {mode!r}")


def parallel_for_groups(n_groups: int, task, cfg: ExecConfig | None = None) -> list:
    """task(group_id) for every id, results in id order (engine.py:106-161).

    Kept for API compatibility with host-side callers; the integrators do not use it --
    their work-groups are CUDA thread blocks.  Runs serially; the first failure is wrapped
    in GroupTaskError with its group id, as in the reference.
    """
    n_groups = int(n_groups)
    if n_groups < 0:
        raise ValueError("n_groups must be >= 0")
    out = []
    for gid in range(n_groups):
        try:
            out.append(task(gid))
        except Exception as exc:  # noqa: BLE001
            raise GroupTaskError(gid, exc) from exc
    return out
