"""ctypes binding of libparcube_b200.so (the C-ABI declared in include/parcube_b200.h).

This module is the only place that touches the shared library.  It fails loudly:
a missing library or a missing CUDA device raises, nothing falls back to the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

MAX_DIM = 12
LIB_NAME = os.environ.get("PCB_LIB_NAME", "libparcube_b200.so")   # PCB_LIB_NAME: A/B builds in experiments
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

PCB_OK, PCB_NONFINITE, PCB_BUDGET, PCB_INVALID, PCB_CUDA, PCB_ABORTED = range(6)
RNG_REFERENCE_HASH, RNG_PHILOX, RNG_INJECTED = range(3)
ERR_MODES = {"two-level": 0, "max-null": 1, "max-pairwise": 2}
STOP_REASONS = ("tolerance met", "max iterations reached", "no active regions left", "region cap reached")
FAMILY_IDS = {"f1": 0, "f2": 1, "f3": 2, "f4": 3, "f5": 4, "f6": 5, "sum": 6, "one": 7}


class NativeError(RuntimeError):
    """CUDA / library level failure (status PCB_CUDA)."""


class NonFiniteStatus(Exception):
    """Internal carrier of a PCB_NONFINITE report; the API layers translate it."""

    def __init__(self, region_index, point_index, value, point, message):
        super().__init__(message)
        self.region_index, self.point_index, self.value, self.point = region_index, point_index, value, point


class BudgetStatus(Exception):
    """Internal carrier of PCB_BUDGET."""


# --------------------------------------------------------------------------- C structs
class IntegrandC(C.Structure):
    _fields_ = [("family", C.c_int32), ("d", C.c_int32), ("bounded", C.c_int32), ("reserved", C.c_int32),
                ("param", C.c_double * MAX_DIM), ("low", C.c_double * MAX_DIM), ("width", C.c_double * MAX_DIM),
                ("jac", C.c_double)]


class RuleC(C.Structure):
    _fields_ = [("d", C.c_int32), ("f_eval", C.c_int32), ("offsets", C.c_double * 7),
                ("weights", (C.c_double * 5) * 5), ("corner_parity", C.c_int32 * 5), ("reserved", C.c_int32),
                ("split_weights", C.c_double * 2), ("null_high", C.c_int32 * 4), ("null_scale", C.c_double * 4)]


class PaganiConfigC(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iterations", C.c_int32), ("group_size", C.c_int32),
                ("region_cap", C.c_int64), ("initial_regions", C.c_int32), ("err_mode", C.c_int32),
                ("rel_floor", C.c_double), ("abs_tol", C.c_double)]


class NonFiniteC(C.Structure):
    _fields_ = [("region_index", C.c_int64), ("point_index", C.c_int64), ("value", C.c_double),
                ("point", C.c_double * MAX_DIM)]


class PaganiProgressC(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("reserved", C.c_int32), ("n_regions", C.c_int64), ("active", C.c_int64),
                ("estimate", C.c_double), ("errorest", C.c_double)]


class PaganiResultC(C.Structure):
    _fields_ = [("estimate", C.c_double), ("errorest", C.c_double), ("iterations", C.c_int32),
                ("converged", C.c_int32), ("regions_processed", C.c_int64), ("reason", C.c_int32),
                ("n_records", C.c_int32), ("seconds_device", C.c_double), ("kernel_launches", C.c_int64)]


class McubesPlanC(C.Structure):
    _fields_ = [("d", C.c_int32), ("g", C.c_int32), ("p", C.c_int32), ("group_size", C.c_int32), ("m", C.c_int64),
                ("s", C.c_int64), ("n_bins", C.c_int32), ("reserved", C.c_int32)]


class McubesIterationC(C.Structure):
    _fields_ = [("integral", C.c_double), ("variance", C.c_double), ("n_samples", C.c_int64),
                ("clamp_events", C.c_int64)]


class McubesProgressC(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("reserved", C.c_int32), ("estimate", C.c_double), ("errorest", C.c_double),
                ("chi2_per_dof", C.c_double), ("iter_integral", C.c_double), ("iter_variance", C.c_double)]


class McubesShardBuffersC(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("row", C.c_void_p), ("gathered", C.c_void_p), ("table", C.c_void_p),
                ("row_doubles", C.c_int64), ("table_doubles", C.c_int64), ("thread_begin", C.c_int64),
                ("thread_end", C.c_int64)]


class PaganiShardRowsC(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("row", C.c_void_p), ("gathered", C.c_void_p), ("row_doubles", C.c_int64)]


PAGANI_PROGRESS_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(PaganiProgressC))
MCUBES_PROGRESS_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(McubesProgressC))

_DP = C.POINTER(C.c_double)
# every exported symbol of include/parcube_b200.h with its signature (tests check the list)
SIGNATURES = {
    "pcb_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "pcb_ctx_destroy": (None, [C.c_void_p]),
    "pcb_last_error": (C.c_char_p, [C.c_void_p]),
    "pcb_ctx_abort": (None, [C.c_void_p]),
    "pcb_ctx_reserve": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "pcb_device_info": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "pcb_launch_count": (C.c_int64, [C.c_void_p]),
    "pcb_measure_fp64_peak": (C.c_int, [C.c_void_p, _DP]),
    "pcb_profile_begin": (C.c_int, [C.c_void_p]),
    "pcb_profile_end": (C.c_int, [C.c_void_p, C.c_int32, _DP, C.POINTER(C.c_int64), _DP]),
    "pcb_eval_points": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.c_int64, C.c_void_p, C.c_void_p]),
    "pcb_qmc_shift_sums": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "pcb_bench_invoke": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.c_int64, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_void_p, _DP]),
    "pcb_pagani_evaluate": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.POINTER(RuleC), C.POINTER(PaganiConfigC),
                                      C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.POINTER(NonFiniteC)]),
    "pcb_pagani_evaluate_dev": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.POINTER(RuleC), C.POINTER(PaganiConfigC),
                                          C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.POINTER(NonFiniteC)]),
    "pcb_apply_rules": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(NonFiniteC)]),
    "pcb_pagani_refine": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.POINTER(RuleC), C.POINTER(PaganiConfigC),
                                    C.POINTER(PaganiResultC), C.POINTER(PaganiProgressC), PAGANI_PROGRESS_FN, C.c_void_p,
                                    C.POINTER(NonFiniteC)]),
    "pcb_tree_sum": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, _DP]),
    "pcb_pagani_shard_init": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.POINTER(RuleC), C.POINTER(PaganiConfigC),
                                        C.c_int32, C.c_int64, C.c_int64, C.POINTER(NonFiniteC)]),
    "pcb_pagani_shard_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pcb_pagani_shard_reduce": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                                          C.c_void_p, C.POINTER(C.c_int64)]),
    "pcb_pagani_shard_max_error": (C.c_int, [C.c_void_p, _DP]),
    "pcb_pagani_shard_classify": (C.c_int, [C.c_void_p, C.c_double, C.c_int32, C.c_double, C.POINTER(C.c_int64)]),
    "pcb_pagani_shard_split": (C.c_int, [C.c_void_p]),
    "pcb_pagani_shard_export": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    "pcb_pagani_shard_rebuild": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                           C.c_void_p, C.c_void_p]),
    "pcb_pagani_shard_evaluate": (C.c_int, [C.c_void_p, C.POINTER(NonFiniteC)]),
    "pcb_pagani_shard_deferred": (C.c_int, [C.c_void_p, C.c_int32]),
    "pcb_pagani_shard_pack": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int32,
                                        C.POINTER(PaganiShardRowsC)]),
    "pcb_pagani_shard_global_sums": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, _DP, C.POINTER(C.c_int32)]),
    "pcb_pagani_shard_nonfinite": (C.c_int, [C.c_void_p, C.POINTER(NonFiniteC)]),
    "pcb_pagani_shard_classify_dev": (C.c_int, [C.c_void_p, C.c_double, C.c_int32, C.c_double, C.c_int32, C.POINTER(C.c_void_p),
                                                C.POINTER(C.c_void_p)]),
    "pcb_pagani_shard_split_dev": (C.c_int, [C.c_void_p, C.c_int64]),
    "pcb_pagani_shard_list_dev": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int64)]),
    "pcb_pagani_shard_rebuild_dev": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]),
    "pcb_mcubes_sample": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.POINTER(McubesPlanC), C.c_void_p, C.c_uint64,
                                    C.c_int32, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.POINTER(McubesIterationC),
                                    C.c_void_p, C.c_void_p, C.POINTER(NonFiniteC)]),
    "pcb_mcubes_sample_cube": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.POINTER(McubesPlanC), C.c_void_p, C.c_int64,
                                         C.c_void_p, _DP, _DP, C.c_void_p, C.c_void_p, C.POINTER(NonFiniteC)]),
    "pcb_grid_refine": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_double, C.c_int32,
                                  C.c_void_p]),
    "pcb_mcubes_run": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.POINTER(McubesPlanC), C.c_int32, C.c_uint64,
                                 C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(McubesIterationC),
                                 C.POINTER(C.c_int32), MCUBES_PROGRESS_FN, C.c_void_p, C.c_void_p, C.c_void_p, _DP,
                                 C.POINTER(NonFiniteC)]),
    "pcb_mcubes_shard_begin": (C.c_int, [C.c_void_p, C.POINTER(IntegrandC), C.POINTER(McubesPlanC), C.c_int32, C.c_uint64,
                                         C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_double, C.c_double, C.c_int32,
                                         C.c_int32, C.c_int32, C.POINTER(McubesShardBuffersC)]),
    "pcb_mcubes_shard_pass": (C.c_int, [C.c_void_p, C.c_int32]),
    "pcb_mcubes_shard_finish": (C.c_int, [C.c_void_p, C.c_int32]),
    "pcb_mcubes_shard_wait": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(McubesIterationC), C.POINTER(C.c_int32),
                                        C.POINTER(NonFiniteC)]),
    "pcb_mcubes_shard_end": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, _DP]),
    "pcb_grid_transform": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p]),
    "pcb_debug_divide": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p]),
    "pcb_user_family_load": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.c_uint64, C.c_void_p]),
    "pcb_user_family_unload": (C.c_int, [C.c_void_p, C.c_int32]),
    "pcb_uniforms": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
}

_lib = None
_lock = threading.Lock()
_contexts: dict = {}


def load_library():
    """dlopen the in-tree library and bind every declared symbol; raises if anything is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} is missing: build it with `python -m paper_2302_05730_b200._build` "
                              "(nvcc, sm_100a). There is no CPU fallback.")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError if the symbol is not exported
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class Context:
    """One pcb_ctx (device, stream, scratch buffers).  One in-flight call at a time."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        handle = C.c_void_p()
        status = self.lib.pcb_ctx_create(int(device), C.byref(handle))
        self.handle = handle
        if status != PCB_OK:
            msg = self.last_error()
            if handle:
                self.lib.pcb_ctx_destroy(handle)
            self.handle = None
            raise NativeError(f"cannot create a B200 context on device {device}: {msg} (no CPU fallback exists)")
        self.device = int(device)
        self.call_lock = threading.Lock()
        # CUDA-event time of the most recent refine / mcubes_run on this context (reporting only: the public API
        # returns the reference's result types, which have no field for it)
        self.last_device_seconds = 0.0

    def last_error(self) -> str:
        if not self.handle:
            return "no context"
        return (self.lib.pcb_last_error(self.handle) or b"").decode(errors="replace")

    def close(self):
        if self.handle:
            self.lib.pcb_ctx_destroy(self.handle)
            self.handle = None

    def check(self, status: int, bad: NonFiniteC | None = None, d: int = 0):
        if status == PCB_OK:
            return
        msg = self.last_error()
        if status == PCB_NONFINITE:
            point = np.array(bad.point[:d]) if bad is not None else np.full(max(d, 1), np.nan)
            raise NonFiniteStatus(bad.region_index if bad is not None else None,
                                  bad.point_index if bad is not None else None,
                                  bad.value if bad is not None else float("nan"), point, msg)
        if status == PCB_BUDGET:
            raise BudgetStatus(msg)
        if status == PCB_INVALID:
            raise ValueError(msg)
        raise NativeError(msg)

    # ------------------------------------------------------------------ info
    def device_info(self):
        name = C.create_string_buffer(256)
        sms, khz = C.c_int32(), C.c_int32()
        self.check(self.lib.pcb_device_info(self.handle, name, 256, C.byref(sms), C.byref(khz)))
        return name.value.decode(), sms.value, khz.value

    def reserve(self, n_bytes: int) -> int:
        """Grow the context's device memory pool to at least n_bytes now; returns the pool size."""
        out = C.c_uint64()
        self.check(self.lib.pcb_ctx_reserve(self.handle, int(n_bytes), C.byref(out)))
        return int(out.value)

    def launch_count(self) -> int:
        return int(self.lib.pcb_launch_count(self.handle))

    def profile_begin(self):
        self.check(self.lib.pcb_profile_begin(self.handle))

    def profile_end(self, kind: int):
        """(kernel_ms, launches, units) of the evaluate (0) or V-Sample (1) launches since profile_begin."""
        ms, n, units = C.c_double(), C.c_int64(), C.c_double()
        self.check(self.lib.pcb_profile_end(self.handle, kind, C.byref(ms), C.byref(n), C.byref(units)))
        return ms.value, n.value, units.value

    def measure_fp64_peak(self) -> float:
        out = C.c_double()
        self.check(self.lib.pcb_measure_fp64_peak(self.handle, C.byref(out)))
        return out.value


def default_device() -> int:
    env = os.environ.get("PARCUBE_B200_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


def context(device: int | None = None) -> Context:
    """Process-wide context cache, one per device ordinal."""
    dev = default_device() if device is None else int(device)
    with _lock:
        ctx = _contexts.get(dev)
    if ctx is None:
        ctx = Context(dev)
        with _lock:
            _contexts.setdefault(dev, ctx)
            ctx = _contexts[dev]
    return ctx


# --------------------------------------------------------------------------- marshalling helpers
def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and out.shape != shape:
        raise ValueError(f"expected shape {shape}, got {out.shape}")
    return out


class DeviceSpec:
    """(family, d, params, optional bounds) -> pcb_integrand."""

    def __init__(self, family: str, d: int, param=(), low=None, width=None, jac=1.0):
        self.family, self.d = family, int(d)
        self.param = tuple(float(v) for v in param)
        self.low, self.width, self.jac = low, width, float(jac)

    @property
    def bounded(self) -> bool:
        return self.low is not None

    def with_bounds(self, low, width, jac) -> "DeviceSpec":
        return DeviceSpec(self.family, self.d, self.param, np.array(low, dtype=float), np.array(width, dtype=float), jac)

    def to_c(self) -> IntegrandC:
        c = IntegrandC()
        c.family, c.d, c.bounded = FAMILY_IDS[self.family], self.d, int(self.bounded)
        for i, v in enumerate(self.param):
            c.param[i] = v
        if self.bounded:
            for j in range(self.d):
                c.low[j], c.width[j] = float(self.low[j]), float(self.width[j])
        c.jac = self.jac
        return c


def rule_to_c(orbit) -> RuleC:
    c = RuleC()
    c.d, c.f_eval = orbit.d, orbit.f_eval
    for i in range(7):
        c.offsets[i] = float(orbit.offsets[i])
    for k in range(5):
        for o in range(5):
            c.weights[k][o] = float(orbit.weights[k, o])
        c.corner_parity[k] = int(orbit.corner_parity[k])
    c.split_weights[0], c.split_weights[1] = float(orbit.split_weights[0]), float(orbit.split_weights[1])
    for k in range(4):
        c.null_high[k] = int(orbit.high_mask[k])
        c.null_scale[k] = float(orbit.null_scales[k])
    return c


def pagani_config_to_c(cfg) -> PaganiConfigC:
    c = PaganiConfigC()
    c.rel_tol, c.max_iterations, c.group_size = float(cfg.rel_tol), int(cfg.max_iterations), int(cfg.group_size)
    c.region_cap, c.initial_regions = int(cfg.region_cap), int(cfg.initial_regions)
    c.err_mode, c.rel_floor = ERR_MODES[cfg.err_mode], float(cfg.rel_floor)
    c.abs_tol = float(getattr(cfg, "abs_tol", 0.0))
    return c


def plan_to_c(plan, n_bins: int) -> McubesPlanC:
    c = McubesPlanC()
    c.d, c.g, c.p, c.group_size, c.m, c.s, c.n_bins = plan.d, plan.g, plan.p, plan.group_size, plan.m, plan.s, int(n_bins)
    return c


# --------------------------------------------------------------------------- calls
def eval_points(spec: DeviceSpec, points: np.ndarray, device=None) -> np.ndarray:
    ctx = context(device)
    pts = _f64(points)
    out = np.empty(pts.shape[0], dtype=np.float64)
    fc = spec.to_c()
    with ctx.call_lock:
        ctx.check(ctx.lib.pcb_eval_points(ctx.handle, C.byref(fc), pts.shape[0], _ptr(pts), _ptr(out)))
    return out


def qmc_shift_sums(spec: DeviceSpec, log2_points: int, shifts: np.ndarray, device=None) -> np.ndarray:
    ctx = context(device)
    sh = _f64(shifts)
    out = np.empty(sh.shape[0])
    fc = spec.to_c()
    with ctx.call_lock:
        ctx.check(ctx.lib.pcb_qmc_shift_sums(ctx.handle, C.byref(fc), int(log2_points), sh.shape[0], _ptr(sh), _ptr(out)))
    return out


def tree_sum_1d(values: np.ndarray, device=None) -> float:
    ctx = context(device)
    v = _f64(values).ravel()
    out = C.c_double()
    with ctx.call_lock:
        ctx.check(ctx.lib.pcb_tree_sum(ctx.handle, v.size, _ptr(v), C.byref(out)))
    return out.value


def pagani_evaluate(spec: DeviceSpec, orbit, cfg, lefts: np.ndarray, lengths: np.ndarray, device=None):
    ctx = context(device)
    n, d = lefts.shape
    lefts, lengths = _f64(lefts), _f64(lengths)
    i_out, e_out = np.empty(n), np.empty(n)
    k_out = np.empty(n, dtype=np.int64)
    fc, rc, cc, bad = spec.to_c(), rule_to_c(orbit), pagani_config_to_c(cfg), NonFiniteC()
    with ctx.call_lock:
        st = ctx.lib.pcb_pagani_evaluate(ctx.handle, C.byref(fc), C.byref(rc), C.byref(cc), n, _ptr(lefts), _ptr(lengths),
                                         _ptr(i_out), _ptr(e_out), _ptr(k_out), C.byref(bad))
        ctx.check(st, bad, d)
    return i_out, e_out, k_out


def pagani_refine(spec: DeviceSpec, orbit, cfg, progress=None, device=None):
    ctx = context(device)
    fc, rc, cc, bad = spec.to_c(), rule_to_c(orbit), pagani_config_to_c(cfg), NonFiniteC()
    res = PaganiResultC()
    records = (PaganiProgressC * (int(cfg.max_iterations) + 1))()
    failure = []

    def _cb(_user, rec):
        if progress is None or failure:
            return
        try:
            r = rec.contents
            progress({"iteration": r.iteration, "n_regions": int(r.n_regions), "active": int(r.active),
                      "estimate": r.estimate, "errorest": r.errorest})
        except BaseException as exc:  # noqa: BLE001 - the driver stops at once; re-raised when the native call returns
            failure.append(exc)
            ctx.lib.pcb_ctx_abort(ctx.handle)

    cb = PAGANI_PROGRESS_FN(_cb) if progress is not None else C.cast(None, PAGANI_PROGRESS_FN)
    with ctx.call_lock:
        st = ctx.lib.pcb_pagani_refine(ctx.handle, C.byref(fc), C.byref(rc), C.byref(cc), C.byref(res), records, cb, None,
                                       C.byref(bad))
        if failure:
            raise failure[0]
        ctx.check(st, bad, spec.d)
        ctx.last_device_seconds = float(res.seconds_device)
    history = [(records[i].estimate, records[i].errorest, int(records[i].n_regions)) for i in range(res.n_records)]
    return res, history


def apply_rules_single(spec: DeviceSpec, rule, left, length, device=None):
    ctx = context(device)
    fc, bad = spec.to_c(), NonFiniteC()
    gen, w = _f64(rule.generators), _f64(rule.weights)
    left, length = _f64(left), _f64(length)
    values, fx = np.empty(5), np.empty(rule.f_eval)
    with ctx.call_lock:
        st = ctx.lib.pcb_apply_rules(ctx.handle, C.byref(fc), rule.f_eval, _ptr(gen), _ptr(w), _ptr(left), _ptr(length),
                                     _ptr(values), _ptr(fx), C.byref(bad))
        ctx.check(st, bad, spec.d)
    return values, fx


def mcubes_sample(spec: DeviceSpec, plan, boundaries: np.ndarray, seed: int, rng_kind: int = RNG_REFERENCE_HASH,
                  injected=None, squared_weighted: bool = True, thread_range=None, want_group_partials=False, device=None):
    ctx = context(device)
    d, nb = boundaries.shape[0], boundaries.shape[1] - 1
    b = _f64(boundaries)
    fc, pc, it, bad = spec.to_c(), plan_to_c(plan, nb), McubesIterationC(), NonFiniteC()
    t0, t1 = (0, plan.n_threads) if thread_range is None else thread_range
    contrib = np.empty((d, nb))
    n_groups = -(-(t1 - t0) // plan.group_size)
    partials = np.empty((n_groups, 2)) if want_group_partials else None
    inj = None if injected is None else _f64(injected).ravel()
    if inj is not None and inj.size != plan.m * plan.p * d:
        raise ValueError("injected uniforms must have m*p*d entries")
    with ctx.call_lock:
        st = ctx.lib.pcb_mcubes_sample(ctx.handle, C.byref(fc), C.byref(pc), _ptr(b), C.c_uint64(seed & (2**64 - 1)),
                                       rng_kind, None if inj is None else _ptr(inj), int(bool(squared_weighted)), t0, t1,
                                       C.byref(it), _ptr(contrib), None if partials is None else _ptr(partials),
                                       C.byref(bad))
        ctx.check(st, bad, d)
    return it, contrib, partials


def mcubes_sample_cube(spec: DeviceSpec, plan, boundaries: np.ndarray, cube_index: int, uniforms: np.ndarray, device=None):
    """(S1, S2, bins (p,d) int64, weights (p)) of one sub-cube from caller-drawn uniforms (mcubes.py:143-164)."""
    ctx = context(device)
    d, nb = boundaries.shape[0], boundaries.shape[1] - 1
    b, u = _f64(boundaries), _f64(uniforms, (plan.p, d))
    fc, pc, bad = spec.to_c(), plan_to_c(plan, nb), NonFiniteC()
    s1, s2 = C.c_double(), C.c_double()
    bins, weights = np.empty((plan.p, d), dtype=np.int64), np.empty(plan.p)
    with ctx.call_lock:
        st = ctx.lib.pcb_mcubes_sample_cube(ctx.handle, C.byref(fc), C.byref(pc), _ptr(b), int(cube_index), _ptr(u),
                                            C.byref(s1), C.byref(s2), _ptr(bins), _ptr(weights), C.byref(bad))
        ctx.check(st, bad, d)
    return s1.value, s2.value, bins, weights


def grid_refine(boundaries: np.ndarray, contributions: np.ndarray, alpha: float, smoothing: bool, device=None):
    ctx = context(device)
    d, nb1 = boundaries.shape
    b, c = _f64(boundaries), _f64(contributions, (d, nb1 - 1))
    out = np.empty_like(b)
    with ctx.call_lock:
        ctx.check(ctx.lib.pcb_grid_refine(ctx.handle, d, nb1 - 1, _ptr(b), _ptr(c), float(alpha), int(bool(smoothing)),
                                          _ptr(out)))
    return out


def mcubes_run(spec: DeviceSpec, plan, n_bins: int, iterations: int, seed: int, rng_kind: int, adapt: bool, alpha: float,
               smoothing: bool, rel_tol: float = 0.0, progress=None, keep_contributions=True, device=None, abs_tol: float = 0.0):
    ctx = context(device)
    d = plan.d
    fc, pc, bad = spec.to_c(), plan_to_c(plan, n_bins), NonFiniteC()
    its = (McubesIterationC * iterations)()
    n_done, seconds = C.c_int32(), C.c_double()
    contribs = np.empty((iterations, d, n_bins)) if keep_contributions else None
    final_b = np.empty((d, n_bins + 1))
    failure = []

    def _cb(_user, rec):
        if progress is None or failure:
            return
        try:
            r = rec.contents
            progress({"iteration": r.iteration, "estimate": r.estimate, "errorest": r.errorest,
                      "chi2_per_dof": r.chi2_per_dof, "iter_integral": r.iter_integral,
                      "iter_sd": float(np.sqrt(r.iter_variance))})
        except BaseException as exc:  # noqa: BLE001 - as in pagani_refine: stop the run, re-raise afterwards
            failure.append(exc)
            ctx.lib.pcb_ctx_abort(ctx.handle)

    # no Python trampoline per iteration unless somebody listens (each call back into Python costs ~10 us)
    cb = MCUBES_PROGRESS_FN(_cb) if progress is not None else C.cast(None, MCUBES_PROGRESS_FN)
    with ctx.call_lock:
        st = ctx.lib.pcb_mcubes_run(ctx.handle, C.byref(fc), C.byref(pc), int(iterations), C.c_uint64(seed & (2**64 - 1)),
                                    rng_kind, int(bool(adapt)), float(alpha), int(bool(smoothing)), float(rel_tol), float(abs_tol), its,
                                    C.byref(n_done), cb, None, None if contribs is None else _ptr(contribs),
                                    _ptr(final_b), C.byref(seconds), C.byref(bad))
        if failure:
            raise failure[0]
        ctx.check(st, bad, d)
        ctx.last_device_seconds = float(seconds.value)
    done = n_done.value
    return [its[i] for i in range(done)], (None if contribs is None else contribs[:done]), final_b, seconds.value


class DeviceArray:
    """A float64 device buffer of the library as a `__cuda_array_interface__` object: torch.as_tensor(view, device=...)
    aliases it without a copy, so the collectives of the sharded drivers run on the library's own buffers."""

    def __init__(self, ptr: int, count: int):
        self.ptr, self.count = int(ptr), int(count)
        self.__cuda_array_interface__ = {"shape": (self.count,), "typestr": "<f8", "data": (self.ptr, False),
                                         "version": 3, "strides": None}


class McubesShardRun:
    """One rank's side of a device-resident sharded m-Cubes run (pcb_mcubes_shard_*).  One live run per context."""

    def __init__(self, spec: DeviceSpec, plan, n_bins: int, iterations: int, seed: int, rng_kind: int, adapt: bool,
                 alpha: float, smoothing: bool, rel_tol: float, abs_tol: float, keep_tables: bool, rank: int, world: int,
                 device=None, ctx: "Context | None" = None):
        self.ctx = ctx or context(device)
        self.plan, self.n_bins, self.iterations, self.d = plan, int(n_bins), int(iterations), plan.d
        self.keep_tables = bool(keep_tables)
        fc, pc = spec.to_c(), plan_to_c(plan, n_bins)
        self.buffers = McubesShardBuffersC()
        with self.ctx.call_lock:
            self.ctx.check(self.ctx.lib.pcb_mcubes_shard_begin(
                self.ctx.handle, C.byref(fc), C.byref(pc), self.iterations, C.c_uint64(seed & (2**64 - 1)), int(rng_kind),
                int(bool(adapt)), float(alpha), int(bool(smoothing)), float(rel_tol), float(abs_tol), int(self.keep_tables),
                int(rank), int(world), C.byref(self.buffers)))
        b = self.buffers
        self.stream = int(b.stream or 0)
        self.row = DeviceArray(b.row, b.row_doubles)
        self.gathered = DeviceArray(b.gathered, b.row_doubles * world)
        self.table = DeviceArray(b.table, b.table_doubles)
        self.thread_range = (int(b.thread_begin), int(b.thread_end))

    def enqueue_pass(self, it: int):
        self.ctx.check(self.ctx.lib.pcb_mcubes_shard_pass(self.ctx.handle, int(it)))

    def enqueue_finish(self, it: int):
        self.ctx.check(self.ctx.lib.pcb_mcubes_shard_finish(self.ctx.handle, int(it)))

    def wait(self, it: int):
        """(record, stop) of iteration `it`; raises NonFiniteStatus on every rank alike."""
        rec, stop, bad = McubesIterationC(), C.c_int32(), NonFiniteC()
        self.ctx.check(self.ctx.lib.pcb_mcubes_shard_wait(self.ctx.handle, int(it), C.byref(rec), C.byref(stop), C.byref(bad)),
                       bad, self.d)
        return rec, bool(stop.value)

    def end(self, n_done: int):
        """(per-iteration tables or None, final boundaries, device seconds)."""
        contribs = np.empty((n_done, self.d, self.n_bins)) if self.keep_tables else None
        final_b = np.empty((self.d, self.n_bins + 1))
        secs = C.c_double()
        self.ctx.check(self.ctx.lib.pcb_mcubes_shard_end(self.ctx.handle, int(n_done), None if contribs is None else _ptr(contribs),
                                                         _ptr(final_b), C.byref(secs)))
        self.ctx.last_device_seconds = float(secs.value)
        return contribs, final_b, secs.value


def uniforms(seed: int, streams, counters, rng_kind: int = RNG_REFERENCE_HASH, device=None) -> np.ndarray:
    ctx = context(device)
    s = np.ascontiguousarray(np.broadcast_to(np.asarray(streams, dtype=np.uint64), np.broadcast(streams, counters).shape)).ravel()
    c = np.ascontiguousarray(np.broadcast_to(np.asarray(counters, dtype=np.uint64), np.broadcast(streams, counters).shape)).ravel()
    out = np.empty(s.size)
    with ctx.call_lock:
        ctx.check(ctx.lib.pcb_uniforms(ctx.handle, C.c_uint64(seed & (2**64 - 1)), rng_kind, s.size, _ptr(s), _ptr(c), _ptr(out)))
    return out


def grid_transform(boundaries: np.ndarray, y: np.ndarray, device=None):
    ctx = context(device)
    d, nb1 = boundaries.shape
    b, yy = _f64(boundaries), _f64(y)
    n = yy.shape[0]
    x, jac, bins = np.empty((n, d)), np.empty(n), np.empty((n, d), dtype=np.int64)
    with ctx.call_lock:
        ctx.check(ctx.lib.pcb_grid_transform(ctx.handle, d, nb1 - 1, _ptr(b), n, _ptr(yy), _ptr(x), _ptr(jac), _ptr(bins)))
    return x, jac, bins


def debug_divide(x: np.ndarray, g: int, device=None) -> np.ndarray:
    ctx = context(device)
    xx = _f64(x).ravel()
    out = np.empty_like(xx)
    with ctx.call_lock:
        ctx.check(ctx.lib.pcb_debug_divide(ctx.handle, xx.size, _ptr(xx), int(g), _ptr(out)))
    return out


class PaganiShard:
    """The local slice of a sharded PAGANI refinement, resident on one device (pcb_pagani_shard_*)."""

    TREE_SPAN = 1024

    def __init__(self, spec: DeviceSpec, orbit, cfg, device=None, ctx: "Context | None" = None):
        self.ctx = ctx or context(device)  # the shard state lives in the context: one shard per context
        self.d = spec.d
        self._f, self._r, self._c = spec.to_c(), rule_to_c(orbit), pagani_config_to_c(cfg)

    def _call(self, fn, *args, bad=None):
        with self.ctx.call_lock:
            self.ctx.check(fn(self.ctx.handle, *args), bad, self.d)

    def init(self, g: int, first: int, count: int):
        bad = NonFiniteC()
        self._call(self.ctx.lib.pcb_pagani_shard_init, C.byref(self._f), C.byref(self._r), C.byref(self._c), int(g),
                   int(first), int(count), C.byref(bad), bad=bad)

    def counts(self):
        a, r = C.c_int64(), C.c_int64()
        self._call(self.ctx.lib.pcb_pagani_shard_count, C.byref(a), C.byref(r))
        return a.value, r.value

    def reduce(self, which: int, head: int):
        n_active, n_ret = self.counts()
        n = n_active if which < 2 else n_ret
        head_vals, tail_vals = np.empty(self.TREE_SPAN), np.empty(self.TREE_SPAN)
        blocks = np.empty(n // self.TREE_SPAN + 1)
        nb, nt = C.c_int64(), C.c_int64()
        self._call(self.ctx.lib.pcb_pagani_shard_reduce, int(which), int(head), _ptr(head_vals), C.byref(nb), _ptr(blocks),
                   _ptr(tail_vals), C.byref(nt))
        return head_vals[: min(head, n)].copy(), blocks[: nb.value].copy(), tail_vals[: nt.value].copy()

    def max_error(self) -> float:
        out = C.c_double()
        self._call(self.ctx.lib.pcb_pagani_shard_max_error, C.byref(out))
        return out.value

    def classify(self, budget: float, mode: int, emax: float) -> int:
        out = C.c_int64()
        self._call(self.ctx.lib.pcb_pagani_shard_classify, float(budget), int(mode), float(emax), C.byref(out))
        return out.value

    def split(self):
        self._call(self.ctx.lib.pcb_pagani_shard_split)

    def export(self, begin: int, end: int):
        n = end - begin
        lefts, lengths = np.empty((n, self.d)), np.empty((n, self.d))
        self._call(self.ctx.lib.pcb_pagani_shard_export, int(begin), int(end), _ptr(lefts), _ptr(lengths))
        return lefts, lengths

    def rebuild(self, keep_begin, keep_end, front, back):
        fl, fh = (_f64(front[0]), _f64(front[1])) if front is not None and len(front[0]) else (None, None)
        bl, bh = (_f64(back[0]), _f64(back[1])) if back is not None and len(back[0]) else (None, None)
        self._call(self.ctx.lib.pcb_pagani_shard_rebuild, int(keep_begin), int(keep_end),
                   0 if fl is None else fl.shape[0], None if fl is None else _ptr(fl), None if fh is None else _ptr(fh),
                   0 if bl is None else bl.shape[0], None if bl is None else _ptr(bl), None if bh is None else _ptr(bh))

    def evaluate(self):
        bad = NonFiniteC()
        self._call(self.ctx.lib.pcb_pagani_shard_evaluate, C.byref(bad), bad=bad)

    def tree_sum(self, values) -> float:
        v = _f64(values).ravel()
        out = C.c_double()
        self._call(self.ctx.lib.pcb_tree_sum, v.size, _ptr(v), C.byref(out))
        return out.value

    # ---- device-collective mode (the product path of sharded.pagani_refine_sharded) --------------------------
    def deferred(self, on: bool = True):
        self._call(self.ctx.lib.pcb_pagani_shard_deferred, int(bool(on)))

    def pack(self, head_active: int, head_retired: int, with_retired: bool, width: int, world: int):
        """(stream, row, gathered) -- device views of this rank's packed row and of the all-gather target."""
        rows = PaganiShardRowsC()
        self._call(self.ctx.lib.pcb_pagani_shard_pack, int(head_active), int(head_retired), int(bool(with_retired)), int(width),
                   int(world), C.byref(rows))
        return int(rows.stream or 0), DeviceArray(rows.row, rows.row_doubles), DeviceArray(rows.gathered, rows.row_doubles * world)

    def global_sums(self, world: int, n_active_total: int, n_retired_total: int):
        sums, bad_rank = (C.c_double * 4)(), C.c_int32()
        self._call(self.ctx.lib.pcb_pagani_shard_global_sums, int(world), int(n_active_total), int(n_retired_total), sums,
                   C.byref(bad_rank))
        return [sums[i] for i in range(4)], int(bad_rank.value)

    def nonfinite(self):
        """(local region, point index, value, abscissa) of this rank's first non-finite evaluation."""
        bad = NonFiniteC()
        with self.ctx.call_lock:
            st = self.ctx.lib.pcb_pagani_shard_nonfinite(self.ctx.handle, C.byref(bad))
        if st != PCB_NONFINITE:
            self.ctx.check(st)
        return int(bad.region_index), int(bad.point_index), float(bad.value), np.array(bad.point[: self.d])

    def classify_dev(self, budget: float, mode: int, emax: float, world: int):
        row, gathered = C.c_void_p(), C.c_void_p()
        self._call(self.ctx.lib.pcb_pagani_shard_classify_dev, float(budget), int(mode), float(emax), int(world), C.byref(row),
                   C.byref(gathered))
        return DeviceArray(row.value, 2), DeviceArray(gathered.value, 2 * world)

    def split_dev(self, n_split: int):
        self._call(self.ctx.lib.pcb_pagani_shard_split_dev, int(n_split))

    def list_dev(self):
        """(lefts view, lengths view, n, ld): the local list, structure of arrays [d][ld] on the device."""
        lefts, lengths, n, ld = C.c_void_p(), C.c_void_p(), C.c_int64(), C.c_int64()
        self._call(self.ctx.lib.pcb_pagani_shard_list_dev, C.byref(lefts), C.byref(lengths), C.byref(n), C.byref(ld))
        return DeviceArray(lefts.value, self.d * ld.value), DeviceArray(lengths.value, self.d * ld.value), n.value, ld.value

    def rebuild_dev(self, keep_begin: int, keep_end: int, n_front: int, front_ptr: int, n_back: int, back_ptr: int):
        self._call(self.ctx.lib.pcb_pagani_shard_rebuild_dev, int(keep_begin), int(keep_end), int(n_front),
                   C.c_void_p(front_ptr or None), int(n_back), C.c_void_p(back_ptr or None))


def bench_invoke(spec: DeviceSpec, points: np.ndarray, blocks: int, threads: int, repetitions: int, device=None):
    ctx = context(device)
    pts = _f64(points)
    fc = spec.to_c()
    ms = np.empty(repetitions)
    acc = C.c_double()
    with ctx.call_lock:
        ctx.check(ctx.lib.pcb_bench_invoke(ctx.handle, C.byref(fc), pts.shape[0], _ptr(pts), int(blocks), int(threads),
                                           int(repetitions), _ptr(ms), C.byref(acc)))
    return ms, acc.value
