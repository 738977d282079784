"""ctypes binding of include/recon_b200.h.

One `ReconLib` wraps any shared library that exports the C-ABI: the product
library (paper_2504_06182_b200/lib/librecon_b200.so, CUDA), and — for tests
and bench baselines only — the C oracle (oracle/librecon_oracle.so) and the
compiled reference (oracle/_ref/librecon_ref.so).  Methods take and return
numpy arrays; statuses are raised as the reference's exception types
(geometry.hpp:18-30).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
U64P = C.POINTER(C.c_uint64)

RECON_OK = 0
RECON_ERR_INPUT = 1
RECON_ERR_INFEASIBLE = 2
RECON_ERR_COLLISION = 3
RECON_ERR_LOGIC = 4
RECON_ERR_CAPACITY = 5
RECON_ERR_CUDA = 6
RECON_ERR_ARGUMENT = 7

PRESET_NONE = 0
PRESET_COLUMN_DIRECTION = 1

DETAIL_MESSAGES = {
    1: "fewer sources than targets (|S| < |T|)",
    2: "targets must form a centered full-width band",
    3: "target band height must be in (0, H)",
    4: "target band is empty",
    5: "select_best_pair: no deficit column remains",
    6: "select_best_pair: deficit column with no admissible donor",
    7: "batching made no progress (blocked dependency structure)",
    8: "batching requires an acyclic dependency dag",
    9: "chain length must be positive",
    10: "source vertex out of bounds",
    11: "source vertices must be strictly increasing",
    12: "target vertex out of bounds",
    13: "target vertices must be strictly increasing",
    14: "source multiplicity must be at least 1",
    15: "source min_use outside [0, multiplicity]",
    16: "source positions must be strictly increasing",
    17: "target positions must be strictly increasing",
    18: "insufficient tokens for targets",
    19: "mandatory draws exceed target count",
    20: "no assignment satisfies the usage bounds",
    21: "dag edge endpoint out of range",
    22: "grid dimensions must be positive",
    23: "fewer sources than targets",
    24: "CUDA runtime failure",
}


class ReconError(RuntimeError):
    status = -1

    def __init__(self, msg: str, detail: int = 0):
        super().__init__(msg)
        self.detail = detail


class InputError(ReconError):
    """recon::InputError (geometry.hpp:19-21)."""
    status = RECON_ERR_INPUT


class InfeasibleError(ReconError):
    """recon::InfeasibleError (geometry.hpp:24-26)."""
    status = RECON_ERR_INFEASIBLE


class CollisionError(ReconError):
    """recon::CollisionError (geometry.hpp:28-30)."""
    status = RECON_ERR_COLLISION


class LogicError(ReconError):
    """std::logic_error (redrec.cpp:82-84)."""
    status = RECON_ERR_LOGIC


class CapacityError(ReconError):
    status = RECON_ERR_CAPACITY


class CudaError(ReconError):
    status = RECON_ERR_CUDA


_EXC = {
    RECON_ERR_INPUT: InputError,
    RECON_ERR_INFEASIBLE: InfeasibleError,
    RECON_ERR_COLLISION: CollisionError,
    RECON_ERR_LOGIC: LogicError,
    RECON_ERR_CAPACITY: CapacityError,
    RECON_ERR_CUDA: CudaError,
    RECON_ERR_ARGUMENT: ReconError,
}


def raise_status(status: int, detail: int = 0, extra: str = ""):
    if status == RECON_OK:
        return
    cls = _EXC.get(status, ReconError)
    msg = DETAIL_MESSAGES.get(detail, f"status {status}")
    if extra:
        msg = f"{msg} ({extra})"
    raise cls(msg, detail)


class GridSolution(C.Structure):
    _fields_ = [
        ("path_src", I32P), ("path_dst", I32P), ("path_event", I32P),
        ("path_capacity", C.c_int64), ("path_count", C.c_int64),
        ("displaced_tokens", C.c_int64), ("total_displacement", C.c_int64),
        ("events", I32P), ("event_capacity", C.c_int32), ("event_count", C.c_int32),
        ("dag_src", I32P), ("dag_dst", I32P), ("dag_capacity", C.c_int64), ("dag_count", C.c_int64),
    ]


class GridBatch(C.Structure):
    _fields_ = [
        ("occ", C.c_void_p), ("count", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
        ("h_prime", C.c_int32), ("path_src", C.c_void_p), ("path_dst", C.c_void_p),
        ("path_event", C.c_void_p), ("path_count", C.c_void_p), ("total_displacement", C.c_void_p),
        ("status", C.c_void_p), ("detail", C.c_void_p), ("events", C.c_void_p),
    ]


class ChainBatch(C.Structure):
    _fields_ = [
        ("occ", C.c_void_p), ("count", C.c_int32), ("n", C.c_int32), ("t_lo", C.c_int32),
        ("t_hi", C.c_int32), ("path_src", C.c_void_p), ("path_dst", C.c_void_p),
        ("total_displacement", C.c_void_p), ("displaced", C.c_void_p), ("status", C.c_void_p),
        ("detail", C.c_void_p),
    ]


class PipelineBatch(C.Structure):
    _fields_ = [
        ("grid", GridBatch), ("solver", C.c_int32), ("preset", C.c_int32),
        ("move_stride", C.c_int64), ("move_batch", C.c_void_p), ("batch_count", C.c_void_p),
    ]


class InstanceStats(C.Structure):
    """recon_instance_stats (include/recon_b200.h)."""
    _fields_ = [
        ("status", C.c_int32), ("detail", C.c_int32), ("path_count", C.c_int32), ("displaced_tokens", C.c_int32),
        ("total_displacement", C.c_int64), ("batch_count", C.c_int64), ("digest", C.c_uint64),
    ]


STATS_DTYPE = np.dtype([("status", np.int32), ("detail", np.int32), ("path_count", np.int32),
                        ("displaced_tokens", np.int32), ("total_displacement", np.int64),
                        ("batch_count", np.int64), ("digest", np.uint64)])
assert STATS_DTYPE.itemsize == C.sizeof(InstanceStats) == 40


class ScheduleRuns(C.Structure):
    """recon_schedule_runs (include/recon_b200.h)."""
    _fields_ = [("run_stride", C.c_int64), ("run_slot", C.c_void_p), ("run_batch", C.c_void_p),
                ("run_count", C.c_void_p)]


def expand_runs(run_slot, run_batch, nruns: int, D: int) -> np.ndarray:
    """move_batch[0, D) of one instance from its runs."""
    out = np.empty(D, np.int32)
    s = np.asarray(run_slot[:nruns], np.int64)
    ends = np.append(s[1:], D)
    for a, e, b in zip(s, ends, np.asarray(run_batch[:nruns], np.int64)):
        out[a:e] = b + np.arange(e - a)
    return out


class ValidateBatch(C.Structure):
    _fields_ = [
        ("occ", C.c_void_p), ("count", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
        ("h_prime", C.c_int32), ("path_src", C.c_void_p), ("path_dst", C.c_void_p), ("path_stride", C.c_int64),
        ("path_count", C.c_void_p), ("total_displacement", C.c_void_p), ("displaced", C.c_void_p),
        ("dag_mode", C.c_int32), ("dag_a", C.c_void_p), ("dag_b", C.c_void_p), ("dag_offset", C.c_void_p),
        ("move_batch", C.c_void_p), ("move_stride", C.c_int64), ("batch_count", C.c_void_p),
        ("preset", C.c_int32), ("verdict", C.c_void_p),
    ]


class LossModel(C.Structure):
    _fields_ = [("p_nu", C.c_double), ("p_alpha", C.c_double), ("tau", C.c_double), ("t_nu", C.c_double),
                ("t_alpha", C.c_double), ("t_meas", C.c_double)]


class SimBatch(C.Structure):
    _fields_ = [
        ("occ", C.c_void_p), ("count", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
        ("h_prime", C.c_int32), ("seed_base", C.c_uint64), ("solver", C.c_int32), ("batching", C.c_int32),
        ("preset", C.c_int32), ("max_cycles", C.c_int32), ("loss", LossModel),
        ("success", C.c_void_p), ("cycles", C.c_void_p), ("status", C.c_void_p), ("n_nu", C.c_void_p),
        ("n_alpha", C.c_void_p), ("nb_nu", C.c_void_p), ("nb_alpha", C.c_void_p), ("atoms_lost", C.c_void_p),
        ("elapsed", C.c_void_p),
    ]


# recon_verdict bits (include/recon_b200.h)
VERDICT_BITS = {
    "PATH_BOUNDS": 1 << 0, "SHARED_SOURCE": 1 << 1, "SHARED_TARGET": 1 << 2, "DAG_CYCLE": 1 << 3,
    "STATS_DISPLACEMENT": 1 << 4, "STATS_DISPLACED": 1 << 5, "EXECUTION": 1 << 6, "TARGETS": 1 << 7,
    "DAG_ORDER": 1 << 8, "TOKEN_EMPTY": 1 << 9, "TOKEN_SECOND_PATH": 1 << 10, "BATCH_CONSERVATION": 1 << 11,
    "BATCH_BOUND": 1 << 12, "BATCH_EMPTY": 1 << 13, "BATCH_DISJOINT": 1 << 14, "BATCH_CONSTRAINT": 1 << 15,
    "BATCH_COLLISION": 1 << 16, "BATCH_TARGETS": 1 << 17, "BATCH_DAG": 1 << 18, "BATCH_ORDER": 1 << 19,
    "TOKEN_MATCH": 1 << 20,
}
DAG_NONE, DAG_EXPLICIT, DAG_OCCUPANCY = 0, 1, 2


def verdict_names(v: int) -> list:
    return [k for k, b in VERDICT_BITS.items() if v & b] + (["UNMAPPED"] if v & (1 << 31) else [])


EXPORTED_SYMBOLS = [
    "recon_detail_message", "recon_last_cuda_error", "recon_abi_version",
    "recon_ctx_create", "recon_ctx_destroy", "recon_ctx_stream", "recon_ctx_launch_count",
    "recon_ctx_set_kernel_timing", "recon_ctx_kernel_times",
    "recon_redrec_solve", "recon_bird_solve", "recon_occupancy_dag",
    "recon_redrec_solve_batch", "recon_bird_solve_batch",
    "recon_redrec_solve_batch_host", "recon_bird_solve_batch_host",
    "recon_redrec_solve_batch_host_packed", "recon_bird_solve_batch_host_packed",
    "recon_assign_1d", "recon_assign_1d_generalized", "recon_solve_1d",
    "recon_solve_1d_batch", "recon_solve_1d_batch_host",
    "recon_batch_moves", "recon_pipeline_batch_run", "recon_pipeline_batch_run_host",
    "recon_validate_batch_run", "recon_validate_batch_run_host",
    "recon_solution_json", "recon_solution_json_host", "recon_batch_schedule_json",
    "recon_batch_schedule_json_host",
    "recon_sim_run_host",
]


def _ptr(a, typ):
    return a.ctypes.data_as(typ) if a is not None else C.cast(None, typ)


def _vp(a):
    return C.c_void_p(a.ctypes.data) if a is not None else C.c_void_p(None)


def words_per_column(h: int) -> int:
    return (h + 63) // 64


@dataclass
class GridResult:
    path_src: np.ndarray
    path_dst: np.ndarray
    path_event: np.ndarray
    displaced_tokens: int
    total_displacement: int
    events: np.ndarray
    dag: np.ndarray | None  # (E, 2) int32


@dataclass
class ChainResult:
    path_src: np.ndarray
    path_dst: np.ndarray
    path_order: np.ndarray
    dag: np.ndarray | None
    total_displacement: int
    displaced: int


class ReconLib:
    """numpy-level wrapper around one library exporting include/recon_b200.h."""

    def __init__(self, path: str, name: str | None = None):
        self.path = os.path.abspath(path)
        self.name = name or os.path.basename(path)
        self.lib = C.CDLL(self.path)
        L = self.lib
        L.recon_ctx_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
        L.recon_ctx_create.restype = C.c_int
        L.recon_ctx_destroy.argtypes = [C.c_void_p]
        L.recon_ctx_destroy.restype = None
        L.recon_ctx_stream.argtypes = [C.c_void_p]
        L.recon_ctx_stream.restype = C.c_void_p
        L.recon_ctx_launch_count.argtypes = [C.c_void_p]
        L.recon_ctx_launch_count.restype = C.c_int64
        L.recon_ctx_set_kernel_timing.argtypes = [C.c_void_p, C.c_int32]
        L.recon_ctx_kernel_times.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        L.recon_last_cuda_error.restype = C.c_char_p
        L.recon_abi_version.restype = C.c_int32
        for fn in ("recon_redrec_solve", "recon_bird_solve"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, U64P, C.c_int32, C.c_int32, C.c_int32,
                          C.POINTER(GridSolution), I32P]
            f.restype = C.c_int
        L.recon_occupancy_dag.argtypes = [C.c_void_p, C.c_int32, C.c_int32, I32P, I32P, C.c_int64,
                                          I32P, I32P, C.c_int64, I64P, I32P]
        L.recon_occupancy_dag.restype = C.c_int
        for fn in ("recon_redrec_solve_batch", "recon_bird_solve_batch",
                   "recon_redrec_solve_batch_host", "recon_bird_solve_batch_host"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, C.POINTER(GridBatch)]
            f.restype = C.c_int
        for fn in ("recon_redrec_solve_batch_host_packed", "recon_bird_solve_batch_host_packed"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, C.POINTER(GridBatch), C.c_void_p]
            f.restype = C.c_int
        L.recon_assign_1d.argtypes = [C.c_void_p, C.c_int32, I32P, C.c_int32, I32P, C.c_int32,
                                      I64P, I64P, I64P, I32P, I32P]
        L.recon_assign_1d.restype = C.c_int
        L.recon_assign_1d_generalized.argtypes = [C.c_void_p, C.c_int32, I64P, I32P, I32P,
                                                  C.c_int32, I64P, I64P, I64P, I64P, I32P, I32P]
        L.recon_assign_1d_generalized.restype = C.c_int
        L.recon_solve_1d.argtypes = [C.c_void_p, C.c_int32, I32P, C.c_int32, I32P, C.c_int32,
                                     I32P, I32P, I32P, I32P, I32P, C.c_int64, I64P, I64P, I32P, I32P]
        L.recon_solve_1d.restype = C.c_int
        for fn in ("recon_solve_1d_batch", "recon_solve_1d_batch_host"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, C.POINTER(ChainBatch)]
            f.restype = C.c_int
        L.recon_batch_moves.argtypes = [C.c_void_p, C.c_int32, C.c_int32, U64P, C.c_int32, I64P,
                                        I32P, C.c_int64, I32P, I32P, C.c_int32, C.c_int32, I32P,
                                        I64P, I32P]
        L.recon_batch_moves.restype = C.c_int
        for fn in ("recon_pipeline_batch_run", "recon_pipeline_batch_run_host"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, C.POINTER(PipelineBatch)]
            f.restype = C.c_int
        L.recon_pipeline_stats.argtypes = [C.c_void_p, C.POINTER(PipelineBatch), C.c_void_p]
        L.recon_pipeline_stats.restype = C.c_int
        for fn in ("recon_pipeline_schedule_runs", "recon_pipeline_batch_run_host_runs"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, C.POINTER(PipelineBatch), C.POINTER(ScheduleRuns)]
            f.restype = C.c_int
        for fn in ("recon_solution_json", "recon_solution_json_host"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                          C.POINTER(C.c_int64)]
            f.restype = C.c_int
        for fn in ("recon_batch_schedule_json", "recon_batch_schedule_json_host"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
            f.restype = C.c_int
        L.recon_sim_run_host.argtypes = [C.c_void_p, C.POINTER(SimBatch)]
        L.recon_sim_run_host.restype = C.c_int
        for fn in ("recon_validate_batch_run", "recon_validate_batch_run_host"):
            f = getattr(L, fn)
            f.argtypes = [C.c_void_p, C.POINTER(ValidateBatch)]
            f.restype = C.c_int
        self._ctx = None

    # -- context -----------------------------------------------------------
    def ctx(self, device: int = 0):
        if self._ctx is None:
            h = C.c_void_p()
            st = self.lib.recon_ctx_create(device, C.byref(h))
            if st != RECON_OK:
                raise_status(st, 24, self.last_cuda_error())
            self._ctx = h
        return self._ctx

    def last_cuda_error(self) -> str:
        return (self.lib.recon_last_cuda_error() or b"").decode()

    def launch_count(self) -> int:
        return int(self.lib.recon_ctx_launch_count(self.ctx()))

    def set_kernel_timing(self, enable: bool) -> None:
        self.lib.recon_ctx_set_kernel_timing(self.ctx(), 1 if enable else 0)

    def kernel_times(self) -> tuple:
        """(planner ms, executor ms) of the last grid solve (timing enabled)."""
        ms = (C.c_float * 2)()
        self.lib.recon_ctx_kernel_times(self.ctx(), ms, 2)
        return float(ms[0]), float(ms[1])

    def close(self):
        if self._ctx is not None:
            self.lib.recon_ctx_destroy(self._ctx)
            self._ctx = None

    def _check(self, st: int, det: C.c_int32 | int):
        d = det.value if isinstance(det, C.c_int32) else int(det)
        extra = self.last_cuda_error() if st == RECON_ERR_CUDA else ""
        raise_status(st, d, extra)

    # -- grid --------------------------------------------------------------
    def grid_solve(self, solver: str, occ: np.ndarray, width: int, height: int, h_prime: int,
                   with_dag: bool = False) -> GridResult:
        occ = np.ascontiguousarray(occ, dtype=np.uint64)
        cap = max(1, width * max(h_prime, 0))
        src = np.zeros(cap, np.int32)
        dst = np.zeros(cap, np.int32)
        ev = np.zeros(cap, np.int32)
        per = 4 if solver == "redrec" else 1
        events = np.zeros(max(1, width) * per, np.int32)
        out = GridSolution()
        out.path_src, out.path_dst, out.path_event = _ptr(src, I32P), _ptr(dst, I32P), _ptr(ev, I32P)
        out.path_capacity = cap
        out.events, out.event_capacity = _ptr(events, I32P), events.size
        dag = None
        if with_dag:
            dcap = 1 << 16
        while True:
            if with_dag:
                ds = np.zeros(dcap, np.int32)
                dd = np.zeros(dcap, np.int32)
                out.dag_src, out.dag_dst, out.dag_capacity = _ptr(ds, I32P), _ptr(dd, I32P), dcap
            det = C.c_int32(0)
            fn = self.lib.recon_redrec_solve if solver == "redrec" else self.lib.recon_bird_solve
            st = fn(self.ctx(), _ptr(occ, U64P), width, height, h_prime, C.byref(out), C.byref(det))
            if with_dag and st == RECON_ERR_CAPACITY and out.dag_count > dcap:
                dcap = int(out.dag_count)
                continue
            break
        self._check(st, det)
        n = int(out.path_count)
        if with_dag:
            m = int(out.dag_count)
            dag = np.stack([ds[:m], dd[:m]], axis=1)
        return GridResult(src[:n].copy(), dst[:n].copy(), ev[:n].copy(), int(out.displaced_tokens),
                          int(out.total_displacement), events[: int(out.event_count) * per].copy(), dag)

    def occupancy_dag(self, width, height, src, dst) -> np.ndarray:
        src = np.ascontiguousarray(src, np.int32)
        dst = np.ascontiguousarray(dst, np.int32)
        cap = max(16, 4 * len(src))
        while True:
            a = np.zeros(cap, np.int32)
            b = np.zeros(cap, np.int32)
            cnt = C.c_int64(0)
            det = C.c_int32(0)
            st = self.lib.recon_occupancy_dag(self.ctx(), width, height, _ptr(src, I32P), _ptr(dst, I32P),
                                              len(src), _ptr(a, I32P), _ptr(b, I32P), cap,
                                              C.byref(cnt), C.byref(det))
            if st == RECON_ERR_CAPACITY and cnt.value > cap:
                cap = int(cnt.value)
                continue
            self._check(st, det)
            m = int(cnt.value)
            return np.stack([a[:m], b[:m]], axis=1)

    def grid_solve_batch(self, solver: str, occ: np.ndarray, count: int, width: int, height: int,
                         h_prime: int, host: bool = True, with_events: bool = True):
        """Batched solve through the *_batch_host entry point (host buffers)."""
        stride = width * h_prime
        out = {
            "path_src": np.zeros(count * stride, np.int32),
            "path_dst": np.zeros(count * stride, np.int32),
            "path_event": np.zeros(count * stride, np.int32),
            "path_count": np.zeros(count, np.int32),
            "total_displacement": np.zeros(count, np.int64),
            "status": np.zeros(count, np.int32),
            "detail": np.zeros(count, np.int32),
            "events": np.zeros(count * width * (4 if solver == "redrec" else 1), np.int32)
            if with_events else None,
        }
        occ = np.ascontiguousarray(occ, np.uint64)
        b = GridBatch(_vp(occ).value, count, width, height, h_prime, _vp(out["path_src"]).value,
                      _vp(out["path_dst"]).value, _vp(out["path_event"]).value,
                      _vp(out["path_count"]).value, _vp(out["total_displacement"]).value,
                      _vp(out["status"]).value, _vp(out["detail"]).value, _vp(out["events"]).value)
        if solver == "redrec":
            fn = self.lib.recon_redrec_solve_batch_host if host else self.lib.recon_redrec_solve_batch
        else:
            fn = self.lib.recon_bird_solve_batch_host if host else self.lib.recon_bird_solve_batch
        st = fn(self.ctx(), C.byref(b))
        self._check(st, 0)
        return out

    def grid_solve_batch_packed(self, solver: str, occ: np.ndarray, count: int, width: int, height: int,
                                h_prime: int):
        """Batched solve through *_batch_host_packed: path_packed[i] = src | dst << 16."""
        stride = width * h_prime
        out = {
            "path_packed": np.zeros(count * stride, np.uint32),
            "path_count": np.zeros(count, np.int32),
            "total_displacement": np.zeros(count, np.int64),
            "status": np.zeros(count, np.int32),
            "detail": np.zeros(count, np.int32),
        }
        occ = np.ascontiguousarray(occ, np.uint64)
        b = GridBatch(_vp(occ).value, count, width, height, h_prime, None, None, None,
                      _vp(out["path_count"]).value, _vp(out["total_displacement"]).value,
                      _vp(out["status"]).value, _vp(out["detail"]).value, None)
        fn = (self.lib.recon_redrec_solve_batch_host_packed if solver == "redrec"
              else self.lib.recon_bird_solve_batch_host_packed)
        st = fn(self.ctx(), C.byref(b), _vp(out["path_packed"]).value)
        self._check(st, 0)
        return out

    # -- chains ------------------------------------------------------------
    def assign_1d(self, n, S, T):
        S = np.ascontiguousarray(S, np.int32)
        T = np.ascontiguousarray(T, np.int32)
        w = C.c_int64(0)
        ps = np.zeros(max(1, len(T)), np.int64)
        pt = np.zeros(max(1, len(T)), np.int64)
        use = np.zeros(max(1, len(S)), np.int32)
        det = C.c_int32(0)
        st = self.lib.recon_assign_1d(self.ctx(), n, _ptr(S, I32P), len(S), _ptr(T, I32P), len(T),
                                      C.byref(w), _ptr(ps, I64P), _ptr(pt, I64P), _ptr(use, I32P),
                                      C.byref(det))
        self._check(st, det)
        return int(w.value), np.stack([ps[: len(T)], pt[: len(T)]], axis=1), use[: len(S)].copy()

    def assign_1d_generalized(self, pos, mult, min_use, targets):
        pos = np.ascontiguousarray(pos, np.int64)
        mult = np.ascontiguousarray(mult, np.int32)
        mu = np.ascontiguousarray(min_use, np.int32)
        tg = np.ascontiguousarray(targets, np.int64)
        w = C.c_int64(0)
        ps = np.zeros(max(1, len(tg)), np.int64)
        pt = np.zeros(max(1, len(tg)), np.int64)
        use = np.zeros(max(1, len(pos)), np.int32)
        det = C.c_int32(0)
        st = self.lib.recon_assign_1d_generalized(self.ctx(), len(pos), _ptr(pos, I64P), _ptr(mult, I32P),
                                                  _ptr(mu, I32P), len(tg), _ptr(tg, I64P), C.byref(w),
                                                  _ptr(ps, I64P), _ptr(pt, I64P), _ptr(use, I32P),
                                                  C.byref(det))
        self._check(st, det)
        return int(w.value), np.stack([ps[: len(tg)], pt[: len(tg)]], axis=1), use[: len(pos)].copy()

    def solve_1d(self, n, S, T, with_dag: bool = True) -> ChainResult:
        S = np.ascontiguousarray(S, np.int32)
        T = np.ascontiguousarray(T, np.int32)
        nt = len(T)
        src = np.zeros(max(1, nt), np.int32)
        dst = np.zeros(max(1, nt), np.int32)
        order = np.zeros(max(1, nt), np.int32)
        cap = max(16, nt * 4)
        while True:
            a = np.zeros(cap, np.int32) if with_dag else None
            b = np.zeros(cap, np.int32) if with_dag else None
            cnt = C.c_int64(0)
            tot = C.c_int64(0)
            disp = C.c_int32(0)
            det = C.c_int32(0)
            st = self.lib.recon_solve_1d(self.ctx(), n, _ptr(S, I32P), len(S), _ptr(T, I32P), nt,
                                         _ptr(src, I32P), _ptr(dst, I32P), _ptr(order, I32P),
                                         _ptr(a, I32P), _ptr(b, I32P), cap, C.byref(cnt), C.byref(tot),
                                         C.byref(disp), C.byref(det))
            if with_dag and st == RECON_ERR_CAPACITY and cnt.value > cap:
                cap = int(cnt.value)
                continue
            break
        self._check(st, det)
        dag = np.stack([a[: cnt.value], b[: cnt.value]], axis=1) if with_dag else None
        return ChainResult(src[:nt].copy(), dst[:nt].copy(), order[:nt].copy(), dag, int(tot.value),
                           int(disp.value))

    def solve_1d_batch(self, occ, count, n, t_lo, t_hi, host: bool = True):
        nt = t_hi - t_lo + 1
        out = {
            "path_src": np.zeros(count * nt, np.int32),
            "path_dst": np.zeros(count * nt, np.int32),
            "total_displacement": np.zeros(count, np.int64),
            "displaced": np.zeros(count, np.int32),
            "status": np.zeros(count, np.int32),
            "detail": np.zeros(count, np.int32),
        }
        occ = np.ascontiguousarray(occ, np.uint64)
        b = ChainBatch(_vp(occ).value, count, n, t_lo, t_hi, _vp(out["path_src"]).value,
                       _vp(out["path_dst"]).value, _vp(out["total_displacement"]).value,
                       _vp(out["displaced"]).value, _vp(out["status"]).value, _vp(out["detail"]).value)
        fn = self.lib.recon_solve_1d_batch_host if host else self.lib.recon_solve_1d_batch
        st = fn(self.ctx(), C.byref(b))
        self._check(st, 0)
        return out

    # -- batching ------------------------------------------------------------
    def batch_moves(self, width, height, occ, path_vertices: list, edges, preset=0, edge_level=False):
        """path_vertices: list of int sequences.  Returns (move_batch, nb)."""
        occ = np.ascontiguousarray(occ, np.uint64)
        P = len(path_vertices)
        off = np.zeros(P + 1, np.int64)
        for i, p in enumerate(path_vertices):
            off[i + 1] = off[i] + len(p)
        verts = np.zeros(max(1, int(off[-1])), np.int32)
        for i, p in enumerate(path_vertices):
            verts[off[i]: off[i + 1]] = p
        edges = np.asarray(edges, np.int32).reshape(-1, 2)
        es = np.ascontiguousarray(edges[:, 0])
        ed = np.ascontiguousarray(edges[:, 1])
        moves = int(off[-1]) - P
        mb = np.full(max(1, moves), -1, np.int32)
        nb = C.c_int64(0)
        det = C.c_int32(0)
        st = self.lib.recon_batch_moves(self.ctx(), width, height, _ptr(occ, U64P), P, _ptr(off, I64P),
                                        _ptr(verts, I32P), len(es), _ptr(es, I32P), _ptr(ed, I32P),
                                        preset, int(edge_level), _ptr(mb, I32P), C.byref(nb),
                                        C.byref(det))
        self._check(st, det)
        return mb[:moves].copy(), int(nb.value)

    def validate(self, occ, count, width, height, h_prime, path_src, path_dst, path_stride, path_count,
                 total_displacement=None, displaced=None, dag_mode=DAG_NONE, dag_a=None, dag_b=None,
                 dag_offset=None, move_batch=None, move_stride=0, batch_count=None, preset=0):
        """recon_validate_batch_run_host: one recon_verdict bit set per instance."""
        arrs = {
            "occ": np.ascontiguousarray(occ, np.uint64),
            "src": np.ascontiguousarray(path_src, np.int32), "dst": np.ascontiguousarray(path_dst, np.int32),
            "pc": np.ascontiguousarray(path_count, np.int32),
            "td": None if total_displacement is None else np.ascontiguousarray(total_displacement, np.int64),
            "dp": None if displaced is None else np.ascontiguousarray(displaced, np.int32),
            "ea": None if dag_a is None else np.ascontiguousarray(dag_a, np.int32),
            "eb": None if dag_b is None else np.ascontiguousarray(dag_b, np.int32),
            "eo": None if dag_offset is None else np.ascontiguousarray(dag_offset, np.int64),
            "mb": None if move_batch is None else np.ascontiguousarray(move_batch, np.int32),
            "nb": None if batch_count is None else np.ascontiguousarray(batch_count, np.int32),
        }
        verdict = np.zeros(count, np.uint32)
        vb = ValidateBatch(_vp(arrs["occ"]).value, count, width, height, h_prime, _vp(arrs["src"]).value,
                           _vp(arrs["dst"]).value, path_stride, _vp(arrs["pc"]).value, _vp(arrs["td"]).value,
                           _vp(arrs["dp"]).value, dag_mode, _vp(arrs["ea"]).value, _vp(arrs["eb"]).value,
                           _vp(arrs["eo"]).value, _vp(arrs["mb"]).value, move_stride, _vp(arrs["nb"]).value,
                           preset, _vp(verdict).value)
        st = self.lib.recon_validate_batch_run_host(self.ctx(), C.byref(vb))
        self._check(st, 0)
        return verdict

    def _json(self, call) -> bytes:
        n = C.c_int64(0)
        st = call(None, 0, C.byref(n))
        if st == RECON_ERR_CAPACITY or (st == RECON_OK and n.value > 0):
            buf = C.create_string_buffer(max(1, n.value))
            st = call(buf, n.value, C.byref(n))
            self._check(st, 0)
            return buf.raw[:n.value]
        self._check(st, 0)
        return b""

    def solution_json(self, width, height, src, dst, order=None, dag=None, displaced=0, total=0) -> bytes:
        """recon_solution_json_host: the reference's solution_to_json text."""
        src = np.ascontiguousarray(src, np.int32)
        dst = np.ascontiguousarray(dst, np.int32)
        order = None if order is None else np.ascontiguousarray(order, np.int32)
        dag = np.zeros((0, 2), np.int32) if dag is None else np.ascontiguousarray(dag, np.int32).reshape(-1, 2)
        ea, eb = np.ascontiguousarray(dag[:, 0]), np.ascontiguousarray(dag[:, 1])
        return self._json(lambda out, cap, n: self.lib.recon_solution_json_host(
            self.ctx(), width, height, len(src), _vp(src), _vp(dst), _vp(order), len(ea), _vp(ea), _vp(eb),
            displaced, total, out, cap, n))

    def batch_schedule_json(self, width, height, src, dst, move_batch, batch_count, preset=0) -> bytes:
        """recon_batch_schedule_json_host: the reference's batch_schedule_to_json text."""
        src = np.ascontiguousarray(src, np.int32)
        dst = np.ascontiguousarray(dst, np.int32)
        mb = np.ascontiguousarray(move_batch, np.int32)
        return self._json(lambda out, cap, n: self.lib.recon_batch_schedule_json_host(
            self.ctx(), width, height, len(src), _vp(src), _vp(dst), _vp(mb), batch_count, preset, out, cap, n))

    def sim_run(self, occ, count, width, height, h_prime, seed_base, solver="redrec", batching=False, preset=0,
                max_cycles=20, p_nu=0.985, p_alpha=0.985, tau=0.0, t_nu=100e-6, t_alpha=300e-6, t_meas=20e-3):
        """recon_sim_run_host: one outcome record per trial (SPEC.md sim.run_trial)."""
        occ = np.ascontiguousarray(occ, np.uint64)
        out = {k: np.zeros(count, np.int32) for k in ("success", "cycles", "status")}
        out.update({k: np.zeros(count, np.int64) for k in ("n_nu", "n_alpha", "nb_nu", "nb_alpha", "atoms_lost")})
        out["elapsed"] = np.zeros(count, np.float64)
        sb = SimBatch(_vp(occ).value, count, width, height, h_prime, seed_base, 1 if solver == "bird" else 0,
                      1 if batching else 0, preset, max_cycles, LossModel(p_nu, p_alpha, tau, t_nu, t_alpha, t_meas),
                      *[_vp(out[k]).value for k in ("success", "cycles", "status", "n_nu", "n_alpha", "nb_nu",
                                                     "nb_alpha", "atoms_lost", "elapsed")])
        st = self.lib.recon_sim_run_host(self.ctx(), C.byref(sb))
        self._check(st, 0)
        return out

    def pipeline_stats_host(self, out: dict, count, width, h_prime, move_stride) -> np.ndarray:
        """recon_pipeline_stats over a pipeline_batch result held in host memory
        (the CPU checkers: oracle / compiled reference)."""
        g = GridBatch(None, count, width, 0, h_prime, _vp(out["path_src"]).value, _vp(out["path_dst"]).value, None,
                      _vp(out["path_count"]).value, _vp(out["total_displacement"]).value,
                      _vp(out["status"]).value, _vp(out["detail"]).value, None)
        pb = PipelineBatch(g, 0, 0, move_stride, _vp(out["move_batch"]).value, _vp(out["batch_count"]).value)
        st = np.zeros(count, STATS_DTYPE)
        r = self.lib.recon_pipeline_stats(None, C.byref(pb), st.ctypes.data)
        self._check(r, 0)
        return st

    def pipeline_batch_runs(self, solver: str, occ, count, width, height, h_prime, preset, move_stride,
                            run_stride=None, pinned=False):
        """recon_pipeline_batch_run_host_runs: the pipeline_batch outputs with the
        schedule as runs (run_slot, run_batch, run_count) instead of move_batch.
        pinned: the run arrays in page-locked memory (torch), which the library
        writes from the device instead of copying."""
        stride = width * h_prime
        run_stride = run_stride or stride + 4096
        if pinned:
            import torch
            keep = torch.zeros(2 * count * run_stride, dtype=torch.int32).pin_memory()
            both = keep.numpy()
            run_slot, run_batch = both[:count * run_stride], both[count * run_stride:]
        else:
            keep = None
            run_slot, run_batch = np.zeros(count * run_stride, np.int32), np.zeros(count * run_stride, np.int32)
        out = {
            "path_src": np.zeros(count * stride, np.int32), "path_dst": np.zeros(count * stride, np.int32),
            "path_count": np.zeros(count, np.int32), "total_displacement": np.zeros(count, np.int64),
            "status": np.zeros(count, np.int32), "detail": np.zeros(count, np.int32),
            "batch_count": np.zeros(count, np.int32), "run_slot": run_slot,
            "run_batch": run_batch, "run_count": np.zeros(count, np.int64),
        }
        occ = np.ascontiguousarray(occ, np.uint64)
        g = GridBatch(_vp(occ).value, count, width, height, h_prime, _vp(out["path_src"]).value,
                      _vp(out["path_dst"]).value, None, _vp(out["path_count"]).value,
                      _vp(out["total_displacement"]).value, _vp(out["status"]).value, _vp(out["detail"]).value, None)
        pb = PipelineBatch(g, 1 if solver == "bird" else 0, preset, move_stride, None, _vp(out["batch_count"]).value)
        runs = ScheduleRuns(run_stride, _vp(out["run_slot"]).value, _vp(out["run_batch"]).value,
                            _vp(out["run_count"]).value)
        st = self.lib.recon_pipeline_batch_run_host_runs(self.ctx(), C.byref(pb), C.byref(runs))
        self._check(st, 0)
        out["run_stride"] = run_stride
        out["_pinned"] = keep
        return out

    def pipeline_batch(self, solver: str, occ, count, width, height, h_prime, preset, move_stride):
        stride = width * h_prime
        out = {
            "path_src": np.zeros(count * stride, np.int32),
            "path_dst": np.zeros(count * stride, np.int32),
            "path_event": np.zeros(count * stride, np.int32),
            "path_count": np.zeros(count, np.int32),
            "total_displacement": np.zeros(count, np.int64),
            "status": np.zeros(count, np.int32),
            "detail": np.zeros(count, np.int32),
            "move_batch": np.full(count * move_stride, -1, np.int32),
            "batch_count": np.zeros(count, np.int32),
        }
        occ = np.ascontiguousarray(occ, np.uint64)
        g = GridBatch(_vp(occ).value, count, width, height, h_prime, _vp(out["path_src"]).value,
                      _vp(out["path_dst"]).value, _vp(out["path_event"]).value,
                      _vp(out["path_count"]).value, _vp(out["total_displacement"]).value,
                      _vp(out["status"]).value, _vp(out["detail"]).value, None)
        pb = PipelineBatch(g, 1 if solver == "bird" else 0, preset, move_stride,
                           _vp(out["move_batch"]).value, _vp(out["batch_count"]).value)
        st = self.lib.recon_pipeline_batch_run_host(self.ctx(), C.byref(pb))
        self._check(st, 0)
        return out
