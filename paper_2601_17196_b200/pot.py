"""Python mirror of the reference's ``namespace pot`` solver API over the
C-ABI in include/potgpu.h (libpotgpu.so, sm_100a).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/pot/{core,solvers}.hpp:

* ``Instance`` (core.hpp:108-118), ``SolverConfig`` (core.hpp:241-267),
  ``SolveResult`` (solvers.hpp:176-186), ``TraceRecord`` (core.hpp:269-275),
  ``TheoryBounds`` (solvers.hpp:139-144);
* ``solve`` (solvers.hpp:591), ``aspot_solve`` (:265),
  ``feasible_sinkhorn_solve`` (:516), ``tuned_sinkhorn_solve`` (:547/:586);
* failures raise ``PotError`` carrying the reference's ``ErrorCode``.

There is no CPU fallback: importing works anywhere (the library is
self-contained), but every solve runs on a CUDA device and raises if none is
present or the library is missing.
"""
from __future__ import annotations

import ctypes
import enum
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpotgpu.so")


class ErrorCode(enum.IntEnum):  # core.hpp:21-39 (order preserved)
    DimensionMismatch = 0
    NegativeEntry = 1
    NonFiniteEntry = 2
    BudgetExceedsMass = 3
    Overflow = 4
    NonPositiveArgument = 5
    DegenerateInstance = 6
    PenaltyTooSmall = 7
    UnbalancedMarginals = 8
    ZeroEntropy = 9
    Infeasible = 10
    SizeLimitExceeded = 11
    ZeroMassPlan = 12
    DegenerateSvd = 13
    EmptyInput = 14
    InvalidArgument = 15
    IoFailure = 16
    # appended by the device boundary (no reference counterpart)
    CudaError = 17
    NcclError = 18
    Unsupported = 19


class PotError(RuntimeError):
    """core.hpp:64-74."""

    def __init__(self, code: ErrorCode, message: str):
        super().__init__(f"{code.name}: {message}")
        self.code = code


class SolverKind(enum.IntEnum):  # core.hpp:223
    Aspot = 0
    FeasibleSinkhorn = 1
    TunedSinkhorn = 2


class BlockRule(enum.IntEnum):  # core.hpp:221
    Greedy = 0
    RoundRobin = 1


class SolveStatus(enum.IntEnum):  # core.hpp:284
    Converged = 0
    MaxIterationsExceeded = 1
    StepSizeUnderflow = 2


class DType(enum.IntEnum):
    F64 = 0
    F32 = 1


# --------------------------------------------------------------- C structs --
class _Problem(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("dtype", ctypes.c_int), ("cost_kind", ctypes.c_int),
        ("C", ctypes.POINTER(ctypes.c_double)), ("ldc", ctypes.c_int64), ("row_major", ctypes.c_int),
        ("X", ctypes.POINTER(ctypes.c_double)), ("Y", ctypes.POINTER(ctypes.c_double)), ("d", ctypes.c_int),
        ("cost_scale", ctypes.c_double),
        ("r", ctypes.POINTER(ctypes.c_double)), ("c", ctypes.POINTER(ctypes.c_double)), ("s", ctypes.c_double),
        ("device_ptrs", ctypes.c_int), ("producer_stream", ctypes.c_int64),
    ]


class _Config(ctypes.Structure):
    _fields_ = [
        ("epsilon", ctypes.c_double), ("gamma_override", ctypes.c_double), ("max_iterations", ctypes.c_int64),
        ("block_rule", ctypes.c_int), ("tuning_exponent_p", ctypes.c_double), ("deterministic", ctypes.c_int),
        ("log_every", ctypes.c_int64), ("record_rounded_cost", ctypes.c_int), ("materialize_plan", ctypes.c_int),
        ("collect_iter_log", ctypes.c_int), ("use_graphs", ctypes.c_int), ("sync_every", ctypes.c_int),
    ]


class _Trace(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("error", ctypes.c_double), ("phi", ctypes.c_double),
                ("rounded_cost", ctypes.c_double), ("elapsed_s", ctypes.c_double)]


class _IterLog(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("halvings", ctypes.c_int32), ("block_hat", ctypes.c_int32),
                ("zbest_is_check", ctypes.c_int32), ("block_check", ctypes.c_int32), ("error", ctypes.c_double),
                ("phi_check", ctypes.c_double), ("phi_hat", ctypes.c_double), ("theta", ctypes.c_double)]


class _Summary(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int), ("iterations", ctypes.c_int64), ("gamma", ctypes.c_double),
        ("tolerance", ctypes.c_double), ("final_error", ctypes.c_double), ("wall_seconds", ctypes.c_double),
        ("loop_seconds", ctypes.c_double), ("has_bounds", ctypes.c_int), ("bound_R", ctypes.c_double),
        ("bound_L", ctypes.c_double), ("bound_mu_f", ctypes.c_double), ("iteration_bound", ctypes.c_double),
        ("cost", ctypes.c_double), ("feasibility_gap", ctypes.c_double), ("mass", ctypes.c_double),
        ("phi", ctypes.c_double), ("trace_len", ctypes.c_int64), ("iter_log_len", ctypes.c_int64),
        ("sweeps", ctypes.c_int64), ("attempts", ctypes.c_int64), ("stopping_iterate", ctypes.c_char * 24),
    ]


class _RegConfig(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("gamma0", ctypes.c_double), ("anneal_rate", ctypes.c_double),
                ("transform_threshold", ctypes.c_double), ("max_registrations", ctypes.c_int)]


class _RegRecord(ctypes.Structure):
    _fields_ = [("round", ctypes.c_int32), ("inner_iterations", ctypes.c_int64),
                ("accumulated_iterations", ctypes.c_int64), ("cost", ctypes.c_double), ("increment", ctypes.c_double),
                ("gamma", ctypes.c_double)]


class _RegResult(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3), ("converged", ctypes.c_int),
                ("rounds", ctypes.c_int64)]


class _Outputs(ctypes.Structure):
    _fields_ = [
        ("X", ctypes.POINTER(ctypes.c_double)), ("row_slack", ctypes.POINTER(ctypes.c_double)),
        ("col_slack", ctypes.POINTER(ctypes.c_double)), ("trace", ctypes.POINTER(_Trace)), ("trace_cap", ctypes.c_int64),
        ("iter_log", ctypes.POINTER(_IterLog)), ("iter_log_cap", ctypes.c_int64),
        ("u", ctypes.POINTER(ctypes.c_double)), ("v", ctypes.POINTER(ctypes.c_double)),
        ("w", ctypes.POINTER(ctypes.c_double)),
    ]


# potgpu_host_allreduce_fn: void (double* buf, int64_t count, int op, void* user)
HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(None, ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_void_p)
REDUCE_SUM, REDUCE_MAX = 0, 2

# Every symbol include/potgpu.h declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = (
    "potgpu_abi_version", "potgpu_last_error", "potgpu_config_default", "potgpu_create", "potgpu_destroy",
    "potgpu_solve", "potgpu_dual_eval", "potgpu_round_pot", "potgpu_comm_unique_id", "potgpu_comm_init",
    "potgpu_make_synthetic", "potgpu_make_config", "potgpu_session_begin", "potgpu_session_iterate",
    "potgpu_session_finish", "potgpu_session_destroy", "potgpu_ctx_stream", "potgpu_session_time_sweep", "potgpu_session_time_one_sided",
    "potgpu_session_stats", "potgpu_solve_batched", "potgpu_comm_init_local", "potgpu_comm_info",
    "potgpu_release_cached_memory", "potgpu_reg_config_default", "potgpu_register_point_clouds", "potgpu_fit_rigid",
    "potgpu_kmeans_quantize", "potgpu_round_balanced", "potgpu_dual_matrix", "potgpu_session_read_state",
    "potgpu_session_carry_stats", "potgpu_comm_init_host",
)

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpotgpu.so; raises (no fallback) when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise PotError(ErrorCode.CudaError, f"{path} is missing: run __graft_entry__.build() (make -C paper_2601_17196_b200)")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    dp = P(ctypes.c_double)
    lib.potgpu_last_error.restype = ctypes.c_char_p
    lib.potgpu_create.argtypes = [ctypes.c_int, P(ctypes.c_void_p)]
    lib.potgpu_destroy.argtypes = [ctypes.c_void_p]
    lib.potgpu_config_default.argtypes = [P(_Config)]
    lib.potgpu_solve.argtypes = [ctypes.c_void_p, ctypes.c_int, P(_Problem), P(_Config), P(_Summary), P(_Outputs)]
    lib.potgpu_dual_eval.argtypes = [ctypes.c_void_p, P(_Problem), ctypes.c_double, dp, dp, ctypes.c_double, dp, dp, dp]
    lib.potgpu_session_begin.argtypes = [ctypes.c_void_p, ctypes.c_int, P(_Problem), P(_Config), ctypes.c_int64,
                                         ctypes.c_int64, P(ctypes.c_void_p)]
    lib.potgpu_session_iterate.argtypes = [ctypes.c_void_p, ctypes.c_int64, dp, P(ctypes.c_int64), P(ctypes.c_int)]
    lib.potgpu_session_finish.argtypes = [ctypes.c_void_p, P(_Summary), P(_Outputs)]
    lib.potgpu_session_destroy.argtypes = [ctypes.c_void_p]
    lib.potgpu_ctx_stream.argtypes = [ctypes.c_void_p]
    lib.potgpu_ctx_stream.restype = ctypes.c_void_p
    lib.potgpu_session_time_sweep.argtypes = [ctypes.c_void_p, ctypes.c_int, dp, dp, dp]
    lib.potgpu_session_time_one_sided.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, dp]
    lib.potgpu_solve_batched.argtypes = [ctypes.c_void_p, ctypes.c_int, P(_Problem), ctypes.c_int64, P(_Config),
                                         P(_Summary), P(_Outputs), ctypes.c_int]
    lib.potgpu_session_stats.argtypes = [ctypes.c_void_p, P(ctypes.c_int64), P(ctypes.c_int64), P(ctypes.c_int64)]
    lib.potgpu_session_carry_stats.argtypes = [ctypes.c_void_p, P(ctypes.c_int64), P(ctypes.c_int64)]
    lib.potgpu_reg_config_default.argtypes = [P(_RegConfig)]
    lib.potgpu_register_point_clouds.argtypes = [ctypes.c_void_p, ctypes.c_int, dp, ctypes.c_int64, dp, ctypes.c_int64,
                                                 P(_RegConfig), P(_Config), ctypes.c_int, P(_RegResult), P(_RegRecord),
                                                 ctypes.c_int64]
    lib.potgpu_fit_rigid.argtypes = [ctypes.c_void_p, dp, ctypes.c_int64, ctypes.c_int64, dp, dp, dp, dp]
    lib.potgpu_kmeans_quantize.argtypes = [ctypes.c_void_p, dp, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, dp, dp,
                                           P(ctypes.c_int32)]
    lib.potgpu_round_pot.argtypes = [ctypes.c_void_p, ctypes.c_int64, dp, dp, dp, ctypes.c_double, dp]
    lib.potgpu_round_balanced.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, dp, dp, dp, dp]
    lib.potgpu_dual_matrix.argtypes = [ctypes.c_void_p, P(_Problem), ctypes.c_double, dp, dp, ctypes.c_double,
                                       ctypes.c_int, dp]
    lib.potgpu_session_read_state.argtypes = [ctypes.c_void_p, ctypes.c_int, dp, dp, dp, dp]
    lib.potgpu_comm_unique_id.argtypes = [ctypes.c_char_p]
    lib.potgpu_comm_init.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
    lib.potgpu_comm_init_local.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.potgpu_comm_init_host.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, HOST_ALLREDUCE_FN,
                                          ctypes.c_void_p]
    lib.potgpu_comm_info.argtypes = [ctypes.c_void_p, P(ctypes.c_int), P(ctypes.c_int), P(ctypes.c_int)]
    lib.potgpu_make_synthetic.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, dp, dp, dp, dp]
    lib.potgpu_make_config.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, dp, dp, dp, dp,
                                       P(ctypes.c_int), dp, dp]
    _lib = lib
    return lib


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check(rc: int):
    if rc != 0:
        msg = load_library().potgpu_last_error().decode(errors="replace")
        raise PotError(ErrorCode(rc - 1), msg)


# ------------------------------------------------------------ public types --
@dataclass
class Instance:
    """core.hpp:108-118. Either a dense cost C (n x n) or, for the on-the-fly
    squared-Euclidean kernel, point coordinates X, Y (n x d) with
    C_ij = cost_scale |x_i - y_j|^2 (cost_scale None -> 1 / max)."""
    r: np.ndarray
    c: np.ndarray
    s: float
    C: Optional[np.ndarray] = None
    X: Optional[np.ndarray] = None
    Y: Optional[np.ndarray] = None
    cost_scale: Optional[float] = None
    dtype: DType = DType.F64
    stored: bool = False  # points given, cost materialised once on the device and streamed

    def size(self) -> int:
        return int(self.r.shape[0]) if hasattr(self.r, "shape") else len(self.r)

    def source_mass(self) -> float:
        return float(np.sum(self.r))

    def target_mass(self) -> float:
        return float(np.sum(self.c))


@dataclass
class SolverConfig:  # core.hpp:241-267
    epsilon: float = 0.1
    gamma_override: Optional[float] = None
    max_iterations: int = 50000
    block_rule: BlockRule = BlockRule.Greedy
    tuning_exponent_p: float = 1.0
    deterministic: bool = True
    log_every: int = 1
    # device options (no reference counterpart)
    record_rounded_cost: bool = True
    materialize_plan: bool = True
    collect_iter_log: bool = False
    use_graphs: bool = True
    sync_every: int = 8


@dataclass
class TraceRecord:  # core.hpp:269-275
    t: int
    error: float
    phi: float
    rounded_cost: Optional[float]
    elapsed_s: float


@dataclass
class TheoryBounds:  # solvers.hpp:139-144
    R: float
    L: float
    mu_f: float
    iteration_bound: float


@dataclass
class TransportPlan:  # core.hpp:179-197 (X is None unless materialised)
    X: Optional[np.ndarray]
    row_slack: np.ndarray
    col_slack: np.ndarray
    mass: float


@dataclass
class SolveResult:  # solvers.hpp:176-186 (+ plan metrics computed on the device)
    plan: TransportPlan
    trace: List[TraceRecord]
    stopping_iterate: str
    status: SolveStatus
    iterations: int
    gamma: float
    tolerance: float
    final_error: float
    wall_seconds: float
    bounds: Optional[TheoryBounds]
    cost: float
    feasibility_gap: float
    phi: float
    loop_seconds: float = 0.0
    sweeps: int = 0
    attempts: int = 0
    iter_log: Optional[np.ndarray] = None
    u: Optional[np.ndarray] = None
    v: Optional[np.ndarray] = None
    w: Optional[float] = None


ITER_LOG_FIELDS = ("t", "halvings", "block_hat", "zbest_is_check", "block_check", "error", "phi_check", "phi_hat",
                   "theta")


class Context:
    """Owns a device, a stream and the workspaces (potgpu_create)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.potgpu_create(int(device), ctypes.byref(h)))
        self._h = h
        self.device = device

    def shard_local(self, shards: int) -> "Context":
        """Run the row-sharded arithmetic with `shards` shards in this
        process (potgpu_comm_init_local): the multi-GPU data path on one GPU."""
        _check(load_library().potgpu_comm_init_local(self._h, int(shards)))
        return self

    def init_comm(self, rank: int, world_size: int, unique_id: bytes) -> "Context":
        """Join a row-sharded multi-GPU job (potgpu_comm_init, NCCL)."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        _check(load_library().potgpu_comm_init(self._h, int(rank), int(world_size), bytes(unique_id)))
        return self

    def init_host_comm(self, rank: int, world_size: int, allreduce) -> "Context":
        """Join a row-sharded job whose cross-process reduction is the Python
        callable `allreduce(array, op)` (potgpu_comm_init_host): `array` is a
        float64 numpy view of the host buffer to reduce in place, `op` is
        REDUCE_SUM or REDUCE_MAX. Runs on a CUDA host-callback thread."""
        def trampoline(buf, count, op, user):
            try:
                allreduce(np.ctypeslib.as_array(buf, shape=(int(count),)), int(op))
            except BaseException as e:  # an exception cannot cross the C boundary
                import traceback
                traceback.print_exc()
                print(f"host all-reduce failed: {e}", flush=True)
                os._exit(70)
        self._host_fn = HOST_ALLREDUCE_FN(trampoline)  # kept alive with the context
        _check(load_library().potgpu_comm_init_host(self._h, int(rank), int(world_size), self._host_fn, None))
        return self

    def comm_info(self) -> Tuple[int, int, int]:
        """(rank, world_size, shards_per_rank)."""
        r, w, v = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(load_library().potgpu_comm_info(self._h, ctypes.byref(r), ctypes.byref(w), ctypes.byref(v)))
        return r.value, w.value, v.value

    def close(self):
        if self._h:
            load_library().potgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def release_cached_memory() -> None:
    """potgpu_release_cached_memory: return cached device / pinned blocks."""
    load_library().potgpu_release_cached_memory()


def nccl_unique_id() -> bytes:
    """potgpu_comm_unique_id: the 128-byte NCCL id rank 0 broadcasts."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().potgpu_comm_unique_id(buf))
    return buf.raw


def shard_rows(n: int, world: int, shards_per_rank: int = 1) -> List[Tuple[int, int]]:
    """Row range [lo, hi) of every shard of a sharded job, in shard order
    (rank r owns shards r*shards_per_rank ...); the split of shard.cuh Comm."""
    total = world * shards_per_rank
    return [((n * s) // total, (n * (s + 1)) // total) for s in range(total)]


def init_distributed(ctx: Context, group=None) -> Context:
    """Join the torch.distributed job this process belongs to as one rank of
    a row-sharded solve: rank 0 creates the NCCL id, torch.distributed
    broadcasts it (any backend), every rank initialises its communicator."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return ctx.init_comm(rank, world, box[0])


def init_distributed_host(ctx: Context, group=None) -> Context:
    """Join the torch.distributed job this process belongs to through the
    host collective backend: every sweep's all-reduce vector goes through
    torch.distributed.all_reduce on a CPU tensor (e.g. the gloo backend).
    Works with several ranks on one GPU; for correctness tests and
    portability (NCCL: init_distributed)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ops = {REDUCE_SUM: dist.ReduceOp.SUM, REDUCE_MAX: dist.ReduceOp.MAX}

    def allreduce(arr, op):
        t = torch.from_numpy(arr)  # shares the pinned buffer
        dist.all_reduce(t, op=ops[op], group=group)

    return ctx.init_host_comm(rank, world, allreduce)


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("POTGPU_USE_LOCAL_RANK") else 0)
    return _default_ctx


def _cuda_ptr(a, shape, what: str):
    """Device pointer of a float64 C-contiguous CUDA array (__cuda_array_interface__)."""
    cai = a.__cuda_array_interface__
    if cai.get("typestr") not in ("<f8", "=f8"):
        raise PotError(ErrorCode.InvalidArgument, f"{what}: device arrays must be float64")
    if tuple(cai["shape"]) != tuple(shape):
        raise PotError(ErrorCode.DimensionMismatch, f"{what} has shape {tuple(cai['shape'])}, expected {tuple(shape)}")
    strides = cai.get("strides")
    if strides is not None and tuple(strides) != tuple(8 * int(np.prod(shape[k + 1:])) for k in range(len(shape))):
        raise PotError(ErrorCode.InvalidArgument, f"{what}: device arrays must be C-contiguous")
    return ctypes.cast(ctypes.c_void_p(cai["data"][0]), ctypes.POINTER(ctypes.c_double))


def _producer_stream(arrays) -> int:
    """potgpu_problem.producer_stream from the arrays' __cuda_array_interface__
    v3 "stream" keys: the one stream they name (the solver orders its reads
    after work queued on it), -1 when every array says "no sync needed"
    (None), 0 (synchronise the device) when absent or when they disagree."""
    seen = set()
    for a in arrays:
        if type(a).__module__.startswith("torch"):
            # torch exports CAI v2 (no "stream"); its producer is the current
            # stream of the tensor's device (handle 0 = the legacy default)
            import torch
            h = int(torch.cuda.current_stream(a.device).cuda_stream)
            seen.add(h if h else 1)
            continue
        cai = a.__cuda_array_interface__
        if "stream" not in cai:
            return 0
        seen.add(-1 if cai["stream"] is None else int(cai["stream"]))
    if len(seen) == 1:
        return seen.pop()
    return 0


def _is_cuda(a) -> bool:
    return a is not None and hasattr(a, "__cuda_array_interface__")


def _problem_device(inst: Instance, keep: list) -> _Problem:
    """Every array on the device (device_ptrs = 1): no host copies of C."""
    n = int(inst.r.shape[0])
    p = _Problem()
    p.n, p.dtype, p.device_ptrs, p.s = n, int(inst.dtype), 1, float(inst.s)
    p.r, p.c = _cuda_ptr(inst.r, (n,), "r"), _cuda_ptr(inst.c, (n,), "c")
    keep += [inst.r, inst.c]
    if inst.C is not None:
        p.cost_kind, p.C, p.ldc, p.row_major = 0, _cuda_ptr(inst.C, (n, n), "C"), n, 1
        keep.append(inst.C)
    else:
        d = int(inst.X.shape[1])
        p.cost_kind, p.X, p.Y, p.d = (2 if inst.stored else 1), _cuda_ptr(inst.X, (n, d), "X"), \
            _cuda_ptr(inst.Y, (n, d), "Y"), d
        p.cost_scale = float(inst.cost_scale) if inst.cost_scale else 0.0
        keep += [inst.X, inst.Y]
    p.producer_stream = _producer_stream([a for a in (inst.r, inst.c, inst.C, inst.X, inst.Y) if a is not None])
    return p


def _dense_layout(C, n: int):
    """(array, ldc, row_major) of a float64 n x n cost without a copy when its
    layout is one the C-ABI reads directly: C order, Fortran order (Eigen's
    column-major MatrixXd), or a row / column view with a padded leading
    dimension (e.g. C[:n, :n] of a wider array); anything else is copied."""
    C = np.asarray(C)
    if C.shape != (n, n):
        raise PotError(ErrorCode.DimensionMismatch, f"cost matrix is {C.shape}, expected {(n, n)}")
    if C.dtype == np.float64 and n > 0:
        s0, s1 = C.strides
        if C.flags.c_contiguous:
            return C, n, 1
        if C.flags.f_contiguous:
            return C, n, 0
        if s1 == 8 and s0 > 0 and s0 % 8 == 0 and s0 // 8 >= n:
            return C, s0 // 8, 1
        if s0 == 8 and s1 > 0 and s1 % 8 == 0 and s1 // 8 >= n:
            return C, s1 // 8, 0
    return np.ascontiguousarray(C, dtype=np.float64), n, 1


def _problem(inst: Instance, keep: list) -> _Problem:
    if _is_cuda(inst.r):
        return _problem_device(inst, keep)
    n = inst.size()
    p = _Problem()
    p.n = n
    p.dtype = int(inst.dtype)
    r = np.ascontiguousarray(inst.r, dtype=np.float64)
    c = np.ascontiguousarray(inst.c, dtype=np.float64)
    keep += [r, c]
    p.r, p.c, p.s = _dp(r), _dp(c), float(inst.s)
    if inst.C is not None:
        C, ldc, row_major = _dense_layout(inst.C, n)
        keep.append(C)
        p.cost_kind, p.C, p.ldc, p.row_major = 0, ctypes.cast(ctypes.c_void_p(C.ctypes.data),
                                                             ctypes.POINTER(ctypes.c_double)), ldc, row_major
    else:
        X = np.ascontiguousarray(inst.X, dtype=np.float64)
        Y = np.ascontiguousarray(inst.Y, dtype=np.float64)
        keep += [X, Y]
        p.cost_kind, p.X, p.Y, p.d = (2 if inst.stored else 1), _dp(X), _dp(Y), int(X.shape[1])
        p.cost_scale = float(inst.cost_scale) if inst.cost_scale else 0.0
    return p


def _config(cfg: SolverConfig) -> _Config:
    c = _Config()
    c.epsilon = cfg.epsilon
    c.gamma_override = cfg.gamma_override if cfg.gamma_override is not None else 0.0
    if cfg.gamma_override is not None and not cfg.gamma_override > 0:
        raise PotError(ErrorCode.InvalidArgument, "gamma override must be positive")
    c.max_iterations = int(cfg.max_iterations)
    c.block_rule = int(cfg.block_rule)
    c.tuning_exponent_p = cfg.tuning_exponent_p
    c.deterministic = int(cfg.deterministic)
    c.log_every = int(cfg.log_every)
    c.record_rounded_cost = int(cfg.record_rounded_cost)
    c.materialize_plan = int(cfg.materialize_plan)
    c.collect_iter_log = int(cfg.collect_iter_log)
    c.use_graphs = int(cfg.use_graphs)
    c.sync_every = int(cfg.sync_every)
    return c


class _OutBufs:
    def __init__(self, kind: SolverKind, n: int, cfg: SolverConfig, trace_cap: int, iter_log_cap: int):
        self.X = np.empty((n, n), dtype=np.float64) if cfg.materialize_plan else None
        self.rs = np.empty(n, dtype=np.float64)
        self.cs = np.empty(n, dtype=np.float64)
        m = n + 1 if kind != SolverKind.Aspot else n
        self.u = np.empty(m, dtype=np.float64)
        self.v = np.empty(m, dtype=np.float64)
        self.w = np.zeros(1, dtype=np.float64)
        self.trace_cap = trace_cap
        self.trace = (_Trace * max(trace_cap, 1))()
        self.cap = iter_log_cap if cfg.collect_iter_log else 0
        self.ilog = (_IterLog * max(self.cap, 1))()
        out = _Outputs()
        out.X, out.row_slack, out.col_slack = _dp(self.X), _dp(self.rs), _dp(self.cs)
        out.trace, out.trace_cap = self.trace, trace_cap
        out.iter_log, out.iter_log_cap = self.ilog, self.cap
        out.u, out.v, out.w = _dp(self.u), _dp(self.v), _dp(self.w)
        self.out = out

    def result(self, sm: _Summary) -> SolveResult:
        tl = min(int(sm.trace_len), self.trace_cap)
        tr = self.trace
        recs = [TraceRecord(int(tr[k].t), tr[k].error, tr[k].phi,
                            None if math.isnan(tr[k].rounded_cost) else tr[k].rounded_cost, tr[k].elapsed_s)
                for k in range(tl)]
        il = None
        if self.cap:
            k = min(int(sm.iter_log_len), self.cap)
            il = np.array([[getattr(self.ilog[i], f) for f in ITER_LOG_FIELDS] for i in range(k)],
                          dtype=np.float64).reshape(k, 9)
        bounds = TheoryBounds(sm.bound_R, sm.bound_L, sm.bound_mu_f, sm.iteration_bound) if sm.has_bounds else None
        return SolveResult(
            plan=TransportPlan(self.X, self.rs, self.cs, sm.mass), trace=recs,
            stopping_iterate=sm.stopping_iterate.decode(), status=SolveStatus(sm.status),
            iterations=int(sm.iterations), gamma=sm.gamma, tolerance=sm.tolerance, final_error=sm.final_error,
            wall_seconds=sm.wall_seconds, bounds=bounds, cost=sm.cost, feasibility_gap=sm.feasibility_gap,
            phi=sm.phi, loop_seconds=sm.loop_seconds, sweeps=int(sm.sweeps), attempts=int(sm.attempts),
            iter_log=il, u=self.u, v=self.v, w=float(self.w[0]))


def _run(kind: SolverKind, inst: Instance, cfg: SolverConfig, ctx: Optional[Context], trace_cap: int = 4096,
         iter_log_cap: int = 0) -> SolveResult:
    lib = load_library()
    ctx = ctx or default_context()
    keep: list = []
    prob = _problem(inst, keep)
    conf = _config(cfg)
    bufs = _OutBufs(kind, inst.size(), cfg, trace_cap, iter_log_cap)
    sm = _Summary()
    _check(lib.potgpu_solve(ctx._h, int(kind), ctypes.byref(prob), ctypes.byref(conf), ctypes.byref(sm),
                            ctypes.byref(bufs.out)))
    return bufs.result(sm)


class Session:
    """potgpu_session_*: begin (setup + first evaluation), iterate(k) with
    device timing, finish (final rounding + outputs)."""

    def __init__(self, kind: SolverKind, inst: Instance, config: SolverConfig = SolverConfig(),
                 ctx: Optional[Context] = None, trace_cap: int = 4096, iter_log_cap: int = 0):
        self.lib = load_library()
        self.ctx = ctx or default_context()
        self.kind = SolverKind(kind)
        self.cfg = config
        self._keep: list = []
        prob = _problem(inst, self._keep)
        conf = _config(config)
        self.bufs = _OutBufs(self.kind, inst.size(), config, trace_cap, iter_log_cap)
        h = ctypes.c_void_p()
        _check(self.lib.potgpu_session_begin(self.ctx._h, int(kind), ctypes.byref(prob), ctypes.byref(conf),
                                             trace_cap, iter_log_cap if config.collect_iter_log else 0,
                                             ctypes.byref(h)))
        self._h = h

    def iterate(self, k: int):
        """Returns (device_ms, iterations_done, finished)."""
        ms = np.zeros(1)
        it = ctypes.c_int64(0)
        fin = ctypes.c_int(0)
        _check(self.lib.potgpu_session_iterate(self._h, int(k), _dp(ms), ctypes.byref(it), ctypes.byref(fin)))
        return float(ms[0]), int(it.value), bool(fin.value)

    def time_sweep(self, reps: int = 10):
        """(ms per sweep launch, elements per launch, HBM bytes per launch)."""
        ms, el, by = np.zeros(1), np.zeros(1), np.zeros(1)
        _check(self.lib.potgpu_session_time_sweep(self._h, int(reps), _dp(ms), _dp(el), _dp(by)))
        return float(ms[0]), float(el[0]), float(by[0])

    def time_one_sided(self, block: int, reps: int = 10) -> float:
        """ms per launch of the one-sided pass (block 0 = u, 1 = v; fused with
        the next z_bar under K1'') at the current z_check. No iterate() after."""
        ms = np.zeros(1)
        _check(self.lib.potgpu_session_time_one_sided(self._h, int(reps), int(block), _dp(ms)))
        return float(ms[0])

    def carry_stats(self):
        """(carried, exact): CTAs of the fp32 points sweep that used a carried
        shift / the exact row maxima so far."""
        a, b = ctypes.c_int64(0), ctypes.c_int64(0)
        _check(self.lib.potgpu_session_carry_stats(self._h, ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    def stats(self):
        """(kernel launches by iterate(), attempts, sweeps) so far."""
        k, a, w = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
        _check(self.lib.potgpu_session_stats(self._h, ctypes.byref(k), ctypes.byref(a), ctypes.byref(w)))
        return int(k.value), int(a.value), int(w.value)

    def finish(self) -> SolveResult:
        sm = _Summary()
        _check(self.lib.potgpu_session_finish(self._h, ctypes.byref(sm), ctypes.byref(self.bufs.out)))
        return self.bufs.result(sm)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.potgpu_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def aspot_solve(inst: Instance, config: SolverConfig = SolverConfig(), ctx: Optional[Context] = None,
                observer=None, **kw) -> SolveResult:
    """solvers.hpp:265-385. observer(AspotIterate) (solvers.hpp:188-204,
    364-367) is called after every accepted iteration: the device loop then
    advances one iteration at a time and the points are copied to the host
    (a diagnostic slow path)."""
    if observer is None or inst.s == 0 or inst.size() < 2:
        return _run(SolverKind.Aspot, inst, config, ctx, **kw)
    st = aspot_setup(inst, config.epsilon)
    gamma = config.gamma_override if config.gamma_override else st.gamma
    ectx = EntropicContext(inst.C if inst.C is not None else dense_cost(inst.X, inst.Y, inst.cost_scale), gamma,
                           st.mixed_r, st.mixed_c, inst.s)
    sess = Session(SolverKind.Aspot, inst, config, ctx=ctx, **kw)
    n = inst.size()
    try:
        while True:
            _, it, fin = sess.iterate(1)
            if it:
                pts, sc = [], np.zeros(6)
                for k in range(4):
                    u, v, w = np.empty(n), np.empty(n), np.zeros(1)
                    _check(sess.lib.potgpu_session_read_state(sess._h, k, _dp(u), _dp(v), _dp(w), _dp(sc)))
                    pts.append(DualPoint(u, v, float(w[0])))
                observer(AspotIterate(int(sc[0]), sc[1], sc[2], ectx, pts[3], pts[2], pts[0], pts[1], sc[3], sc[4],
                                      sc[5]))
            if fin:
                break
        return sess.finish()
    finally:
        sess.close()


def feasible_sinkhorn_solve(inst: Instance, config: SolverConfig = SolverConfig(), ctx: Optional[Context] = None,
                            **kw) -> SolveResult:
    """solvers.hpp:516-542."""
    return _run(SolverKind.FeasibleSinkhorn, inst, config, ctx, **kw)


def tuned_sinkhorn_solve(inst: Instance, epsilon_or_config=None, p: Optional[float] = None,
                         config: Optional[SolverConfig] = None, ctx: Optional[Context] = None, **kw) -> SolveResult:
    """solvers.hpp:547-589: (inst, epsilon, p, config) or (inst, config)."""
    if isinstance(epsilon_or_config, SolverConfig) or epsilon_or_config is None:
        cfg = epsilon_or_config or config or SolverConfig()
    else:
        base = config or SolverConfig()
        cfg = SolverConfig(**{**base.__dict__, "epsilon": float(epsilon_or_config),
                              "tuning_exponent_p": float(p if p is not None else base.tuning_exponent_p)})
    return _run(SolverKind.TunedSinkhorn, inst, cfg, ctx, **kw)


def solve(inst: Instance, kind: SolverKind, config: SolverConfig = SolverConfig(), ctx: Optional[Context] = None,
          **kw) -> SolveResult:
    """solvers.hpp:591-599."""
    return _run(SolverKind(kind), inst, config, ctx, **kw)


def solve_batched(kind: SolverKind, instances: List[Instance], config: SolverConfig = SolverConfig(),
                  ctx: Optional[Context] = None, concurrency: int = 8, trace_cap: int = 16,
                  iter_log_cap: int = 0) -> List[SolveResult]:
    """Independent problems solved concurrently (potgpu_solve_batched;
    BASELINE configs[4]). Each of the `concurrency` workers plans its grids
    for its share of the SMs, so per-problem results agree with `solve` to
    rounding (different reduction grouping) and are deterministic for a given
    concurrency. ASPOT on fp32 stored costs (n <= 4096) runs as ONE
    persistent launch, one problem per thread-block cluster
    (csrc/batch_cluster.cuh; $POTGPU_BATCH_CLUSTER=0 selects the workers)."""
    lib = load_library()
    ctx = ctx or default_context()
    keep: list = []
    k = len(instances)
    probs = (_Problem * max(k, 1))()
    outs = (_Outputs * max(k, 1))()
    sums = (_Summary * max(k, 1))()
    bufs = []
    for i, inst in enumerate(instances):
        probs[i] = _problem(inst, keep)
        b = _OutBufs(SolverKind(kind), inst.size(), config, trace_cap, iter_log_cap)
        bufs.append(b)
        outs[i] = b.out
    conf = _config(config)
    _check(lib.potgpu_solve_batched(ctx._h, int(kind), probs, k, ctypes.byref(conf), sums, outs, int(concurrency)))
    return [bufs[i].result(sums[i]) for i in range(k)]


@dataclass
class DualEval:
    row: np.ndarray     # B 1
    col: np.ndarray     # B^T 1
    total: float
    max_exponent: float
    phi: float
    error: float
    grad_w: float


def dual_eval(inst: Instance, gamma: float, u, v, w: float, ctx: Optional[Context] = None) -> DualEval:
    """b_matrix / dual_objective / dual_gradient / feasibility_error sums at
    z = (u, v, w) for logK = -C/gamma with the instance's marginals as given
    (dual.hpp:104-141). Raises PotError(Overflow) like the reference."""
    lib = load_library()
    ctx = ctx or default_context()
    keep: list = []
    prob = _problem(inst, keep)
    n = inst.size()
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    row = np.empty(n)
    col = np.empty(n)
    sc = np.empty(6)
    _check(lib.potgpu_dual_eval(ctx._h, ctypes.byref(prob), float(gamma), _dp(u), _dp(v), float(w), _dp(row),
                                _dp(col), _dp(sc)))
    return DualEval(row, col, sc[0], sc[1], sc[2], sc[3], sc[4])


def make_synthetic_instance(n: int, seed: int, mass_r: float, mass_c: float, s_frac: float) -> Instance:
    """synthetic.hpp:15-54 (bit-identical draw order)."""
    lib = load_library()
    r, c, C, s = np.empty(n), np.empty(n), np.empty((n, n)), np.empty(1)
    rc = lib.potgpu_make_synthetic(n, seed, mass_r, mass_c, s_frac, _dp(r), _dp(c), _dp(C), _dp(s))
    if rc:
        raise PotError(ErrorCode(rc - 1), "invalid synthetic instance parameters")
    return Instance(r=r, c=c, s=float(s[0]), C=C)


def make_scaling_instance(n: int, seed: int) -> Instance:  # synthetic.hpp:58-60
    return make_synthetic_instance(n, seed, 5.0, 3.0, 0.2)


def make_config_points(config_id: int, n: int, seed: int = 1):
    """BASELINE.json configs[config_id - 1] as points: returns
    (r, c, X, Y, s, cost_scale)."""
    lib = load_library()
    r, c = np.empty(n), np.empty(n)
    X, Y = np.empty((n, 3)), np.empty((n, 3))
    d = ctypes.c_int(0)
    s, sc = np.empty(1), np.empty(1)
    rc = lib.potgpu_make_config(config_id, n, seed, _dp(r), _dp(c), _dp(X), _dp(Y), ctypes.byref(d), _dp(s), _dp(sc))
    if rc:
        raise PotError(ErrorCode(rc - 1), "invalid config id / size")
    dd = d.value
    X = X.reshape(-1)[: n * dd].reshape(n, dd).copy()
    Y = Y.reshape(-1)[: n * dd].reshape(n, dd).copy()
    return r, c, X, Y, float(s[0]), float(sc[0])


def dense_cost(X: np.ndarray, Y: np.ndarray, cost_scale: float) -> np.ndarray:
    """C_ij = cost_scale * |x_i - y_j|^2 with the cost views' fp64 association."""
    C = np.zeros((X.shape[0], Y.shape[0]))
    for k in range(X.shape[1]):
        D = X[:, k][:, None] - Y[:, k][None, :]
        C = C + D * D
    return C * cost_scale


def points_scale(X: np.ndarray, Y: np.ndarray, chunk: int = 1024) -> float:
    """1 / max_ij |x_i - y_j|^2 (same fp64 association as the device)."""
    m = 0.0
    for a in range(0, X.shape[0], chunk):
        m = max(m, float(dense_cost(X[a:a + chunk], Y, 1.0).max()))
    return 1.0 / m if m > 0 else 1.0


def config_instance(config_id: int, n: Optional[int] = None, seed: int = 1, dense: Optional[bool] = None,
                    dtype: Optional[DType] = None) -> Instance:
    """Instance for a BASELINE.json workload."""
    defaults = {1: (1000, True, DType.F64), 2: (4096, True, DType.F64), 3: (16384, False, DType.F32),
                4: (65536, False, DType.F32), 5: (2048, True, DType.F32)}
    n0, dense0, dt0 = defaults[config_id]
    n = n or n0
    dense = dense0 if dense is None else dense
    dtype = dt0 if dtype is None else dtype
    r, c, X, Y, s, scale = make_config_points(config_id, n, seed)
    if dtype == DType.F32:  # fp32 instances: coordinates are rounded once, here
        X = X.astype(np.float32).astype(np.float64)
        Y = Y.astype(np.float32).astype(np.float64)
        scale = points_scale(X, Y) if (dense or n <= 8192) else 0.0  # 0: derived on the device
    if dense:
        C = dense_cost(X, Y, scale)
        if dtype == DType.F32:
            C = C.astype(np.float32).astype(np.float64)
        return Instance(r=r, c=c, s=s, C=C, dtype=dtype)
    return Instance(r=r, c=c, s=s, X=X, Y=Y, cost_scale=scale if scale > 0 else None, dtype=dtype)


# ------------------------------------------------------------------ registration --
@dataclass
class RigidTransform:  # registration.hpp:13-33: y -> R y + t
    R: np.ndarray = field(default_factory=lambda: np.eye(3))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def apply(self, y) -> np.ndarray:
        return self.R @ np.asarray(y, dtype=np.float64) + self.t

    def apply_all(self, pts) -> np.ndarray:
        pts = np.asarray(pts, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != 3:
            raise PotError(ErrorCode.DimensionMismatch, "point cloud must be N x 3")
        return pts @ self.R.T + self.t

    @staticmethod
    def compose(a: "RigidTransform", b: "RigidTransform") -> "RigidTransform":
        return RigidTransform(a.R @ b.R, a.R @ b.t + a.t)


@dataclass
class RegistrationConfig:  # registration.hpp:75-100
    alpha: float = 0.4
    gamma0: float = 4.4e-3
    anneal_rate: float = 0.83
    transform_threshold: float = 1e-5
    max_registrations: int = 60
    solve: SolverConfig = field(default_factory=SolverConfig)


@dataclass
class RegistrationRecord:  # registration.hpp:102-109
    round: int
    inner_iterations: int
    accumulated_iterations: int
    cost: float
    increment: float
    gamma: float


@dataclass
class RegistrationResult:  # registration.hpp:111-115
    transform: RigidTransform
    converged: bool
    rounds: List[RegistrationRecord]


def _cloud(a, name: str) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 3:
        raise PotError(ErrorCode.DimensionMismatch, f"{name}: point clouds must be N x 3")
    return a


def register_point_clouds(reference, moving, config: RegistrationConfig = RegistrationConfig(),
                          kind: SolverKind = SolverKind.Aspot, dtype: DType = DType.F64,
                          ctx: Optional[Context] = None) -> RegistrationResult:
    """register_point_clouds (registration.hpp:127-199) on the device."""
    lib = load_library()
    ctx = ctx or default_context()
    ref, mov = _cloud(reference, "reference"), _cloud(moving, "moving")
    rc = _RegConfig(config.alpha, config.gamma0, config.anneal_rate, config.transform_threshold,
                    int(config.max_registrations))
    sc = _config(config.solve)
    res = _RegResult()
    cap = max(int(config.max_registrations), 1)
    recs = (_RegRecord * cap)()
    _check(lib.potgpu_register_point_clouds(ctx._h, int(kind), _dp(ref), ref.shape[0], _dp(mov), mov.shape[0],
                                            ctypes.byref(rc), ctypes.byref(sc), int(dtype), ctypes.byref(res), recs,
                                            cap))
    rounds = [RegistrationRecord(int(r.round), int(r.inner_iterations), int(r.accumulated_iterations), float(r.cost),
                                 float(r.increment), float(r.gamma)) for r in recs[:min(res.rounds, cap)]]
    T = RigidTransform(np.array(res.R[:], dtype=np.float64).reshape(3, 3), np.array(res.t[:], dtype=np.float64))
    return RegistrationResult(T, bool(res.converged), rounds)


def fit_rigid(pi, x_pts, y_pts, ctx: Optional[Context] = None) -> RigidTransform:
    """fit_rigid (registration.hpp:40-71): coupling reductions on the device."""
    lib = load_library()
    ctx = ctx or default_context()
    x, y = _cloud(x_pts, "x_pts"), _cloud(y_pts, "y_pts")
    pi = np.ascontiguousarray(pi, dtype=np.float64)
    if pi.shape != (x.shape[0], y.shape[0]):
        raise PotError(ErrorCode.DimensionMismatch, "coupling shape does not match the clouds")
    R, t = np.zeros(9), np.zeros(3)
    _check(lib.potgpu_fit_rigid(ctx._h, _dp(pi), pi.shape[0], pi.shape[1], _dp(x), _dp(y), _dp(R), _dp(t)))
    return RigidTransform(R.reshape(3, 3), t)


# ---------------------------------------------------------------- colour transfer --
@dataclass
class ColorHistogram:  # color_transfer.hpp:15-19
    centroids: np.ndarray  # k x 3
    weights: np.ndarray    # cluster sizes / N
    assignments: np.ndarray  # pixel -> centroid (int32)


def kmeans_quantize(points, k: int, seed: int, ctx: Optional[Context] = None) -> ColorHistogram:
    """kmeans_quantize (color_transfer.hpp:34-118): seeded k-means++ start
    (the reference's draws), Lloyd rounds on the device."""
    lib = load_library()
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2 or (pts.shape[0] and pts.shape[1] != 3):
        raise PotError(ErrorCode.DimensionMismatch, "points must be N x 3")
    n = pts.shape[0]
    C = np.zeros((max(k, 1), 3))
    W = np.zeros(max(k, 1))
    A = np.zeros(max(n, 1), dtype=np.int32)
    _check(lib.potgpu_kmeans_quantize(ctx._h, _dp(pts) if n else None, n, int(k), int(seed), _dp(C), _dp(W),
                                      A.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    return ColorHistogram(C[:k], W[:k], A[:n])


def image_to_points(rgb: np.ndarray) -> np.ndarray:
    """image_to_points (color_transfer.hpp:21-30): uint8 RGB -> [0, 1]^3."""
    return np.asarray(rgb, dtype=np.float64).reshape(-1, 3) / 255.0


def barycentric_projection(plan, source_colors, target_colors) -> np.ndarray:
    """Plan-weighted average of target colours per source row; rows without
    mass keep their source colour (color_transfer.hpp:128-141)."""
    plan = np.asarray(plan, dtype=np.float64)
    src = np.asarray(source_colors, dtype=np.float64)
    tgt = np.asarray(target_colors, dtype=np.float64)
    if plan.shape != (src.shape[0], tgt.shape[0]):
        raise PotError(ErrorCode.DimensionMismatch, "plan/color shape mismatch")
    out = src.copy()
    mass = plan.sum(axis=1)
    live = mass > 0
    out[live] = (plan[live] @ tgt) / mass[live, None]
    return out


@dataclass
class ColorTransferResult:  # color_transfer.hpp:120-124
    recolored: np.ndarray
    solve: SolveResult
    instance: Instance


def color_transfer(source: ColorHistogram, target: ColorHistogram, s_frac: float, kind: SolverKind,
                   config: SolverConfig = SolverConfig(), ctx: Optional[Context] = None) -> ColorTransferResult:
    """color_transfer (color_transfer.hpp:146-185): normalised histograms,
    squared RGB cost scaled to unit max, budget s_frac of the smaller mass,
    the solve on the device, barycentric recolouring."""
    if source.centroids.shape[0] != source.weights.shape[0] or target.centroids.shape[0] != target.weights.shape[0]:
        raise PotError(ErrorCode.DimensionMismatch, "histogram shape mismatch")
    if source.centroids.shape[0] != target.centroids.shape[0]:
        raise PotError(ErrorCode.DimensionMismatch, "histograms must have equal color counts")
    if s_frac < 0 or s_frac > 1:
        raise PotError(ErrorCode.InvalidArgument, "s_frac must lie in [0, 1]")
    norm = max(source.weights.sum(), target.weights.sum())
    if not norm > 0:
        raise PotError(ErrorCode.EmptyInput, "empty histograms")
    r, c = source.weights / norm, target.weights / norm
    d = source.centroids[:, None, :] - target.centroids[None, :, :]
    C = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
    cmax = C.max()
    if cmax > 0:
        C = C / cmax
    inst = Instance(r=r, c=c, s=s_frac * min(r.sum(), c.sum()), C=C)
    cfg = SolverConfig(**{**config.__dict__, "materialize_plan": True})
    res = solve(inst, kind, cfg, ctx=ctx)
    return ColorTransferResult(barycentric_projection(res.plan.X, source.centroids, target.centroids), res, inst)


def recolor_points(assignments, recolored) -> np.ndarray:
    """recolor_image's per-pixel rule (color_transfer.hpp:187-203) on [0,1]
    colours: each pixel takes its cluster's recoloured value, clamped and
    rounded to 8 bits."""
    vals = np.clip(np.asarray(recolored)[np.asarray(assignments)], 0.0, 1.0)
    return np.floor(vals * 255.0 + 0.5).astype(np.uint8)


# ------------------------------------------------------------- rounding / extend --
def round_pot(X, inst: Instance, ctx: Optional[Context] = None) -> TransportPlan:
    """round_pot (rounding.hpp:46-77) on the device: X projected onto U(r, c, s)."""
    lib = load_library()
    ctx = ctx or default_context()
    X = np.ascontiguousarray(X, dtype=np.float64)
    n = inst.size()
    if X.shape != (n, n):
        raise PotError(ErrorCode.DimensionMismatch, "plan shape does not match the instance")
    r = np.ascontiguousarray(inst.r, dtype=np.float64)
    c = np.ascontiguousarray(inst.c, dtype=np.float64)
    out = np.empty_like(X)
    _check(lib.potgpu_round_pot(ctx._h, n, _dp(X), _dp(r), _dp(c), float(inst.s), _dp(out)))
    return TransportPlan(X=out, row_slack=r - out.sum(axis=1), col_slack=c - out.sum(axis=0), mass=float(out.sum()))


def round_balanced(X, r, c, ctx: Optional[Context] = None) -> np.ndarray:
    """round_balanced (rounding.hpp:14-39) on the device."""
    lib = load_library()
    ctx = ctx or default_context()
    X = np.ascontiguousarray(X, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    if X.shape != (r.size, c.size):
        raise PotError(ErrorCode.DimensionMismatch, "plan/marginal shape mismatch")
    out = np.empty_like(X)
    _check(lib.potgpu_round_balanced(ctx._h, X.shape[0], X.shape[1], _dp(X), _dp(r), _dp(c), _dp(out)))
    return out


@dataclass
class ExtendedOtInstance:  # extend.hpp:11-18
    C_ext: np.ndarray
    r_ext: np.ndarray
    c_ext: np.ndarray
    penalty_A: float

    def original_size(self) -> int:
        return self.r_ext.size - 1


def extend(inst: Instance, penalty_A: float) -> ExtendedOtInstance:
    """extend (extend.hpp:22-39): the balanced dummy-node extension."""
    C = inst.C if inst.C is not None else dense_cost(inst.X, inst.Y, inst.cost_scale)
    if not penalty_A > C.max():
        raise PotError(ErrorCode.PenaltyTooSmall, f"penalty must exceed max cost {C.max()}")
    n = inst.size()
    Ce = np.zeros((n + 1, n + 1))
    Ce[:n, :n] = C
    Ce[n, n] = penalty_A
    r_ext = np.append(inst.r, max(inst.c.sum() - inst.s, 0.0))
    c_ext = np.append(inst.c, max(inst.r.sum() - inst.s, 0.0))
    return ExtendedOtInstance(Ce, r_ext, c_ext, float(penalty_A))


@dataclass
class BlockDecomposition:  # extend.hpp:41-46
    block: np.ndarray
    dummy_col: np.ndarray
    dummy_row: np.ndarray
    corner: float


def extract_block(X_ext) -> BlockDecomposition:
    """extract_block (extend.hpp:48-60)."""
    X_ext = np.asarray(X_ext, dtype=np.float64)
    if X_ext.ndim != 2 or X_ext.shape[0] != X_ext.shape[1] or X_ext.shape[0] < 2:
        raise PotError(ErrorCode.DimensionMismatch, "extended plan must be square with side >= 2")
    n = X_ext.shape[0] - 1
    return BlockDecomposition(X_ext[:n, :n].copy(), X_ext[:n, n].copy(), X_ext[n, :n].copy(), float(X_ext[n, n]))


# ------------------------------------------------------------- core / dual helpers --
def solver_kind_from_name(name: str) -> Optional[SolverKind]:  # core.hpp:225-231
    return {"aspot": SolverKind.Aspot, "sinkhorn": SolverKind.FeasibleSinkhorn,
            "tuned-sinkhorn": SolverKind.TunedSinkhorn}.get(name)


@dataclass
class Violation:  # core.hpp:76-79
    code: ErrorCode
    detail: str


class ValidationError(PotError):  # core.hpp:82-104: carries every violation
    def __init__(self, violations: List[Violation]):
        code = violations[0].code if violations else ErrorCode.InvalidArgument
        msg = "invalid instance" + "".join(f"; {v.code.name} ({v.detail})" for v in violations)
        super().__init__(code, msg)
        self.violations = violations


def validation_report(inst: Instance) -> List[Violation]:  # core.hpp:131-162
    out: List[Violation] = []
    r, c = np.asarray(inst.r, dtype=np.float64), np.asarray(inst.c, dtype=np.float64)
    n = r.size
    if n == 0:
        return [Violation(ErrorCode.EmptyInput, "marginals are empty")]
    C = inst.C
    if c.size != n:
        out.append(Violation(ErrorCode.DimensionMismatch, f"r has {n} entries, c has {c.size}"))
    if C is not None and np.shape(C) != (n, n):
        out.append(Violation(ErrorCode.DimensionMismatch, f"cost matrix is {np.shape(C)}, expected {n}x{n}"))
    Cf = np.asarray(C if C is not None else np.zeros(0), dtype=np.float64)
    if not (np.all(np.isfinite(r)) and np.all(np.isfinite(c)) and np.all(np.isfinite(Cf)) and math.isfinite(inst.s)):
        out.append(Violation(ErrorCode.NonFiniteEntry, "non-finite entry in r, c, C or s"))
    else:
        if np.any(r < 0) or np.any(c < 0):
            out.append(Violation(ErrorCode.NegativeEntry, "negative marginal entry"))
        if Cf.size and np.any(Cf < 0):
            out.append(Violation(ErrorCode.NegativeEntry, "negative cost entry"))
        if inst.s < 0:
            out.append(Violation(ErrorCode.NegativeEntry, "negative budget"))
        if c.size == n and inst.s > min(r.sum(), c.sum()) + 1e-12:
            out.append(Violation(ErrorCode.BudgetExceedsMass,
                                 f"budget {inst.s} exceeds min marginal mass {min(r.sum(), c.sum())}"))
    return out


def validate(inst: Instance) -> Instance:  # core.hpp:164-169
    v = validation_report(inst)
    if v:
        raise ValidationError(v)
    return inst


@dataclass
class DualPoint:  # dual.hpp:15-43
    u: np.ndarray
    v: np.ndarray
    w: float = 0.0

    @staticmethod
    def zero(n: int) -> "DualPoint":
        return DualPoint(np.zeros(n), np.zeros(n), 0.0)

    def all_finite(self) -> bool:
        return bool(np.all(np.isfinite(self.u)) and np.all(np.isfinite(self.v)) and math.isfinite(self.w))

    def __add__(self, o):
        return DualPoint(self.u + o.u, self.v + o.v, self.w + o.w)

    def __sub__(self, o):
        return DualPoint(self.u - o.u, self.v - o.v, self.w - o.w)

    def __rmul__(self, a: float):
        return DualPoint(a * self.u, a * self.v, a * self.w)


kMaxExponent = 700.0  # dual.hpp:47


class EntropicContext:  # dual.hpp:52-75 (logK built on access; reductions on the device)
    def __init__(self, C, gamma: float, r, c, s: float):
        if not (gamma > 0) or not math.isfinite(gamma):
            raise PotError(ErrorCode.InvalidArgument, "gamma must be positive")
        self.C = np.ascontiguousarray(C, dtype=np.float64)
        self.r, self.c = np.asarray(r, dtype=np.float64), np.asarray(c, dtype=np.float64)
        if self.C.shape != (self.r.size, self.c.size):
            raise PotError(ErrorCode.DimensionMismatch, "cost/marginal shape mismatch")
        self.gamma, self.s = float(gamma), float(s)

    @staticmethod
    def from_instance(inst: Instance, gamma: float) -> "EntropicContext":
        C = inst.C if inst.C is not None else dense_cost(inst.X, inst.Y, inst.cost_scale)
        return EntropicContext(C, gamma, inst.r, inst.c, inst.s)

    @property
    def logK(self) -> np.ndarray:
        return (-self.C) / self.gamma

    def size(self) -> int:
        return self.r.size

    def _inst(self) -> Instance:
        return Instance(r=self.r, c=self.c, s=self.s, C=self.C)


def _eexp(x):  # Eigen's packet exp (clamped argument)
    x = np.asarray(x, dtype=np.float64)
    return np.where(np.isnan(x) | (x == np.inf), np.exp(x), np.exp(np.clip(x, -709.784, 709.784)))


def _check_dual(ectx: EntropicContext, z: DualPoint, ranges=True):
    if z.u.size != ectx.size() or z.v.size != ectx.size():
        raise PotError(ErrorCode.DimensionMismatch, "dual point shape mismatch")
    if ranges:
        for x, what in ((z.u, "exp(u)"), (z.v, "exp(v)")):
            m = np.max(x) if x.size else -np.inf
            if not (m <= kMaxExponent):
                raise PotError(ErrorCode.Overflow, f"{what} exponent exceeds representable range")


def _dual_matrix(ectx: EntropicContext, z: DualPoint, which: int, ctx=None) -> np.ndarray:
    lib = load_library()
    ctx = ctx or default_context()
    keep: list = []
    prob = _problem(ectx._inst(), keep)
    n = ectx.size()
    out = np.empty((n, n))
    u, v = np.ascontiguousarray(z.u, dtype=np.float64), np.ascontiguousarray(z.v, dtype=np.float64)
    _check(lib.potgpu_dual_matrix(ctx._h, ctypes.byref(prob), ectx.gamma, _dp(u), _dp(v), float(z.w), which, _dp(out)))
    return out


def exponent_matrix(ectx: EntropicContext, z: DualPoint, ctx=None) -> np.ndarray:  # dual.hpp:92-99
    _check_dual(ectx, z, ranges=False)
    return _dual_matrix(ectx, z, 0, ctx)


def b_matrix(ectx: EntropicContext, z: DualPoint, ctx=None) -> np.ndarray:  # dual.hpp:103-109
    _check_dual(ectx, z, ranges=False)
    return _dual_matrix(ectx, z, 1, ctx)


def dual_gradient(ectx: EntropicContext, z: DualPoint, ctx=None) -> DualPoint:  # dual.hpp:122-133
    _check_dual(ectx, z)
    ev = dual_eval(ectx._inst(), ectx.gamma, z.u, z.v, z.w, ctx=ctx)
    return DualPoint((ev.row + _eexp(z.u)) - ectx.r, (ev.col + _eexp(z.v)) - ectx.c, ev.total - ectx.s)


def dual_objective(ectx: EntropicContext, z: DualPoint, ctx=None) -> float:  # dual.hpp:111-120
    _check_dual(ectx, z)
    ev = dual_eval(ectx._inst(), ectx.gamma, z.u, z.v, z.w, ctx=ctx)
    return ((((ev.total + _eexp(z.u).sum()) + _eexp(z.v).sum()) - float(z.u @ ectx.r)) - float(z.v @ ectx.c)) \
        - z.w * ectx.s


def feasibility_error(ectx: EntropicContext, z: DualPoint, ctx=None) -> float:  # dual.hpp:135-139
    g = dual_gradient(ectx, z, ctx)
    return float(np.abs(g.u).sum() + np.abs(g.v).sum() + abs(g.w))


def rho(a: float, b: float) -> float:  # dual.hpp:141-146
    if not (a > 0) or not (b > 0):
        raise PotError(ErrorCode.NonPositiveArgument, "rho requires a, b > 0")
    return b - a + a * math.log(a / b)


def rho_limit(a: float, b: float) -> float:  # dual.hpp:150-158
    if not (a > 0):
        return b
    if not (b > 0):
        return math.inf
    return rho(a, b)


def greenkhorn_step(ectx: EntropicContext, z: DualPoint, rule: BlockRule, t: int, ctx=None) -> DualPoint:
    """solvers.hpp:43-89: sums on the device, block choice / update on the host."""
    _check_dual(ectx, z)
    ev = dual_eval(ectx._inst(), ectx.gamma, z.u, z.v, z.w, ctx=ctx)
    row, col = ev.row + _eexp(z.u), ev.col + _eexp(z.v)
    if rule == BlockRule.RoundRobin:
        block = t % 3
    else:
        su = sum(rho_limit(a, b) for a, b in zip(ectx.r, row))
        sv = sum(rho_limit(a, b) for a, b in zip(ectx.c, col))
        sw = rho_limit(ectx.s, ev.total)
        block, best = 0, su
        if sv > best:
            block, best = 1, sv
        if sw > best:
            block = 2
    with np.errstate(divide="ignore", invalid="ignore"):
        if block == 0:
            out = DualPoint(z.u + (np.log(ectx.r) - np.log(row)), z.v.copy(), z.w)
        elif block == 1:
            out = DualPoint(z.u.copy(), z.v + (np.log(ectx.c) - np.log(col)), z.w)
        else:
            out = DualPoint(z.u.copy(), z.v.copy(), z.w + (math.log(ectx.s) - math.log(ev.total)
                                                           if ectx.s > 0 and ev.total > 0 else -math.inf))
    if not out.all_finite():
        raise PotError(ErrorCode.Overflow, "block update left the exp range")
    return out


@dataclass
class AspotSetup:  # solvers.hpp:94-99
    gamma: float
    eps_tilde: float
    mixed_r: np.ndarray
    mixed_c: np.ndarray


def aspot_setup(inst: Instance, epsilon: float) -> AspotSetup:  # solvers.hpp:100-133
    validate(inst)
    if not (epsilon > 0) or not math.isfinite(epsilon):
        raise PotError(ErrorCode.InvalidArgument, "epsilon must be positive")
    n = inst.size()
    if n < 2:
        raise PotError(ErrorCode.DegenerateInstance, "accelerated setup needs n >= 2 (log n vanishes)")
    gamma = epsilon / (4.0 * math.log(float(n)))
    C = inst.C if inst.C is not None else dense_cost(inst.X, inst.Y, inst.cost_scale)
    cmax = float(np.max(C))
    eps_t = epsilon / (8.0 * cmax) if cmax > 0 else math.inf
    sr, sc = float(np.sum(inst.r)), float(np.sum(inst.c))
    if sr > 1:
        eps_t = min(eps_t, 8.0 * (sr - inst.s) / (sr - 1.0))
    if sc > 1:
        eps_t = min(eps_t, 8.0 * (sc - inst.s) / (sc - 1.0))
    if not (gamma > 0) or not math.isfinite(gamma):
        raise PotError(ErrorCode.DegenerateInstance, "derived gamma is not positive")
    if not (eps_t > 0):
        raise PotError(ErrorCode.DegenerateInstance, "stopping tolerance collapsed to zero (budget equals mass)")
    lam = min(eps_t / 8.0, 0.5)
    return AspotSetup(gamma, eps_t, (1.0 - lam) * np.asarray(inst.r) + lam / n, (1.0 - lam) * np.asarray(inst.c) + lam / n)


def theta_next(theta: float) -> float:  # solvers.hpp:32-37
    return theta * (math.sqrt(theta * theta + 4.0) - theta) / 2.0


def entropy(x) -> float:  # solvers.hpp:19-28
    x = np.asarray(x, dtype=np.float64)
    if np.any(x < 0):
        raise PotError(ErrorCode.NegativeEntry, "entropy requires x >= 0")
    xp = x[x > 0]
    return float(-(xp * np.log(xp)).sum())


def dummy_penalty(cmax: float, epsilon: float) -> float:  # solvers.hpp:485-490
    A = 8.0 * cmax / epsilon if cmax > 0 else 0.0
    if not (A > cmax) or not math.isfinite(A):
        A = 2.0 * cmax if cmax > 0 else 1.0
    return A


@dataclass
class AspotIterate:  # solvers.hpp:188-202
    t: int
    theta: float
    error: float
    ctx: EntropicContext
    z_grave: DualPoint
    z_hat: DualPoint
    z_best: DualPoint
    z_check: DualPoint
    phi_hat: float
    phi_best: float
    phi_check: float


def theory_bounds(inst: Instance, gamma: float, eps_prime: float) -> TheoryBounds:  # solvers.hpp:146-174
    if not (gamma > 0) or not math.isfinite(gamma):
        raise PotError(ErrorCode.InvalidArgument, "gamma must be positive")
    if not (eps_prime > 0) or not math.isfinite(eps_prime):
        raise PotError(ErrorCode.InvalidArgument, "eps_prime must be positive")
    sr, sc = float(np.sum(inst.r)), float(np.sum(inst.c))
    M = max(sr, sc)
    if not (M > inst.s):
        raise PotError(ErrorCode.DegenerateInstance, "dual radius is infinite when budget equals max mass")
    me = min(float(np.min(inst.r)), float(np.min(inst.c)))
    if not (me > 0):
        raise PotError(ErrorCode.DegenerateInstance, "dual radius needs strictly positive marginals")
    C = inst.C if inst.C is not None else dense_cost(inst.X, inst.Y, inst.cost_scale)
    R = float(np.max(C)) * M / (gamma * (M - inst.s)) - math.log(me)
    mu = gamma / (sr + sc - inst.s)
    L = 3.0 / mu
    return TheoryBounds(R, L, mu, 1.0 + (12.0 * math.sqrt(14.0 * inst.size() * L) * R / eps_prime) ** (2.0 / 3.0))
