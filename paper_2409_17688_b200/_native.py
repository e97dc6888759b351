"""Thin ctypes binding of libminplus.so (include/minplus.h).

Argument marshalling only: every step of the path runs in the library's CUDA kernels.
There is no CPU fallback -- if the shared library is missing this module raises at import,
and every computing call raises MinplusError(MP_ERR_CUDA) when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _build

MP_INF = 0xFFFF
MP_FINITE_MAX = 0x7FFE
MP_MAX_K = 256
MP_MAX_N = 13

STATUS = {0: "MP_OK", 1: "MP_ERR_DOMAIN", 2: "MP_ERR_RANGE", 3: "MP_ERR_RESOURCE",
          4: "MP_ERR_NOT_PERIODIC", 5: "MP_ERR_CUDA", 6: "MP_ERR_COMM"}

# Every symbol include/minplus.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "mp_count_words", "build_transition_matrix", "build_transition_matrix_into", "mp_free",
    "minplus_mul", "minplus_mul_device", "minplus_power_until_periodic",
    "minplus_power_until_periodic_device", "minplus_power_rows", "mp_set_stream",
    "gamma2_cylinder",
    "mp_gamma2_readoff", "mp_dist_set", "mp_shard_range", "mp_fingerprint_unit",
    "mp_repeat_candidate", "mp_last_error", "mp_shutdown", "mp_version", "mp_kernel_launches",
    "mp_last_profile", "mp_set_options", "mp_set_grouping", "mp_set_spmm_width", "mp_gamma2_formula", "mp_gamma2_record",
    "mp_set_symmetry", "mp_set_word_symmetry", "mp_word_reversal", "minplus_mul_strided_batched_device",
    "minplus_closure", "mp_set_power_observer", "mp_column_plan", "mp_set_small_path",
    "mp_set_transfer_hint", "mp_set_row_reuse", "mp_dist_set_allgather",
]


class MinplusError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {message}")


class _PeriodicResult(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_int32), ("lambda_", ctypes.c_int32), ("offset", ctypes.c_int32),
                ("k_last", ctypes.c_int32), ("dense_from", ctypes.c_int32),
                ("diag_min", ctypes.c_uint16 * (MP_MAX_K + 1)),
                ("fingerprint", ctypes.c_uint64 * (MP_MAX_K + 1))]


class PowerStats(ctypes.Structure):
    _fields_ = [("fingerprint", ctypes.c_int64), ("inf_count", ctypes.c_int64),
                ("diag_min", ctypes.c_int64), ("ref", ctypes.c_int64)]


class _Formula(ctypes.Structure):
    _fields_ = [("a", ctypes.c_int32), ("b", ctypes.c_int32), ("n0", ctypes.c_int32),
                ("r0_k50", ctypes.c_int32),
                ("alpha", ctypes.c_int32 * MP_MAX_K), ("n_exceptions", ctypes.c_int32),
                ("exception_m", ctypes.c_int64 * MP_MAX_K), ("exception_gamma2", ctypes.c_int64 * MP_MAX_K)]


class _Profile(ctypes.Structure):
    _fields_ = [("product_ms", ctypes.c_double), ("product_launches", ctypes.c_int64),
                ("dense_steps", ctypes.c_double), ("issued_steps", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("setup_ms", ctypes.c_double), ("stats_ms", ctypes.c_double),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
                ("kernel", ctypes.c_int32), ("spmm_cols", ctypes.c_int32),
                ("local_cols", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("spmm_ms", ctypes.c_double), ("row_levels", ctypes.c_int32), ("row_parents", ctypes.c_int64),
                ("fold_bytes", ctypes.c_double)]


OBSERVER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                ctypes.c_void_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.c_void_p)


def _so_path() -> str:
    """The product library, or a diagnostic build named by MP_LIB_PATH (bench_tools variants
    are loaded this way; nothing ever overwrites the product .so)."""
    return os.environ.get("MP_LIB_PATH") or _build.SO


def _load() -> ctypes.CDLL:
    so = _so_path()
    if not os.path.exists(so):
        raise ImportError(f"{so} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(so)
    P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    sig = {
        "mp_count_words": ([i32, P], i32),
        "build_transition_matrix": ([i32, P, P], i32),
        "build_transition_matrix_into": ([i32, P, i64], i32),
        "mp_free": ([P], None),
        "minplus_mul": ([P, P, P, i64, i64, i64], i32),
        "minplus_mul_device": ([P, i64, P, i64, P, i64, i64, i64, i64, P], i32),
        "minplus_power_until_periodic": ([P, i64, i32, P], i32),
        "minplus_power_rows": ([P, i64, i32, P, i32, P], i32),
        "minplus_power_until_periodic_device": ([P, i64, i64, i32, P], i32),
        "mp_set_stream": ([P], i32),
        "gamma2_cylinder": ([i32, i64, P], i32),
        "mp_gamma2_readoff": ([P, i64, P], i32),
        "mp_dist_set": ([i32, i32, ALLREDUCE_FN, P], i32),
        "mp_shard_range": ([i64, i32, i32, P, P], i32),
        "mp_fingerprint_unit": ([i64], ctypes.c_uint64),
        "mp_repeat_candidate": ([P, P, ctypes.c_uint64, P], i32),
        "mp_last_error": ([], ctypes.c_char_p),
        "mp_shutdown": ([], None),
        "mp_version": ([], ctypes.c_char_p),
        "mp_kernel_launches": ([], i64),
        "mp_last_profile": ([P], i32),
        "mp_set_options": ([i32, i64], i32),
        "mp_set_grouping": ([i32], i32),
        "mp_set_spmm_width": ([i32], i32),
        "mp_set_symmetry": ([ctypes.c_void_p, i64], i32),
        "minplus_mul_strided_batched_device": ([P, i64, i64, P, i64, i64, P, i64, i64, i64, i64, i64, i64, P], i32),
        "minplus_closure": ([P, i64, P, ctypes.c_void_p], i32),
        "mp_set_word_symmetry": ([i32], i32),
        "mp_word_reversal": ([i32, ctypes.c_void_p, i64], i32),
        "mp_gamma2_formula": ([P, P], i32),
        "mp_gamma2_record": ([i32, P], i32),
        "mp_set_power_observer": ([OBSERVER_FN, P], i32),
        "mp_column_plan": ([i64, i64, P, P, P], i32),
        "mp_set_small_path": ([i32], i32),
        "mp_set_transfer_hint": ([i32], i32),
        "mp_set_row_reuse": ([i32], i32),
        "mp_dist_set_allgather": ([ALLGATHER_FN, P], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


lib = _load()


def _check(status: int) -> None:
    if status != 0:
        raise MinplusError(status, lib.mp_last_error().decode(errors="replace"))


def _host_u16(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a), dtype=np.uint16)
    return a


# --------------------------------------------------------------------------------- a1
def count_words(n: int) -> int:
    N = ctypes.c_int64(0)
    _check(lib.mp_count_words(n, ctypes.byref(N)))
    return N.value


def build_transition_matrix(n: int) -> np.ndarray:
    """A(D_n), N x N uint16 with 0xFFFF = +inf (Algorithm 1)."""
    N = count_words(n)
    A = np.empty((N, N), dtype=np.uint16)
    _check(lib.build_transition_matrix_into(n, A.ctypes.data, N))
    return A


# --------------------------------------------------------------------------------- a3
def minplus_mul(A, B) -> np.ndarray:
    """C = A (x) B for host matrices, computed by the sm_100a kernel."""
    A, B = _host_u16(A), _host_u16(B)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
        raise MinplusError(1, f"shape mismatch {A.shape} x {B.shape}")
    M, K = A.shape
    N = B.shape[1]
    C = np.empty((M, N), dtype=np.uint16)
    _check(lib.minplus_mul(A.ctypes.data, B.ctypes.data, C.ctypes.data, M, K, N))
    return C


def minplus_mul_device(A, B, C=None, stream=None):
    """C = A (x) B for torch CUDA tensors (uint16 or int16 storage, boundary encoding)."""
    import torch
    for t in (A, B):
        if not t.is_cuda or t.element_size() != 2 or t.dim() != 2 or t.stride(1) != 1:
            raise MinplusError(1, "expected 2-D row-major 16-bit CUDA tensors")
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise MinplusError(1, f"shape mismatch {tuple(A.shape)} x {tuple(B.shape)}")
    if C is None:
        C = torch.empty((M, N), dtype=A.dtype, device=A.device)
    if stream is None:
        stream = torch.cuda.current_stream(A.device)
    with torch.cuda.device(A.device):
        _check(lib.minplus_mul_device(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                                      C.data_ptr(), C.stride(0), M, K, N, stream.cuda_stream))
    return C


def minplus_mul_batched_device(A, B, C=None, stream=None):
    """C[b] = A[b] (x) B[b] for 3-D torch CUDA tensors (batch, rows, cols), 16-bit storage,
    row-major matrices (stride(2) == 1); one library call (strided batch)."""
    import torch
    for t in (A, B):
        if not t.is_cuda or t.element_size() != 2 or t.dim() != 3 or t.stride(2) != 1:
            raise MinplusError(1, "expected 3-D 16-bit CUDA tensors with contiguous rows")
    nb, M, K = A.shape
    nb2, K2, N = B.shape
    if nb != nb2 or K != K2:
        raise MinplusError(1, f"shape mismatch {tuple(A.shape)} x {tuple(B.shape)}")
    if C is None:
        C = torch.empty((nb, M, N), dtype=A.dtype, device=A.device)
    if stream is None:
        stream = torch.cuda.current_stream(A.device)
    with torch.cuda.device(A.device):
        _check(lib.minplus_mul_strided_batched_device(
            A.data_ptr(), A.stride(1), A.stride(0), B.data_ptr(), B.stride(1), B.stride(0),
            C.data_ptr(), C.stride(1), C.stride(0), M, K, N, nb, stream.cuda_stream))
    return C


def minplus_closure(W: np.ndarray):
    """(D, t): D = (I (+) W)^(2^t), the all-pairs shortest path lengths of the weighted
    adjacency W (uint16, 0xFFFF = no arc), t = the number of squarings."""
    W = np.ascontiguousarray(W, dtype=np.uint16)
    if W.ndim != 2 or W.shape[0] != W.shape[1]:
        raise MinplusError(1, "expected a square matrix")
    D = np.empty_like(W)
    t = ctypes.c_int32(0)
    _check(lib.minplus_closure(W.ctypes.data, W.shape[0], D.ctypes.data, ctypes.byref(t)))
    return D, t.value


# ----------------------------------------------------------------------------- a3-a5
@dataclass
class PeriodicResult:
    mu: int
    lam: int
    offset: int
    k_last: int
    dense_from: int
    diag_min: list = field(default_factory=list)
    fingerprint: list = field(default_factory=list)
    _raw: object = None

    def gamma2(self, m: int) -> int:
        g = ctypes.c_int64(0)
        _check(lib.mp_gamma2_readoff(ctypes.byref(self._raw), m, ctypes.byref(g)))
        return g.value

    def formula(self) -> dict:
        """Closed formula gamma_2 = ceil(b m / a) + alpha[m mod a] for m >= n0, with the
        exceptions below n0 (Table 7)."""
        f = _Formula()
        _check(lib.mp_gamma2_formula(ctypes.byref(self._raw), ctypes.byref(f)))
        return {"a": f.a, "b": f.b, "n0": f.n0, "r0_k50": f.r0_k50, "alpha": [f.alpha[k] for k in range(f.a)],
                "exceptions": {int(f.exception_m[i]): int(f.exception_gamma2[i]) for i in range(f.n_exceptions)}}


def _result(r: _PeriodicResult) -> PeriodicResult:
    k = r.k_last + 1
    return PeriodicResult(r.mu, r.lambda_, r.offset, r.k_last, r.dense_from, r.diag_min[:k], r.fingerprint[:k], r)


def minplus_power_until_periodic(A, max_k: int = 64) -> PeriodicResult:
    """Powers A^k = A (x) A^{k-1} on the device until A^{mu+lambda} = b (x) A^mu."""
    A = _host_u16(A)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise MinplusError(1, f"A must be square, got {A.shape}")
    r = _PeriodicResult()
    _check(lib.minplus_power_until_periodic(A.ctypes.data, A.shape[0], max_k, ctypes.byref(r)))
    return _result(r)


def minplus_power_until_periodic_device(dA, max_k: int = 64) -> PeriodicResult:
    """Same run with A resident on the device (a 2-D 16-bit torch CUDA tensor)."""
    if not dA.is_cuda or dA.element_size() != 2 or dA.dim() != 2 or dA.stride(1) != 1 \
            or dA.shape[0] != dA.shape[1]:
        raise MinplusError(1, "expected a square row-major 16-bit CUDA tensor")
    import torch
    r = _PeriodicResult()
    # the run is enqueued on the library stream of this device: unless that is torch's current
    # stream (set_stream), wait for whatever torch still has in flight on dA.  (The raw-handle
    # and device getters cost a fraction of the public wrappers: microseconds at small n.)
    dev = dA.device.index
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    handle = raw(dev) if raw else torch.cuda.current_stream(dev).cuda_stream
    if _lib_stream.get(dev) != handle:
        torch.cuda.current_stream(dev).synchronize()
    args = (dA.data_ptr(), dA.stride(0), dA.shape[0], max_k, ctypes.byref(r))
    getdev = getattr(torch._C, "_cuda_getDevice", torch.cuda.current_device)
    if getdev() == dev:  # (the device switch costs microseconds at small n)
        _check(lib.minplus_power_until_periodic_device(*args))
    else:
        with torch.cuda.device(dev):
            _check(lib.minplus_power_until_periodic_device(*args))
    return _result(r)


_lib_stream = {}  # device index -> the cudaStream_t the power runs use (set_stream)


def set_stream(stream) -> None:
    """Run power sequences on `stream` (torch.cuda.Stream or None for the library's own),
    on the current device."""
    import torch
    handle = None if stream is None else stream.cuda_stream
    # torch's default stream is the legacy default stream (handle 0), which the ABI takes as
    # cudaStreamLegacy: NULL would mean "the library's own stream"
    _check(lib.mp_set_stream(None if handle is None else (handle or _CUDA_STREAM_LEGACY)))
    _lib_stream[torch.cuda.current_device()] = handle


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy


def minplus_power_rows(A, rows, kmax: int) -> np.ndarray:
    """Rows of A^1..A^kmax from the device path: array [kmax, len(rows), N]."""
    A = _host_u16(A)
    N = A.shape[0]
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    out = np.empty((kmax, len(r), N), dtype=np.uint16)
    _check(lib.minplus_power_rows(A.ctypes.data, N, kmax, r.ctypes.data, len(r), out.ctypes.data))
    return out


def gamma2_cylinder(n: int, m: int) -> int:
    """gamma_2(P_n x C_m) (Theorems 2 and 3)."""
    g = ctypes.c_int64(0)
    _check(lib.gamma2_cylinder(n, m, ctypes.byref(g)))
    return g.value


def gamma2_record(n: int) -> PeriodicResult:
    """The cached power-sequence record gamma2_cylinder(n, .) reads from."""
    r = _PeriodicResult()
    _check(lib.mp_gamma2_record(n, ctypes.byref(r)))
    return _result(r)


_observer_keep = []


def set_power_observer(fn=None) -> None:
    """Parity hook: fn(k, power) is called for every power A^k of every following run, power
    = the whole N x N matrix (uint16 numpy view of a library buffer, valid only during the
    call: copy what you keep).  fn returning True stops the run (MP_ERR_DOMAIN).  None clears."""
    if fn is None:
        _check(lib.mp_set_power_observer(OBSERVER_FN(), None))
        _observer_keep.clear()
        return

    def cb(ctx, k, ptr, N):
        try:
            buf = (ctypes.c_uint16 * (N * N)).from_address(ptr)
            return 1 if fn(int(k), np.frombuffer(buf, dtype=np.uint16).reshape(N, N)) else 0
        except Exception:  # noqa: BLE001 -- reported to C as a stopped run
            import traceback
            traceback.print_exc()
            return 1

    c = OBSERVER_FN(cb)
    _observer_keep[:] = [c]
    _check(lib.mp_set_power_observer(c, None))


# -------------------------------------------------------------------------- multi-GPU
_keep_alive = []


def dist_set(rank: int, world: int, allreduce) -> None:
    """Registers allreduce(op, dev_ptr, count) -> None (op 0 = SUM, 1 = MIN) for the
    column-sharded power run; allreduce=None clears the context."""
    if allreduce is None:
        _check(lib.mp_dist_set(0, 1, ALLREDUCE_FN(), None))
        _keep_alive.clear()
        _gather_keep.clear()
        return

    def cb(ctx, op, dev_ptr, count, stream):
        try:
            allreduce(int(op), int(dev_ptr), int(count))
            return 0
        except Exception:  # noqa: BLE001 -- reported to C as MP_ERR_COMM
            import traceback
            traceback.print_exc()
            return 1

    fn = ALLREDUCE_FN(cb)
    _keep_alive[:] = [fn]
    _check(lib.mp_dist_set(rank, world, fn, None))


def dist_set_allgather(allgather) -> None:
    """Registers allgather(send_ptr, recv_ptr, nbytes) -> None (device pointers; recv holds
    world * nbytes, rank order) for the sharded general products; None clears it."""
    if allgather is None:
        _check(lib.mp_dist_set_allgather(ALLGATHER_FN(), None))
        _gather_keep.clear()
        return

    def cb(ctx, send, recv, nbytes, stream):
        try:
            allgather(int(send), int(recv), int(nbytes))
            return 0
        except Exception:  # noqa: BLE001 -- reported to C as MP_ERR_COMM
            import traceback
            traceback.print_exc()
            return 1

    fn = ALLGATHER_FN(cb)
    _gather_keep[:] = [fn]
    _check(lib.mp_dist_set_allgather(fn, None))


_gather_keep = []


def dist_set_torch(group=None) -> None:
    """Column sharding over torch.distributed (backend nccl: NVLink/NVSwitch): the per-power
    statistics all-reduce of the power runs and the all-gather of the general products."""
    import torch
    import torch.distributed as dist

    class _Dev:
        def __init__(self, ptr, n, typestr="<i8"):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                             "version": 3, "strides": None, "stream": None}

    def dev():
        return torch.device("cuda", torch.cuda.current_device())

    def allreduce(op, ptr, count):
        t = torch.as_tensor(_Dev(ptr, count), device=dev())
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MIN, group=group)
        torch.cuda.synchronize()

    world = dist.get_world_size(group)

    def allgather(send, recv, nbytes):
        src = torch.as_tensor(_Dev(send, nbytes, "|u1"), device=dev())
        dst = torch.as_tensor(_Dev(recv, nbytes * world, "|u1"), device=dev())
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(dst, src, group=group)
        else:  # gloo (tests on one GPU): the list form
            dist.all_gather(list(dst.view(world, nbytes).unbind(0)), src, group=group)
        torch.cuda.synchronize()

    dist_set(dist.get_rank(group), world, allreduce)
    dist_set_allgather(allgather)


def shard_range(N: int, world: int, rank: int):
    c0, c1 = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib.mp_shard_range(N, world, rank, ctypes.byref(c0), ctypes.byref(c1)))
    return c0.value, c1.value


def column_plan(N: int, w: int) -> dict:
    """SpMM column plan for w local columns of an N x N power: {ld, main_cols, tail_cols}."""
    ld, mc, tc = ctypes.c_int64(0), ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib.mp_column_plan(N, w, ctypes.byref(ld), ctypes.byref(mc), ctypes.byref(tc)))
    return {"ld": ld.value, "main_cols": mc.value, "tail_cols": tc.value}


def fingerprint_unit(N: int) -> int:
    return int(lib.mp_fingerprint_unit(N))


def repeat_candidate(sk: PowerStats, sj: PowerStats, S: int):
    c = ctypes.c_int32(0)
    ok = lib.mp_repeat_candidate(ctypes.byref(sk), ctypes.byref(sj), S, ctypes.byref(c))
    return (c.value if ok else None)


# ------------------------------------------------------------------------ diagnostics
def last_error() -> str:
    return lib.mp_last_error().decode(errors="replace")


def kernel_launches() -> int:
    return int(lib.mp_kernel_launches())


def last_profile() -> dict:
    p = _Profile()
    _check(lib.mp_last_profile(ctypes.byref(p)))
    return {"product_ms": p.product_ms, "product_launches": p.product_launches,
            "dense_steps": p.dense_steps, "issued_steps": p.issued_steps, "total_ms": p.total_ms,
            "setup_ms": p.setup_ms, "stats_ms": p.stats_ms, "h2d_bytes": p.h2d_bytes, "d2h_bytes": p.d2h_bytes,
            "kernel": {0: "dense", 1: "tiles", 2: "spmm", 3: "small"}.get(p.kernel, "?"), "spmm_cols": p.spmm_cols,
            "local_cols": p.local_cols, "ld": p.ld, "row_levels": p.row_levels, "row_parents": p.row_parents,
            "spmm_ms": p.spmm_ms, "fold_bytes": p.fold_bytes}


SPARSITY = {"auto": -1, "dense": 0, "tiles": 1, "spmm": 2}


def set_options(sparsity: str = "auto", device_budget_bytes: int = 0) -> None:
    """Product kernel of the power runs: "auto" | "dense" | "tiles" | "spmm" (all exact)."""
    _check(lib.mp_set_options(SPARSITY[sparsity], device_budget_bytes))


def set_symmetry(sigma=None) -> None:
    """Symmetry hint for the matrix sources: an involution sigma with A[sigma i][sigma j] =
    A[i][j] (verified on the device by every run); None clears it."""
    if sigma is None:
        _check(lib.mp_set_symmetry(None, 0))
        return
    sg = np.ascontiguousarray(sigma, dtype=np.int32)
    _check(lib.mp_set_symmetry(sg.ctypes.data, sg.shape[0]))


def set_word_symmetry(on: bool = True) -> None:
    """Whether gamma2_cylinder / gamma2_record use the word reversal of A(D_n)."""
    _check(lib.mp_set_word_symmetry(1 if on else 0))


def word_reversal(n: int) -> np.ndarray:
    """sigma[i] = index of the reversed word i in A(D_n) (int32)."""
    N = count_words(n)
    out = np.empty(N, dtype=np.int32)
    _check(lib.mp_word_reversal(n, out.ctypes.data, N))
    return out


GROUPING = {"auto": -1, "consecutive": 0, "greedy": 1}


def set_grouping(mode: str = "auto") -> None:
    """Row grouping of the SpMM kernel: "auto" | "consecutive" | "greedy" (same product)."""
    _check(lib.mp_set_grouping(GROUPING[mode]))


def set_spmm_width(cols: int = 0) -> None:
    """CTA width of the SpMM kernel: 0 (automatic), 256, 512 or 1024 columns everywhere, or
    -256 / -512 / -1024 = that main width plus narrower remainder columns (same product)."""
    _check(lib.mp_set_spmm_width(int(cols)))


def set_transfer_hint(n: int = 0) -> None:
    """Matrix sources of order |C_n| are claimed to be A(D_n) (verified on the device by every
    run): enables the row-inclusion reuse for them.  0 clears."""
    _check(lib.mp_set_transfer_hint(int(n)))


def set_row_reuse(on: bool = True) -> None:
    """Row-inclusion reuse for A(D_n) on (default) or off (same results)."""
    _check(lib.mp_set_row_reuse(1 if on else 0))


def set_small_path(on: bool = True) -> None:
    """Whether small single-rank runs (N <= 256) use the one-launch cluster kernel."""
    _check(lib.mp_set_small_path(1 if on else 0))


def version() -> str:
    return lib.mp_version().decode()


def shutdown() -> None:
    lib.mp_shutdown()
    _lib_stream.clear()  # the per-device state, stream choice included, is gone
