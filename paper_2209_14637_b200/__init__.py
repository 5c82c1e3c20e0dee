"""paper_2209_14637_b200 -- B200-native hot path of the tensor-based sketch (arXiv 2209.14637).

Thin Python binding of ``libtsketch.so`` (the C ABI declared in ``include/tsketch.h``).
The functions here carry the same names as the C entry points and only marshal arguments:
every step of the path (Gram, eigensolver, SCW, errors) runs in the library's CUDA kernels.
There is no CPU fallback: importing works without a GPU (so symbol checks can run on CPU),
but every compute call requires the built library and a B200 and raises otherwise.

Tensors may live on the GPU (device pointers, asynchronous on the current torch stream) or
on the CPU (host pointers: the library stages them through device memory and copies results
back, synchronously -- the end-to-end path).
"""
from __future__ import annotations

import ctypes
import os
import threading
import warnings
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtsketch.so")

TSK_OK = 0
TSK_WARN_RANK_CLAMPED = 1
TSK_WARN_NOT_CONVERGED = 2
STATUS_NAMES = {0: "TSK_OK", 1: "TSK_WARN_RANK_CLAMPED", 2: "TSK_WARN_NOT_CONVERGED", -1: "TSK_EINVAL",
                -2: "TSK_ESHAPE", -3: "TSK_ENOMEM", -4: "TSK_ECUDA", -5: "TSK_ENCCL", -6: "TSK_EDEVICE", -7: "TSK_ENONFINITE",
                -8: "TSK_ENULL", -9: "TSK_ENUMERIC"}

# every symbol include/tsketch.h declares (checked by tests/test_abi.py on CPU)
EXPORTED = ["tsk_create", "tsk_destroy", "tsk_set_stream", "tsk_sync", "tsk_status_string", "tsk_launch_count",
            "sketch_gram", "sketch_topk", "sketch_train", "sketch_apply_scw", "scw_error", "sketch_gram_mode2",
            "sketch_train_two_sided", "sketch_apply_two_sided_scw", "two_sided_scw_error", "tsk_gram_probe",
            "tsk_eig_probe", "sketch_train_matrix_free", "tsk_get_unique_id", "tsk_comm_init",
            "tsk_syev_probe", "tsk_allgather_errors", "tsk_allreduce_gram", "tsk_set_scw_error_mode"]


class TskError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {STATUS_NAMES.get(status, status)} ({_status_string(status)})")


class TrainOpts(ctypes.Structure):
    _fields_ = [("oversample", ctypes.c_int), ("max_iters", ctypes.c_int), ("tol", ctypes.c_double),
                ("dense_max_m", ctypes.c_int), ("gemm_chain", ctypes.c_int), ("gemm_splits", ctypes.c_int),
                ("init_S", ctypes.c_void_p), ("check_finite", ctypes.c_int), ("cheb_degree", ctypes.c_int),
                ("tol_active", ctypes.c_int)]


class TrainInfo(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("kyfan", ctypes.c_double), ("max_resid", ctypes.c_double),
                ("gram_splits", ctypes.c_int), ("gram_tiles", ctypes.c_int), ("gap_est", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class HooiOpts(ctypes.Structure):
    _fields_ = [("max_sweeps", ctypes.c_int), ("rel_tol", ctypes.c_double)]


class HooiInfo(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int), ("converged", ctypes.c_int), ("a_fro2", ctypes.c_double),
                ("residual_history", ctypes.c_double * 65)]

    def as_dict(self):
        return {"sweeps": self.sweeps, "converged": bool(self.converged), "a_fro2": self.a_fro2,
                "residual_history": [self.residual_history[i] for i in range(self.sweeps + 1)]}


class MfOpts(ctypes.Structure):
    _fields_ = [("oversample", ctypes.c_int), ("power_iters", ctypes.c_int), ("subspace", ctypes.c_int),
                ("omega", ctypes.c_void_p)]


class MfInfo(ctypes.Structure):
    _fields_ = [("block", ctypes.c_int), ("power_iters", ctypes.c_int), ("width", ctypes.c_int),
                ("passes", ctypes.c_int), ("repairs", ctypes.c_int), ("kyfan", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Load libtsketch.so (built in-tree by ``python paper_2209_14637_b200/build.py``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libtsketch.so not built ({LIB_PATH}); run __graft_entry__.build() -- "
                               "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, f32p, f64p = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
        L.tsk_create.argtypes = [ctypes.POINTER(vp), i32, vp]
        L.tsk_destroy.argtypes = [vp]
        L.tsk_set_stream.argtypes = [vp, vp]
        L.tsk_sync.argtypes = [vp]
        L.tsk_status_string.argtypes = [i32]
        L.tsk_status_string.restype = ctypes.c_char_p
        L.tsk_launch_count.argtypes = [vp]
        L.tsk_launch_count.restype = i64
        L.sketch_gram.argtypes = [vp, f32p, i64, i32, i32, f64p, f32p, i32, vp, vp]
        L.sketch_topk.argtypes = [vp, f64p, i32, i32, f32p, f64p, vp, vp]
        L.sketch_train.argtypes = [vp, f32p, i64, i32, i32, i32, f32p, f64p, f64p, vp, vp]
        L.sketch_apply_scw.argtypes = [vp, f32p, i64, i32, i32, f32p, i32, i32, f32p, f32p, f32p]
        L.scw_error.argtypes = [vp, f32p, i64, i32, i32, f32p, i32, i32, f64p]
        L.sketch_gram_mode2.argtypes = [vp, f32p, i64, i32, i32, f64p, i32]
        L.sketch_train_two_sided.argtypes = [vp, f32p, i64, i32, i32, i32, i32, f32p, f32p, vp, vp]
        L.sketch_apply_two_sided_scw.argtypes = [vp, f32p, i64, i32, i32, f32p, i32, f32p, i32, i32, f32p, f32p,
                                                 f32p]
        L.two_sided_scw_error.argtypes = [vp, f32p, i64, i32, i32, f32p, i32, f32p, i32, i32, f64p]
        L.tsk_gram_probe.argtypes = [vp, f32p, i64, i32, i32, f64p, i32, i32, i32]
        L.tsk_eig_probe.argtypes = [vp, f64p, i32, i32, f64p, f64p, vp]
        L.tsk_syev_probe.argtypes = [vp, f64p, i32, i32, f64p, f64p, vp, ctypes.c_double]
        L.tsk_allgather_errors.argtypes = [vp, f64p, i64, f64p]
        L.tsk_allreduce_gram.argtypes = [vp, f64p, i32]
        L.tsk_set_scw_error_mode.argtypes = [vp, i32, ctypes.c_double]
        L.sketch_train_matrix_free.argtypes = [vp, f32p, i64, i32, i32, i32, f32p, f64p, vp, vp]
        L.tsk_get_unique_id.argtypes = [vp]
        L.tsk_comm_init.argtypes = [vp, i32, i32, vp]
        for f in ("tsk_create", "tsk_destroy", "tsk_set_stream", "tsk_sync", "sketch_gram", "sketch_topk",
                  "sketch_train", "sketch_apply_scw", "scw_error", "sketch_gram_mode2", "sketch_train_two_sided",
                  "sketch_apply_two_sided_scw", "two_sided_scw_error", "tsk_gram_probe", "tsk_eig_probe", "tsk_syev_probe", "tsk_allgather_errors", "tsk_allreduce_gram",
                  "tsk_set_scw_error_mode", "sketch_train_matrix_free", "tsk_get_unique_id", "tsk_comm_init"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _status_string(s: int) -> str:
    try:
        return lib().tsk_status_string(s).decode()
    except Exception:  # library missing
        return "?"


def _check(status: int, what: str) -> int:
    if status < 0:
        raise TskError(status, what)
    if status == TSK_WARN_NOT_CONVERGED:
        warnings.warn(f"{what}: iteration cap reached before the convergence test passed (result valid)",
                      RuntimeWarning)
    elif status == TSK_WARN_RANK_CLAMPED:
        warnings.warn(f"{what}: r > k, clamped to k", RuntimeWarning)
    return status


class Context:
    """A libtsketch context (tsk_ctx) on one CUDA device; follows torch's current stream."""

    def __init__(self, device: int | torch.device | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2209_14637_b200 needs a CUDA (sm_100a) device; no CPU fallback")
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            _check(lib().tsk_create(ctypes.byref(h), self.device.index, ctypes.c_void_p(stream)), "tsk_create")
        self.handle = h

    def _bind_stream(self):
        s = torch.cuda.current_stream(self.device).cuda_stream
        _check(lib().tsk_set_stream(self.handle, ctypes.c_void_p(s)), "tsk_set_stream")

    def sync(self):
        _check(lib().tsk_sync(self.handle), "tsk_sync")

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        """Join the NCCL communicator `uid` (from get_unique_id on one rank, broadcast by the caller) as
        `rank` of `nranks`; afterwards sketch_train all-reduces the Gram of the local shard."""
        if len(uid) != 128:
            raise ValueError("uid must be the 128 bytes of get_unique_id()")
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        _check(lib().tsk_comm_init(self.handle, int(nranks), int(rank), buf), "tsk_comm_init")

    @property
    def launches(self) -> int:
        return int(lib().tsk_launch_count(self.handle))

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().tsk_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def get_unique_id() -> bytes:
    """128-byte NCCL unique id for tsk_comm_init (NCCL loaded at run time; TSK_ENCCL if unavailable)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().tsk_get_unique_id(buf), "tsk_get_unique_id")
    return buf.raw


_ctx_cache: dict = {}
_ctx_lock = threading.Lock()


def context(device=None) -> Context:
    """The default context of (device, current torch stream, calling thread): a ctx owns workspaces that
    its queued work uses, so two threads or two streams never share one (include/tsketch.h: one ctx per
    thread / stream)."""
    if device is None:
        device = torch.cuda.current_device()
    dev = torch.device("cuda", device).index if isinstance(device, int) else torch.device(device).index
    stream = torch.cuda.current_stream(dev).cuda_stream
    key = (dev, stream, threading.get_ident())
    with _ctx_lock:
        ctx = _ctx_cache.get(key)
        if ctx is None:
            ctx = _ctx_cache[key] = Context(dev)
    ctx._bind_stream()
    return ctx


def allreduce_gram(G64: torch.Tensor, ctx: Optional[Context] = None) -> torch.Tensor:
    """tsk_allreduce_gram: sum G64 [m, m] (cuda fp64) in place over the library's NCCL communicator."""
    _need(G64, torch.float64, "G64", 2)
    ctx = ctx or context(G64.device)
    _check(lib().tsk_allreduce_gram(ctx.handle, _ptr(G64), G64.shape[0]), "tsk_allreduce_gram")
    return G64


def allgather_errors(err_local: torch.Tensor, B_total: int, ctx: Optional[Context] = None) -> torch.Tensor:
    """tsk_allgather_errors: the per-matrix errors of all ranks' contiguous test shards, in stream order,
    on every rank (the library's NCCL communicator from tsk_comm_init; a copy without one)."""
    _need(err_local, torch.float64, "err_local", 1)
    ctx = ctx or context(err_local.device)
    out = torch.empty((int(B_total),), dtype=torch.float64, device=err_local.device)
    _check(lib().tsk_allgather_errors(ctx.handle, _ptr(err_local), int(B_total), _ptr(out)), "tsk_allgather_errors")
    return out


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _need(t: torch.Tensor, dtype, name: str, ndim: int):
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or t.dim() != ndim or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor with {ndim} dims")


def _alloc(shape, dtype, like: torch.Tensor):
    if like.is_cuda:
        return torch.empty(shape, dtype=dtype, device=like.device)
    return torch.empty(shape, dtype=dtype, pin_memory=True)


def _opts(opts) -> Optional[TrainOpts]:
    if opts is None:
        return None
    if isinstance(opts, TrainOpts):
        return opts
    o = TrainOpts()
    for k, v in dict(opts).items():
        if isinstance(v, torch.Tensor):  # device array fields (init_S): pass the pointer
            if not v.is_cuda or v.dtype != torch.float32 or not v.is_contiguous():
                raise ValueError(f"{k}: expected a contiguous float32 CUDA tensor")
            v = v.data_ptr()
        setattr(o, k, v)
    return o


def _optref(o):
    return ctypes.byref(o) if o is not None else None


# ------------------------------------------------------------------------------------ C-ABI names
def sketch_gram(A: torch.Tensor, G64: Optional[torch.Tensor] = None, G32: Optional[torch.Tensor] = None,
                accumulate: bool = False, opts=None, ctx: Optional[Context] = None):
    """G64 (+)= sum_d A_d A_d^T for A [D, m, n] fp32.  Returns (G64, info)."""
    _need(A, torch.float32, "A", 3)
    D, m, n = A.shape
    ctx = ctx or context(A.device if A.is_cuda else None)
    if G64 is None:
        if accumulate:
            raise ValueError("accumulate requires G64")
        G64 = _alloc((m, m), torch.float64, A)
    _need(G64, torch.float64, "G64", 2)
    info = TrainInfo()
    o = _opts(opts)
    _check(lib().sketch_gram(ctx.handle, _ptr(A), D, m, n, _ptr(G64), _ptr(G32), int(bool(accumulate)), _optref(o),
                             ctypes.byref(info)), "sketch_gram")
    return G64, info


def sketch_topk(G64: torch.Tensor, k: int, opts=None, ctx: Optional[Context] = None):
    """Top-k eigenvectors of G as rows of S [k, m] fp32 and Ritz values lambda [k] fp64."""
    _need(G64, torch.float64, "G64", 2)
    m = G64.shape[0]
    ctx = ctx or context(G64.device if G64.is_cuda else None)
    S = _alloc((k, m), torch.float32, G64)
    lam = _alloc((k,), torch.float64, G64)
    info = TrainInfo()
    o = _opts(opts)
    st = _check(lib().sketch_topk(ctx.handle, _ptr(G64), m, k, _ptr(S), _ptr(lam), _optref(o), ctypes.byref(info)),
                "sketch_topk")
    return S, lam, info, st


def sketch_train(A: torch.Tensor, k: int, opts=None, G64_out: Optional[torch.Tensor] = None,
                 ctx: Optional[Context] = None):
    """Algorithm 2 lines 1-2 on one GPU.  Returns (S, lambda, info, status)."""
    _need(A, torch.float32, "A", 3)
    D, m, n = A.shape
    ctx = ctx or context(A.device if A.is_cuda else None)
    S = _alloc((k, m), torch.float32, A)
    lam = _alloc((k,), torch.float64, A)
    info = TrainInfo()
    o = _opts(opts)
    st = _check(lib().sketch_train(ctx.handle, _ptr(A), D, m, n, k, _ptr(S), _ptr(lam), _ptr(G64_out), _optref(o),
                                   ctypes.byref(info)), "sketch_train")
    return S, lam, info, st


def sketch_apply_scw(A: torch.Tensor, S: torch.Tensor, r: int, want=("L", "R", "sigma"),
                     ctx: Optional[Context] = None):
    """SCW (Algorithm 1) on a batch A [B, m, n]: A_hat_b = L_b R_b^T."""
    _need(A, torch.float32, "A", 3)
    _need(S, torch.float32, "S", 2)
    B, m, n = A.shape
    k = S.shape[0]
    rr = min(r, k)
    ctx = ctx or context(A.device if A.is_cuda else None)
    L = _alloc((B, m, rr), torch.float32, A) if "L" in want else None
    R = _alloc((B, n, rr), torch.float32, A) if "R" in want else None
    sig = _alloc((B, rr), torch.float32, A) if "sigma" in want else None
    _check(lib().sketch_apply_scw(ctx.handle, _ptr(A), B, m, n, _ptr(S), k, r, _ptr(L), _ptr(R), _ptr(sig)),
           "sketch_apply_scw")
    return L, R, sig


def scw_error(A: torch.Tensor, S: torch.Tensor, r: int, out: Optional[torch.Tensor] = None,
              ctx: Optional[Context] = None) -> torch.Tensor:
    """err[b] = ||A_b - SCW(A_b, S, r)||_F (fp64; formula per set_scw_error_mode, include/tsketch.h)."""
    _need(A, torch.float32, "A", 3)
    _need(S, torch.float32, "S", 2)
    B, m, n = A.shape
    k = S.shape[0]
    ctx = ctx or context(A.device if A.is_cuda else None)
    err = out if out is not None else _alloc((B,), torch.float64, A)
    _check(lib().scw_error(ctx.handle, _ptr(A), B, m, n, _ptr(S), k, r, _ptr(err)), "scw_error")
    return err


def set_scw_error_mode(mode: int, tau: float = 0.0, ctx: Optional[Context] = None) -> None:
    """scw_error's formula on `ctx` (tsk_set_scw_error_mode): 0 = Pythagorean identity with the dense
    residual below tau ||A||^2 (tau <= 0: library default), 1 = dense residual for every matrix."""
    ctx = ctx or context()
    _check(lib().tsk_set_scw_error_mode(ctx.handle, int(mode), float(tau)), "tsk_set_scw_error_mode")


def tsk_gram_probe(A: torch.Tensor, mode: int = 0, chain: int = 0, splits: int = 0, G64=None,
                   ctx: Optional[Context] = None) -> torch.Tensor:
    """Diagnostic Gram launch (see include/tsketch.h): mode bit0 = raw tiles, bit1 = H*H only."""
    _need(A, torch.float32, "A", 3)
    D, m, n = A.shape
    ctx = ctx or context(A.device)
    G64 = G64 if G64 is not None else torch.empty((m, m), dtype=torch.float64, device=A.device)
    _check(lib().tsk_gram_probe(ctx.handle, _ptr(A), D, m, n, _ptr(G64), mode, chain, splits), "tsk_gram_probe")
    return G64


def tsk_eig_probe(H: torch.Tensor, ctx: Optional[Context] = None):
    """Diagnostic: batched symmetric eigensolver (include/tsketch.h).  H [B, p, p] fp64 cuda.
    Returns (W [B, p, p] eigenvectors as columns, lam [B, p] decreasing, sweeps [B])."""
    _need(H, torch.float64, "H", 3)
    B, p, _ = H.shape
    ctx = ctx or context(H.device)
    W = torch.empty_like(H)
    lam = torch.empty((B, p), dtype=torch.float64, device=H.device)
    sw = torch.empty((B,), dtype=torch.int32, device=H.device)
    _check(lib().tsk_eig_probe(ctx.handle, _ptr(H), p, B, _ptr(W), _ptr(lam), _ptr(sw)), "tsk_eig_probe")
    return W, lam, sw


def tsk_syev_probe(H: torch.Tensor, nw: Optional[int] = None, orth_tol: float = 1e-9,
                   ctx: Optional[Context] = None):
    """Diagnostic: the Rayleigh-Ritz eigensolver (include/tsketch.h).  H [p, p] fp64 cuda.
    Returns (W [p, nw] eigenvectors as columns, lam [nw] decreasing, flag (int32 tensor, 1 = unresolved
    cluster))."""
    _need(H, torch.float64, "H", 2)
    p = H.shape[0]
    nw = p if nw is None else nw
    ctx = ctx or context(H.device)
    W = torch.empty((p, nw), dtype=torch.float64, device=H.device)
    lam = torch.empty((nw,), dtype=torch.float64, device=H.device)
    flag = torch.zeros((1,), dtype=torch.int32, device=H.device)
    _check(lib().tsk_syev_probe(ctx.handle, _ptr(H), p, nw, _ptr(W), _ptr(lam), _ptr(flag), orth_tol),
           "tsk_syev_probe")
    return W, lam, flag


# ---------------------------------------------------------------------------- two-sided variant
def sketch_gram_mode2(A: torch.Tensor, G64: Optional[torch.Tensor] = None, accumulate: bool = False,
                      ctx: Optional[Context] = None) -> torch.Tensor:
    """G2 (+)= sum_d A_d^T A_d (n x n fp64), the mode-2 Gram (HOSVD init of Algorithm 5)."""
    _need(A, torch.float32, "A", 3)
    D, m, n = A.shape
    ctx = ctx or context(A.device if A.is_cuda else None)
    G64 = G64 if G64 is not None else _alloc((n, n), torch.float64, A)
    _check(lib().sketch_gram_mode2(ctx.handle, _ptr(A), D, m, n, _ptr(G64), int(accumulate)), "sketch_gram_mode2")
    return G64


def sketch_train_two_sided(A: torch.Tensor, k: int, l: int, max_sweeps: int = 0, rel_tol: float = 0.0,
                           ctx: Optional[Context] = None):
    """Tucker2 by HOOI over modes 1-2 (Eq. (9), Algorithm 5): returns (S [k][m], W [l][n], info dict, status)."""
    _need(A, torch.float32, "A", 3)
    D, m, n = A.shape
    ctx = ctx or context(A.device if A.is_cuda else None)
    S = _alloc((k, m), torch.float32, A)
    W = _alloc((l, n), torch.float32, A)
    o = HooiOpts(max_sweeps, rel_tol)
    info = HooiInfo()
    st = _check(lib().sketch_train_two_sided(ctx.handle, _ptr(A), D, m, n, k, l, _ptr(S), _ptr(W), ctypes.byref(o),
                                             ctypes.byref(info)), "sketch_train_two_sided")
    return S, W, info.as_dict(), st


def sketch_apply_two_sided_scw(A: torch.Tensor, S: torch.Tensor, W: torch.Tensor, r: int,
                               ctx: Optional[Context] = None):
    """Algorithm 3: A_hat_b = L_b R_b^T; returns (L [B][m][r], R [B][n][r], sigma [B][r])."""
    _need(A, torch.float32, "A", 3)
    _need(S, torch.float32, "S", 2)
    _need(W, torch.float32, "W", 2)
    B, m, n = A.shape
    k, l = S.shape[0], W.shape[0]
    rr = min(r, k, l)
    ctx = ctx or context(A.device if A.is_cuda else None)
    L = _alloc((B, m, rr), torch.float32, A)
    R = _alloc((B, n, rr), torch.float32, A)
    sig = _alloc((B, rr), torch.float32, A)
    _check(lib().sketch_apply_two_sided_scw(ctx.handle, _ptr(A), B, m, n, _ptr(S), k, _ptr(W), l, r, _ptr(L),
                                            _ptr(R), _ptr(sig)), "sketch_apply_two_sided_scw")
    return L, R, sig


def two_sided_scw_error(A: torch.Tensor, S: torch.Tensor, W: torch.Tensor, r: int,
                        ctx: Optional[Context] = None) -> torch.Tensor:
    """err[b] = ||A_b - two-sided SCW(A_b, S, W, r)||_F (fp64, dense residual)."""
    _need(A, torch.float32, "A", 3)
    _need(S, torch.float32, "S", 2)
    _need(W, torch.float32, "W", 2)
    B, m, n = A.shape
    ctx = ctx or context(A.device if A.is_cuda else None)
    err = _alloc((B,), torch.float64, A)
    _check(lib().two_sided_scw_error(ctx.handle, _ptr(A), B, m, n, _ptr(S), S.shape[0], _ptr(W), W.shape[0], r,
                                     _ptr(err)), "two_sided_scw_error")
    return err


def sketch_train_matrix_free(A: torch.Tensor, k: int, oversample: int = 0, power_iters: int = -1,
                             subspace: bool = False, omega: Optional[torch.Tensor] = None,
                             ctx: Optional[Context] = None):
    """Matrix-free Tucker1 sketch by randomized block Krylov: returns (S [k][m],
    lambda [k] fp64 Ritz values, info dict, status).  omega: optional [m][p] fp64 start block with
    p = k + oversample rounded up to a multiple of 4 (capped at m)."""
    _need(A, torch.float32, "A", 3)
    D, m, n = A.shape
    ctx = ctx or context(A.device if A.is_cuda else None)
    S = _alloc((k, m), torch.float32, A)
    lam = _alloc((k,), torch.float64, A)
    if omega is not None:
        _need(omega, torch.float64, "omega", 2)
    o = MfOpts(oversample, power_iters, int(bool(subspace)), _ptr(omega))
    info = MfInfo()
    st = _check(lib().sketch_train_matrix_free(ctx.handle, _ptr(A), D, m, n, k, _ptr(S), _ptr(lam), ctypes.byref(o),
                                               ctypes.byref(info)), "sketch_train_matrix_free")
    return S, lam, info.as_dict(), st


from .dist import shard_range, train  # noqa: E402,F401
