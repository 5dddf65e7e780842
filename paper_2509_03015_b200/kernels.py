"""The reference's dense kernel layer on the GPU (drop-in for `blocktri.kernels`,
/root/reference/pkg/src/blocktri/kernels.py).

Same functions, argument meaning, in-place semantics and errors: ``chol_factor_batch`` /
``chol_factor``, ``trsm_lower_batch`` / ``trsm_lower``, ``gemm_acc_batch`` / ``gemm_acc``,
``batched`` + ``KernelBatchView``, ``max_batch_threads`` / ``set_batch_threads``.  The work runs in
the sm_100a seam kernels of ``libblocktri_b200.so`` (csrc/btd_seam.cuh) through the C ABI
(``btd_chol_batch`` / ``btd_trsm_batch`` / ``btd_gemm_batch``):

* torch CUDA tensors are worked on in place, with their own strides (transposed views included,
  as block_cholesky.py:32 passes them);
* numpy arrays / CPU tensors are copied to the device, worked on, and written back in place.

The thread cap of the reference (``BLOCKTRI_THREADS``) is kept as an API knob; a batch is one launch
over all members, so the cap never changes results (the reference guarantees the same,
kernels.py:11-14).  There is no CPU fallback: the native library is required.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DimensionMismatch, NotPositiveDefinite, SingularDiagonal

_batch_threads: int | None = None

#: gemm_acc_batch members per launch (grid.y limit)
_GEMM_MAX_MEMBERS = 65535


def max_batch_threads() -> int:
    """Current cap on threads used to chunk batched kernels (kernels.py:43-54)."""
    if _batch_threads is not None:
        return _batch_threads
    env = os.environ.get("BLOCKTRI_THREADS", "").strip()
    if env:
        try:
            return max(1, int(env))
        except ValueError:
            pass
    return min(8, os.cpu_count() or 1)


def set_batch_threads(count: int | None) -> None:
    """Override the thread cap (None restores the environment default) (kernels.py:57-59)."""
    global _batch_threads
    _batch_threads = None if count is None else max(1, int(count))


@dataclass(frozen=True)
class KernelBatchView:
    """K same-shaped dense panels backed by one shared arena (kernels.py:104-133)."""

    arena: object  # (K, rows, cols) numpy array or torch tensor

    def __post_init__(self):
        if self.arena.ndim != 3:
            raise DimensionMismatch(f"batch view needs a (K, rows, cols) array, got {tuple(self.arena.shape)}")
        if self.arena.shape[0] > 1:
            span = self.arena.shape[1] * self.arena.shape[2]
            if abs(_strides(self.arena)[0]) < span:
                raise ValueError("batch members overlap in memory")

    @property
    def count(self) -> int:
        return self.arena.shape[0]

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self.arena.shape[1:])

    def member(self, k: int):
        return self.arena[k]


# ------------------------------------------------------------------------------------------
# device staging of the operands
# ------------------------------------------------------------------------------------------
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _strides(x) -> tuple:
    """Element strides of a numpy array or torch tensor."""
    if _is_torch(x):
        return tuple(x.stride())
    return tuple(s // x.itemsize for s in x.strides)


class _Dev:
    """A device view of one operand; ``done()`` writes an in-place result back to a host operand."""

    def __init__(self, x, writable: bool):
        import torch
        self.host, self.writable = x, writable
        if _is_torch(x) and x.is_cuda:
            if x.dtype != torch.float64:
                raise TypeError("seam kernels need float64 tensors")
            self.t = x
            self.host = None
            return
        if _is_torch(x):
            src = x
        else:
            a = np.asarray(x)
            if any(s < 0 or s % a.itemsize for s in a.strides):
                a = np.ascontiguousarray(a)
            src = torch.from_numpy(a)
        self.t = src.to(device="cuda", dtype=torch.float64)

    @property
    def ptr(self):
        return self.t.data_ptr()

    def strides(self):
        s = self.t.stride()
        return (ctypes.c_int64 * 3)(*s)

    def done(self):
        if self.host is None or not self.writable:
            return
        import torch
        if _is_torch(self.host):
            self.host.copy_(self.t)
        elif isinstance(self.host, np.ndarray) and all(s >= 0 and s % self.host.itemsize == 0
                                                       for s in self.host.strides):
            torch.from_numpy(self.host).copy_(self.t)
        else:
            np.copyto(self.host, self.t.cpu().numpy())


class _ErrWord:
    """Device error word of one seam call sequence (btd_seam_error_*)."""

    def __init__(self):
        import torch
        L = _native.lib()
        self.buf = torch.empty(int(L.btd_seam_error_bytes()), dtype=torch.uint8, device="cuda")
        self.stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _check(L.btd_seam_error_init(self.buf.data_ptr(), self.stream), None)

    def read(self) -> tuple[int, _native.BtdStatus]:
        st = _native.BtdStatus()
        rc = _native.lib().btd_seam_error_read(self.buf.data_ptr(), self.stream, ctypes.byref(st))
        return rc, st


def _check(rc: int, st) -> None:
    if rc == _native.BTD_OK:
        return
    msg = st.message.decode(errors="replace") if st is not None else f"status {rc}"
    if rc in (_native.BTD_ERR_INVALID_ARGUMENT,):
        raise ValueError(msg)
    from .errors import DeviceError
    raise DeviceError(msg)


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check_batch(arr, square: bool = False) -> None:
    if arr.ndim != 3:
        raise DimensionMismatch(f"expected (K, rows, cols) batch, got shape {tuple(arr.shape)}")
    if square and arr.shape[1] != arr.shape[2]:
        raise DimensionMismatch(f"expected square members, got shape {tuple(arr.shape)}")


# device-level primitives (operands already staged), shared with block_cholesky
def _chol_dev(d: _Dev, count: int, n: int, err: _ErrWord, block: int = 0) -> None:
    st = _native.BtdStatus()
    _check(_native.lib().btd_chol_batch(d.ptr, d.strides(), count, n, block, err.buf.data_ptr(), _stream(),
                                        ctypes.byref(st)), st)


def _trsm_dev(f: _Dev, p: _Dev, count: int, n: int, cols: int, trans: bool, err: _ErrWord) -> None:
    st = _native.BtdStatus()
    _check(_native.lib().btd_trsm_batch(f.ptr, f.strides(), p.ptr, p.strides(), count, n, cols, 1 if trans else 0,
                                        err.buf.data_ptr(), _stream(), ctypes.byref(st)), st)


def _gemm_dev(o: _Dev, a: _Dev, b: _Dev, count: int, m: int, q: int, p: int, ta: bool, tb: bool, alpha: float,
              beta: float) -> None:
    L = _native.lib()
    for k0 in range(0, count, _GEMM_MAX_MEMBERS):
        k1 = min(count, k0 + _GEMM_MAX_MEMBERS)
        views = [_sub(x, k0, k1) for x in (o, a, b)]
        st = _native.BtdStatus()
        _check(L.btd_gemm_batch(views[0].ptr, views[0].strides(), views[1].ptr, views[1].strides(), views[2].ptr,
                                views[2].strides(), k1 - k0, m, q, p, 1 if ta else 0, 1 if tb else 0,
                                float(alpha), float(beta), _stream(), ctypes.byref(st)), st)


def _sub_view(d: _Dev, fn) -> _Dev:
    """A device view ``fn(d.t)`` of a staged operand (no copy; the parent writes back)."""
    v = object.__new__(_Dev)
    v.host, v.writable, v.t = None, False, fn(d.t)
    return v


def _sub(d: _Dev, k0: int, k1: int) -> _Dev:
    if k0 == 0 and k1 == d.t.shape[0]:
        return d
    return _sub_view(d, lambda t: t[k0:k1])


def _raise_err(err: _ErrWord, *, with_block: bool = False) -> None:
    rc, st = err.read()
    if rc == _native.BTD_OK:
        return
    if rc == _native.BTD_ERR_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefinite(int(st.pivot), member=int(st.member),
                                  block=int(st.block) if with_block else None)
    if rc == _native.BTD_ERR_SINGULAR_DIAGONAL:
        raise SingularDiagonal(int(st.pivot), member=int(st.member))
    _check(rc, st)


# ------------------------------------------------------------------------------------------
# the reference API
# ------------------------------------------------------------------------------------------
def chol_factor_batch(blocks) -> None:
    """Factor each symmetric member in place as L with member = L L^T (kernels.py:164-181).

    The strict upper triangle of every member is zeroed.  Raises NotPositiveDefinite(pivot,
    member=...) for the lowest failing member; the batch contents are then unspecified.
    """
    _check_batch(blocks, square=True)
    if blocks.shape[0] == 0:
        return
    d = _Dev(blocks, True)
    err = _ErrWord()
    _chol_dev(d, blocks.shape[0], blocks.shape[1], err)
    try:
        _raise_err(err)
    finally:
        d.done()


def chol_factor(block) -> None:
    """In-place lower Cholesky factor of one symmetric block (kernels.py:184-189)."""
    try:
        chol_factor_batch(block[None])
    except NotPositiveDefinite as err:
        raise NotPositiveDefinite(err.pivot) from None


def trsm_lower_batch(factors, panels, trans: bool = False) -> None:
    """Solve each member's triangular system in place on ``panels`` (kernels.py:215-259).

    ``trans=False`` overwrites panel k with L_k^{-1} B_k, ``trans=True`` with L_k^{-T} B_k, where L_k
    is the lower triangle of ``factors[k]``.  An exactly zero diagonal raises SingularDiagonal(row,
    member) before any panel is modified.
    """
    _check_batch(factors, square=True)
    _check_batch(panels)
    if panels.shape[0] != factors.shape[0] or panels.shape[1] != factors.shape[1]:
        raise DimensionMismatch(
            f"panel batch {tuple(panels.shape)} not conformal with factors {tuple(factors.shape)}")
    if factors.shape[0] == 0:
        return
    f = _Dev(factors, False)
    p = _Dev(panels, True)
    err = _ErrWord()
    _trsm_dev(f, p, factors.shape[0], factors.shape[1], panels.shape[2], trans, err)
    try:
        _raise_err(err)
    finally:
        p.done()


def trsm_lower(factor, panel, trans: bool = False) -> None:
    """Single-block triangular solve, in place on ``panel`` (kernels.py:262-267)."""
    try:
        trsm_lower_batch(factor[None], panel[None], trans=trans)
    except SingularDiagonal as err:
        raise SingularDiagonal(err.row) from None


def gemm_acc_batch(out, a, b, trans_a: bool = False, trans_b: bool = False, alpha: float = 1.0,
                   beta: float = 0.0) -> None:
    """Accumulate ``out <- alpha * op(a) @ op(b) + beta * out`` per member (kernels.py:270-310).

    ``out`` must not alias ``a`` or ``b``.  alpha == 0 skips the product; beta == 0 ignores the
    previous contents of ``out``.
    """
    _check_batch(out)
    _check_batch(a)
    _check_batch(b)
    k = out.shape[0]
    am, aq = (a.shape[2], a.shape[1]) if trans_a else (a.shape[1], a.shape[2])
    bq, bp = (b.shape[2], b.shape[1]) if trans_b else (b.shape[1], b.shape[2])
    if a.shape[0] != k or b.shape[0] != k:
        raise DimensionMismatch("batch counts disagree")
    if bq != aq or out.shape[1] != am or out.shape[2] != bp:
        raise DimensionMismatch(
            f"gemm shapes do not conform: ({k}, {am}, {aq}) @ ({k}, {bq}, {bp}) -> {tuple(out.shape)}")
    if k == 0:
        return
    o = _Dev(out, True)
    _gemm_dev(o, _Dev(a, False), _Dev(b, False), k, am, aq, bp, trans_a, trans_b, alpha, beta)
    o.done()


def gemm_acc(out, a, b, trans_a: bool = False, trans_b: bool = False, alpha: float = 1.0,
             beta: float = 0.0) -> None:
    """Single-block multiply-accumulate, in place on ``out`` (kernels.py:313-318)."""
    gemm_acc_batch(out[None], a[None], b[None], trans_a=trans_a, trans_b=trans_b, alpha=alpha, beta=beta)


def batched(op, *views, **kwargs) -> None:
    """Apply a single-block kernel across every member of the given batches (kernels.py:321-338)."""
    arrays = [v.arena if isinstance(v, KernelBatchView) else (v if _is_torch(v) else np.asarray(v))
              for v in views]
    table = {chol_factor: chol_factor_batch, trsm_lower: trsm_lower_batch, gemm_acc: gemm_acc_batch}
    try:
        impl = table[op]
    except KeyError:
        raise ValueError(f"not a batchable kernel: {op!r}") from None
    impl(*arrays, **kwargs)
