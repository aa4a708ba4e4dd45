"""Device plumbing: the krb context, streams, device sparse matrices, and the
host<->device moves of the drop-in API.  PyTorch supplies device memory and
the current CUDA stream; every computation is a libkrb.so kernel."""

from __future__ import annotations

import ctypes
import weakref
from collections import OrderedDict

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


_CUDA_OK = False


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


@_ALLOC_FN
def _torch_alloc(nbytes, stream):
    try:
        return torch()._C._cuda_cudaCachingAllocator_raw_alloc(int(nbytes), int(stream or 0))
    except Exception:      # out of memory -> NULL -> KRB_ENOMEM
        return None


@_FREE_FN
def _torch_free(p, stream):
    try:
        torch()._C._cuda_cudaCachingAllocator_raw_delete(int(p))
    except Exception:      # interpreter shutdown: torch already torn down
        pass


def require_cuda():
    """Raise KrbError without a CUDA device (no CPU fallback).  The positive
    answer is cached: torch.cuda.is_available() re-queries NVML / the
    environment on every call (~0.1 ms), and this runs once per entry point.
    The first call also makes libkrb allocate its matrices from torch's
    caching allocator (krb_set_allocator), so the library and torch share
    one device pool instead of two that cannot lend each other memory."""
    global _CUDA_OK
    if _CUDA_OK:
        return
    t = torch()
    if not t.cuda.is_available():
        raise _lib.KrbError("no CUDA device: the B200 path has no CPU fallback")
    lib = _lib.load()
    rc = lib.krb_set_allocator(ctypes.cast(_torch_alloc, ctypes.c_void_p),
                               ctypes.cast(_torch_free, ctypes.c_void_p))
    _lib.check(rc, "krb_set_allocator")
    _CUDA_OK = True


def stream_ptr():
    """The current CUDA stream of the current device (raw handle; the direct
    torch._C queries avoid ~20 us of Python per call)."""
    C = torch()._C
    return ctypes.c_void_p(C._cuda_getCurrentRawStream(C._cuda_getDevice()))


# Deferred device launches: a producer (rbicg_solve's next harvest cycle)
# registers its launch before handing a cycle to the cycle_callback; a
# consumer about to run long host-only work (update_recycle_space's
# eigenproblem) calls flush_pending() so the launch overlaps that host work.
# The producer flushes again after the callback returns (a no-op if done).
_PENDING = []


def defer_launch(fn):
    _PENDING.append(fn)


def flush_pending():
    while _PENDING:
        _PENDING.pop(0)()


def drop_pending():
    _PENDING.clear()


def ptr(tensor):
    return ctypes.c_void_p(tensor.data_ptr()) if tensor is not None else None


class Context:
    """One krb_context per process (scratch + graph cache)."""

    _inst = None

    def __init__(self):
        require_cuda()
        h = ctypes.c_void_p()
        _lib.call("krb_context_create", ctypes.byref(h))
        self.h = h
        self._hist = None

    @classmethod
    def get(cls) -> "Context":
        if cls._inst is None:
            cls._inst = Context()
        return cls._inst

    def history_buffers(self, max_itn: int):
        """Device history arrays reused across solves (so the cached CUDA
        graph, which bakes their addresses, stays valid)."""
        need = int(max_itn) + 2
        if self._hist is None or self._hist[0].shape[0] < need:
            t = torch()
            cap = max(need, 1024)
            self._hist = (t.empty(cap, dtype=t.float64, device="cuda"),
                          t.empty(cap, dtype=t.int64, device="cuda"),
                          t.empty(cap, dtype=t.int64, device="cuda"))
        return self._hist


class _Staging:
    """Two reusable pinned host buffers for H2D copies: the host memcpy into
    one overlaps the DMA out of the other; an event guards reuse."""

    def __init__(self):
        self.bufs = [None, None]
        self.events = [None, None]
        self.turn = 0

    def get(self, nbytes):
        t = torch()
        i = self.turn
        self.turn ^= 1
        if self.events[i] is not None:
            self.events[i].synchronize()
        buf = self.bufs[i]
        if buf is None or buf.numel() < nbytes:
            # both buffers at once (a page-locked allocation costs milliseconds:
            # pay it once, not again on the first use of the other buffer)
            cap = max(nbytes, 1 << 24)
            for j in (0, 1):
                if self.events[j] is not None:
                    self.events[j].synchronize()
                if self.bufs[j] is None or self.bufs[j].numel() < cap:
                    self.bufs[j] = t.empty(cap, dtype=t.uint8, pin_memory=True)
            buf = self.bufs[i]
        return i, buf

    def mark(self, i):
        t = torch()
        ev = self.events[i] or t.cuda.Event()
        ev.record()
        self.events[i] = ev


_STAGING = _Staging()
_POOL = None
_PAR_BYTES = 1 << 20     # host copies above this size are split across threads
_CHUNK = 32 << 20        # H2D pipeline chunk (two pinned buffers alternate)


def _host_copy(dst: np.ndarray, src: np.ndarray):
    """dst[:] = src (flat uint8 views), split across threads for large
    arrays: numpy releases the GIL inside the copy loop, so the memcpy into
    pinned staging runs at several times single-thread bandwidth."""
    global _POOL
    n = src.nbytes
    if n < _PAR_BYTES:
        np.copyto(dst, src)
        return
    if _POOL is None:
        import concurrent.futures as cf
        import os
        _POOL = cf.ThreadPoolExecutor(max_workers=max(2, min(8, (os.cpu_count() or 2))))
    parts = _POOL._max_workers
    step = -(-n // parts)
    step = (step + 4095) & ~4095
    futs = [_POOL.submit(np.copyto, dst[o:o + step], src[o:o + step])
            for o in range(0, n, step)]
    for f in futs:
        f.result()
_TDT = {np.dtype(np.float64): "float64", np.dtype(np.int64): "int64",
        np.dtype(np.int32): "int32"}


def to_device(a: np.ndarray, dtype=np.float64, staging=None):
    """Host numpy -> device tensor through reusable pinned staging, in
    chunks: the (multi-threaded) host copy of chunk i+1 into one pinned
    buffer overlaps the DMA of chunk i out of the other.  ``staging``: a
    private _Staging (a background uploader must not share the caller's)."""
    t = torch()
    stg = _STAGING if staging is None else staging
    a = np.asarray(a)
    dtype = np.dtype(dtype)
    if (a.dtype != dtype and a.dtype.kind in "iu" and dtype.kind in "iu"
            and a.ndim == 1 and a.nbytes >= (1 << 16) and not _is_pinned(a)):
        return _to_device_cast(a, dtype, stg)
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.nbytes < (1 << 16):
        # small operands (Ritz coefficients, column scales): a pinned copy
        # from torch's caching host allocator makes the upload asynchronous
        # (a pageable copy would stall the host until the GPU queue drains)
        return t.from_numpy(a).pin_memory().to("cuda", non_blocking=True)
    ht = t.from_numpy(a)
    if ht.is_pinned():
        # caller-owned page-locked memory: one DMA, no staging copy
        return ht.to("cuda", non_blocking=True)
    out = t.empty(a.shape, dtype=getattr(t, _TDT[a.dtype]), device="cuda")
    src = a.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(t.uint8)
    n = a.nbytes
    for o in range(0, n, _CHUNK):
        m = min(_CHUNK, n - o)
        i, buf = stg.get(m)               # waits for this buffer's previous DMA
        _host_copy(buf[:m].numpy(), src[o:o + m])
        dst[o:o + m].copy_(buf[:m], non_blocking=True)
        stg.mark(i)
    return out


def _to_device_cast(a: np.ndarray, dtype, stg):
    """Integer upload narrowed (or widened) during the staging copy itself:
    each chunk is cast straight into the pinned buffer, so an int64 index
    array goes over the link as int32 without a full host-side converted
    copy first."""
    t = torch()
    out = t.empty(a.shape, dtype=getattr(t, _TDT[dtype]), device="cuda")
    per = _CHUNK // dtype.itemsize
    n = a.shape[0]
    for o in range(0, n, per):
        m = min(per, n - o)
        i, buf = stg.get(m * dtype.itemsize)
        dst = buf[:m * dtype.itemsize].numpy().view(dtype)
        _host_copy_cast(dst, a[o:o + m])
        out[o:o + m].copy_(buf[:m * dtype.itemsize].view(out.dtype), non_blocking=True)
        stg.mark(i)
    return out


def _host_copy_cast(dst: np.ndarray, src: np.ndarray):
    """dst[:] = src with an element-type cast, split across the copy pool."""
    global _POOL
    n = src.shape[0]
    if n * src.itemsize < _PAR_BYTES:
        np.copyto(dst, src, casting="unsafe")
        return
    if _POOL is None:
        import concurrent.futures as cf
        import os
        _POOL = cf.ThreadPoolExecutor(max_workers=max(2, min(8, (os.cpu_count() or 2))))
    parts = _POOL._max_workers
    step = -(-n // parts)
    futs = [_POOL.submit(np.copyto, dst[o:o + step], src[o:o + step], casting="unsafe")
            for o in range(0, n, step)]
    for f in futs:
        f.result()


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """A page-locked host copy of ``a`` (numpy view of a pinned torch
    buffer): inputs kept in pinned memory upload by DMA alone."""
    t = torch()
    a = np.ascontiguousarray(a)
    buf = t.empty(max(a.nbytes, 1), dtype=t.uint8, pin_memory=True)
    out = buf.numpy()[:a.nbytes].view(a.dtype).reshape(a.shape)
    out[...] = a
    return out


def to_host(tensor) -> np.ndarray:
    """Device tensor -> host numpy through a page-locked buffer from torch's
    caching host allocator: the device->host copy is plain DMA (a copy into
    pageable memory is staged by the driver at a fraction of the link rate).
    The returned array keeps the pinned buffer alive; freeing it returns the
    buffer to the cache."""
    t = torch()
    src = tensor.detach()
    if not src.is_cuda:
        return src.numpy()
    out = t.empty(src.shape, dtype=src.dtype, pin_memory=True)
    out.copy_(src)   # synchronous: the data is on the host on return
    return out.numpy()


def _ci_dtype(col_idx, n):
    """Column indices travel as int32 whenever they fit (n < 2^31: the
    library stores int32 indices anyway), halving a pageable int64 array's
    upload (cast inside the staging copy); page-locked int64 goes by DMA."""
    if col_idx.dtype == np.int32:
        return np.int32
    if _is_pinned(col_idx) or n >= (1 << 31):
        return np.int64
    return np.int32


def _is_pinned(a) -> bool:
    try:
        return torch().from_numpy(np.ascontiguousarray(a)).is_pinned()
    except Exception:
        return False


# Device copies of FROZEN host index arrays (not writeable: SparseMatrix
# freezes its arrays as the reference does, sparse.py:66-67), keyed on the
# array objects: the matrices of a sequence A_j = s_j E - K share one
# row_ptr / col_idx pair, which then crosses the link once instead of once
# per matrix (C5: 1.9 of the 5.5 GB of every upload).  One pair at a time;
# dropped with the matrix cache.
_IDX_CACHE = {}


def _upload_indices(row_ptr, col_idx, n, staging=None):
    frozen = (isinstance(row_ptr, np.ndarray) and isinstance(col_idx, np.ndarray)
              and not row_ptr.flags.writeable and not col_idx.flags.writeable)
    key = (id(row_ptr), id(col_idx))
    t = torch()
    if frozen:
        hit = _IDX_CACHE.get(key)
        if hit is not None and hit[0] is row_ptr and hit[1] is col_idx:
            # (uploaded on whichever stream was current then -- the copy
            # stream for a prefetch: order this stream behind that upload)
            cur = t.cuda.current_stream()
            cur.wait_event(hit[4])
            for d in hit[2:4]:
                d.record_stream(cur)
            return hit[2], hit[3]
    d_rp = to_device(row_ptr, np.int64, staging=staging)
    d_ci = to_device(col_idx, _ci_dtype(col_idx, n), staging=staging)
    if frozen:
        ev = t.cuda.Event()
        ev.record()
        _IDX_CACHE.clear()
        _IDX_CACHE[key] = (row_ptr, col_idx, d_rp, d_ci, ev)
    return d_rp, d_ci


class _Prefetch:
    """Host->device copies of a matrix's CSR arrays issued ahead of use on a
    side copy stream (run_sequence prefetches matrix i+1 while system i
    solves: the DMA overlaps the kernels).  Page-locked inputs are pure DMA
    and are issued directly; pageable ones go through a background thread
    with its own pinned staging pair (its multi-threaded host copies release
    the GIL, and the solve waiting in libkrb holds none), so a caller handing
    in plain numpy arrays gets the same overlap."""

    def __init__(self):
        self.items = {}
        self.stream = None
        self.staging = None
        import threading
        self.lock = threading.Lock()

    def _upload(self, A, arrs, slot, dev=None):
        t = torch()
        try:
            if dev is not None:
                t.cuda.set_device(dev)   # a new thread starts on device 0
            with t.cuda.stream(self.stream):
                d_rp, d_ci = _upload_indices(arrs[0], arrs[1], len(arrs[0]) - 1,
                                             staging=self.staging)
                d_val = to_device(arrs[2], np.float64, staging=self.staging)
                ev = t.cuda.Event()
                ev.record(self.stream)
            slot["result"] = ((d_rp, d_ci, d_val), ev)
        except BaseException as e:   # reported at take(): the solve uploads itself
            slot["error"] = e

    def issue(self, A) -> bool:
        if getattr(A, "_device", None) is not None or not hasattr(A, "row_ptr"):
            return False
        if id(A) in self.items or MATRICES.items.get(id(A), (None,))[0] is A:
            return False
        arrs = (np.asarray(A.row_ptr), np.asarray(A.col_idx), np.asarray(A.values))
        if np.iscomplexobj(arrs[2]):
            return False
        t = torch()
        require_cuda()
        if self.stream is None:
            self.stream = t.cuda.Stream()
        slot = {}
        if all(_is_pinned(a) for a in arrs):
            self._upload(A, arrs, slot)
            self.items[id(A)] = (A, slot, None)
            return True
        import threading
        with self.lock:
            if self.staging is None:
                self.staging = _Staging()
            # one background upload at a time (the staging pair is shared)
            for _, _, th in self.items.values():
                if th is not None:
                    th.join()
            th = threading.Thread(target=self._upload,
                                  args=(A, arrs, slot, t.cuda.current_device()), daemon=True)
            th.start()
            self.items[id(A)] = (A, slot, th)
        return True

    def take(self, A):
        hit = self.items.pop(id(A), None)
        if hit is None or hit[0] is not A:
            return None
        if hit[2] is not None:
            hit[2].join()
        if "result" not in hit[1]:
            return None
        arrays, ev = hit[1]["result"]
        t = torch()
        cur = t.cuda.current_stream()
        cur.wait_event(ev)
        for d in arrays:
            d.record_stream(cur)   # freed after this stream's use, not the copy stream's
        return arrays

    def clear(self):
        for _, _, th in list(self.items.values()):
            if th is not None:
                th.join()
        self.items.clear()


class DeviceMatrix:
    """A krb_matrix handle (device CSR / SELL-32 + lazily built transpose)."""

    def __init__(self, n, row_ptr, col_idx, values, fmt: int = 0, uploaded=None):
        require_cuda()
        t = torch()
        self.n = int(n)
        self.nnz = int(len(values))
        row_ptr = np.asarray(row_ptr)
        col_idx = np.asarray(col_idx)
        values = np.asarray(values)
        if np.iscomplexobj(values):
            raise NotImplementedError("complex matrices are out of scope on the "
                                      "device path (fp64 real only)")
        h = ctypes.c_void_p()
        s = stream_ptr()
        if uploaded is not None:
            d_rp, d_ci, d_val = uploaded
        else:
            d_rp, d_ci = _upload_indices(row_ptr, col_idx, self.n)
            d_val = to_device(values, np.float64)
        fn = "krb_matrix_create" if d_ci.dtype == t.int32 else "krb_matrix_create_i64"
        try:
            _lib.call(fn, ctypes.byref(h), self.n, self.nnz, ptr(d_rp), ptr(d_ci),
                      ptr(d_val), int(fmt), s)
        except _lib.KrbError as e:
            if "out of memory" not in str(e):
                raise
            # the device memory may sit in torch's cache: hand it back, retry
            t.cuda.synchronize()
            t.cuda.empty_cache()
            _lib.call(fn, ctypes.byref(h), self.n, self.nnz, ptr(d_rp), ptr(d_ci),
                      ptr(d_val), int(fmt), s)
        del d_rp, d_ci, d_val
        self.h = h
        self._finalizer = weakref.finalize(self, _destroy_matrix, h.value)
        n_, nnz_, f_, b_ = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int64()
        _lib.call("krb_matrix_info", h, ctypes.byref(n_), ctypes.byref(nnz_),
                  ctypes.byref(f_), ctypes.byref(b_))
        self.format = {1: "csr", 2: "sell32", 3: "sell32-sigma", 4: "sell32-dict",
                       5: "sell32-dict-vc"}.get(f_.value, "?")
        self.device_bytes = b_.value
        sb, ns, nu, nd = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        _lib.call("krb_matrix_stream_stats", h, ctypes.byref(sb), ctypes.byref(ns),
                  ctypes.byref(nu), ctypes.byref(nd))
        # bytes one SpMV streams in this format; slice statistics
        self.stream_bytes = sb.value
        self.stream_stats = {"nslices": ns.value, "uniform_slices": nu.value, "ndict": nd.value}
        if f_.value == 5:
            ce, vl, cd, df = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
            _lib.call("krb_matrix_value_stats", h, ctypes.byref(ce), ctypes.byref(vl),
                      ctypes.byref(cd), ctypes.byref(df))
            self.stream_stats.update(const_entries=ce.value, templates=vl.value,
                                     const_diagonals=cd.value, diagonal_form=bool(df.value))

    @property
    def shape(self):
        return (self.n, self.n)

    def pattern_info(self):
        """(pattern id, live references, transpose permutation known):
        matrices with equal row_ptr / col_idx share their structure work
        (matrix.cu)."""
        pid, refs, tk = ctypes.c_uint64(), ctypes.c_int(), ctypes.c_int()
        _lib.call("krb_matrix_pattern_info", self.h, ctypes.byref(pid), ctypes.byref(refs),
                  ctypes.byref(tk))
        return pid.value, refs.value, bool(tk.value)

    def spmv(self, x_dev, y_dev=None, transpose=False):
        t = torch()
        if y_dev is None:
            y_dev = t.empty(self.n, dtype=t.float64, device="cuda")
        fn = "krb_spmv_t" if transpose else "krb_spmv"
        call_retry_oom(fn, self.h, ptr(x_dev), ptr(y_dev), stream_ptr())
        return y_dev

    def spmm(self, X_dev, transpose=False, out=None):
        """X_dev: (ncols, n) tensor = column-major n x ncols block."""
        t = torch()
        ncols = X_dev.shape[0]
        if out is None:
            out = t.empty((ncols, self.n), dtype=t.float64, device="cuda")
        if ncols:
            ldx = X_dev.stride(0) if ncols > 1 else self.n
            ldy = out.stride(0) if ncols > 1 else self.n
            call_retry_oom("krb_spmm", self.h, 1 if transpose else 0, ncols,
                      ptr(X_dev), ldx, ptr(out), ldy, stream_ptr())
        return out


def _destroy_matrix(h):
    # stream-ordered on the (single) stream the matrix is used on
    try:
        _lib.load().krb_matrix_destroy_async(ctypes.c_void_p(h), stream_ptr())
    except Exception:
        pass


def call_retry_oom(name, *args):
    """_lib.call, retried once after handing torch's cached device memory
    back when libkrb's stream-ordered pool (matrices, transposes) reports
    out of memory."""
    try:
        return _lib.call(name, *args)
    except _lib.KrbError as e:
        if "out of memory" not in str(e):
            raise
        t = torch()
        t.cuda.synchronize()
        t.cuda.empty_cache()
        return _lib.call(name, *args)


class _MatrixCache:
    """Device copies keyed on the identity of immutable host matrices (the
    reference freezes SparseMatrix arrays, sparse.py:66-67).  A strong
    reference pins each key object so ids cannot be recycled.  LRU of at most
    ``cap`` matrices and at most ``budget_frac`` of the device memory (device
    CSR + SELL + transpose: a C5 matrix is ~23 GB, so a sequence walking
    through C5 systems keeps one or two, not three)."""

    def __init__(self, cap=3, budget_frac=0.30):
        self.cap = cap
        self.budget_frac = budget_frac
        self.items: OrderedDict = OrderedDict()

    @staticmethod
    def _bytes(dev):
        b = ctypes.c_int64()
        try:
            _lib.call("krb_matrix_info", dev.h, None, None, None, ctypes.byref(b))
        except Exception:
            return 0
        return int(b.value)

    def get(self, obj, build, nnz=0):
        key = id(obj)
        hit = self.items.get(key)
        if hit is not None and hit[0] is obj:
            self.items.move_to_end(key)
            return hit[1]
        # make room first: a new matrix with its transpose needs about
        # 2 x (CSR + SELL) = ~50 bytes per stored entry
        budget = self.budget_frac * torch().cuda.get_device_properties(0).total_memory
        need = 50 * int(nnz)
        while self.items and \
                sum(self._bytes(d) for _, d in self.items.values()) + need > budget:
            self.items.popitem(last=False)
        dev = build()
        self.items[key] = (obj, dev)
        self.items.move_to_end(key)
        while len(self.items) > self.cap:
            self.items.popitem(last=False)
        budget = self.budget_frac * torch().cuda.get_device_properties(0).total_memory
        while len(self.items) > 1 and \
                sum(self._bytes(d) for _, d in self.items.values()) > budget:
            self.items.popitem(last=False)
        return dev

    def clear(self):
        self.items.clear()
        _IDX_CACHE.clear()


MATRICES = _MatrixCache()
PREFETCH = _Prefetch()


def prefetch_matrix(A) -> bool:
    """Start the upload of A's CSR arrays ahead of its first solve (pinned
    inputs: DMA on a copy stream; pageable: a background thread stages them);
    returns whether an upload was started."""
    return PREFETCH.issue(A)


def device_matrix(A) -> DeviceMatrix:
    """Resolve any supported operator to its device matrix."""
    if isinstance(A, DeviceMatrix):
        return A
    dev = getattr(A, "_device", None)
    if isinstance(dev, DeviceMatrix):
        return dev
    if hasattr(A, "factors") and hasattr(A, "_A"):
        # split ILUTP operator (ilutp.py:106-128; ours or the reference's)
        from .precond import device_operator
        return device_operator(A)
    inner = getattr(A, "inner", None)
    if inner is not None and not hasattr(A, "row_ptr"):
        return device_matrix(inner)
    if hasattr(A, "row_ptr") and hasattr(A, "col_idx") and hasattr(A, "values"):
        require_cuda()
        n = A.nrows if hasattr(A, "nrows") else A.n
        ncols = A.ncols if hasattr(A, "ncols") else n
        if n != ncols:
            raise ValueError("solver requires a square operator")
        return MATRICES.get(A, lambda: DeviceMatrix(n, A.row_ptr, A.col_idx,
                                                    A.values, uploaded=PREFETCH.take(A)),
                            nnz=len(A.values))
    if isinstance(A, np.ndarray):
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise ValueError("solver requires a square operator")
        import scipy.sparse as sp

        def build():
            S = sp.csr_matrix(A)
            S.sort_indices()
            return DeviceMatrix(A.shape[0], S.indptr, S.indices, S.data)

        if A.flags.writeable:
            # a mutable array may be edited in place between calls (the
            # reference's DenseOperator reads the live array on every
            # product): never serve a cached device copy of it
            return build()
        return MATRICES.get(A, build)
    raise NotImplementedError(
        f"{type(A).__name__} has no CSR representation; the device path "
        "supports SparseMatrix-like CSR operators only (no CPU fallback)")
