"""ctypes binding of libkrb.so (include/krb.h).

This is the only place the product touches native code.  It fails loudly:
there is no CPU fallback — if the shared library is missing or no CUDA device
is present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkrb.so")
CSRC = os.path.join(_HERE, "csrc")

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

KRB_STATUS = {
    1: "converged",
    2: "max_itn",
    3: "breakdown:serious",
    4: "breakdown:omega",
    5: "breakdown:second_kind",
}


class KrbError(RuntimeError):
    pass


class SpaceView(ctypes.Structure):
    _fields_ = [("n", c_i64), ("k", c_i64), ("ld", c_i64),
                ("U", c_vp), ("Ut", c_vp), ("C", c_vp), ("Ct", c_vp),
                ("Chat", c_vp), ("Ccheck", c_vp)]


class SolveConfig(ctypes.Structure):
    _fields_ = [("tol", c_dbl), ("breakdown_tol", c_dbl), ("max_itn", c_i64),
                ("d_shadow", c_vp),
                ("pcg_state_hi", c_u64), ("pcg_state_lo", c_u64),
                ("pcg_inc_hi", c_u64), ("pcg_inc_lo", c_u64),
                ("use_graph", c_int), ("d_phase_stamps", c_vp),
                ("phase_stamps_cap", c_i64), ("d_kernel_times", c_vp),
                ("d_rec_x", c_vp), ("d_rec_r", c_vp), ("d_rec_xc", c_vp),
                ("d_rec_s", c_vp), ("d_rec_t", c_vp), ("d_rec_omega", c_vp)]


class SolveResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("hist_len", c_i64),
                ("matvecs", c_i64), ("rhs_norm", c_dbl),
                ("final_true_resid", c_dbl), ("t_start_ns", c_u64),
                ("iterations_run", c_i64), ("kernel_launches", c_i64),
                ("driver", ctypes.c_int32)]


DRIVERS = {0: "host_loop", 1: "graph", 2: "persistent", 3: "fused", 4: "cluster",
           5: "batch_graph"}


# name -> (restype, argtypes); every symbol declared in include/krb.h
SIGNATURES = {
    "krb_abi_version": (c_int, []),
    "krb_last_error": (ctypes.c_char_p, []),
    "krb_launch_count": (c_i64, []),
    "krb_set_tuning": (c_int, [ctypes.c_char_p, c_i64]),
    "krb_reset_tuning": (c_int, []),
    "krb_set_allocator": (c_int, [c_vp, c_vp]),
    "krb_context_create": (c_int, [ctypes.POINTER(c_vp)]),
    "krb_context_destroy": (c_int, [c_vp]),
    "krb_matrix_create": (c_int, [ctypes.POINTER(c_vp), c_i64, c_i64, c_vp,
                                  c_vp, c_vp, c_int, c_vp]),
    "krb_matrix_create_i64": (c_int, [ctypes.POINTER(c_vp), c_i64, c_i64,
                                      c_vp, c_vp, c_vp, c_int, c_vp]),
    "krb_matrix_destroy": (c_int, [c_vp]),
    "krb_matrix_destroy_async": (c_int, [c_vp, c_vp]),
    "krb_matrix_stream_stats": (c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                                        ctypes.POINTER(c_i64), ctypes.POINTER(c_int)]),
    "krb_matrix_value_stats": (c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_int),
                                       ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "krb_matrix_pattern_info": (c_int, [c_vp, ctypes.POINTER(ctypes.c_uint64),
                                        ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "krb_matrix_info": (c_int, [c_vp, ctypes.POINTER(c_i64),
                                ctypes.POINTER(c_i64), ctypes.POINTER(c_int),
                                ctypes.POINTER(c_i64)]),
    "krb_spmv": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "krb_spmv_t": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "krb_spmm": (c_int, [c_vp, c_int, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "krb_dot": (c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "krb_tdot": (c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "krb_gemv": (c_int, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_int, c_vp,
                         c_vp]),
    "krb_gram": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                         c_vp, c_vp]),
    "krb_gemm": (c_int, [c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64,
                         c_vp]),
    "krb_colnorms": (c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "krb_colscale_div": (c_int, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "krb_colscale_div_to": (c_int, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "krb_uniform_pcg64": (c_int, [c_i64, c_u64, c_u64, c_u64, c_u64, c_dbl,
                                  c_dbl, c_vp, c_vp]),
    "krb_rbicgstab": (c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(SpaceView),
                              ctypes.POINTER(SolveConfig), c_vp, c_vp, c_vp,
                              c_vp, ctypes.POINTER(SolveResult), c_vp]),
    "krb_last_scalars": (c_int, [c_vp, ctypes.POINTER(c_dbl)]),
    "krb_rbicgstab_batch": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp,
                                    ctypes.POINTER(SpaceView),
                                    ctypes.POINTER(SolveConfig), c_vp, c_vp, c_vp,
                                    c_vp, ctypes.POINTER(SolveResult), c_vp]),
    "krb_memcpy_d2d": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "krb_ilutp_factor": (c_int, [c_i64, c_vp, c_vp, c_vp, c_dbl, c_dbl, c_i64,
                                 ctypes.POINTER(c_vp)]),
    "krb_ilutp_sizes": (c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "krb_ilutp_export": (c_int, [c_vp] + [c_vp] * 7),
    "krb_ilutp_free": (c_int, [c_vp]),
    "krb_tri_levels": (c_int, [c_i64, c_vp, c_vp, c_int, c_vp, ctypes.POINTER(ctypes.c_int32)]),
    "krb_precond_create": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp), c_vp]),
    "krb_precond_destroy": (c_int, [c_vp]),
    "krb_precond_apply": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp]),
    "krb_operator_create": (c_int, [c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "krb_colsq": (c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "krb_ritz_combine": (c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64,
                                 c_vp, c_vp, c_vp]),
    "krb_rbicg_create": (c_int, [ctypes.POINTER(c_vp), c_vp, c_vp,
                                 ctypes.POINTER(SpaceView), c_i64, c_i64, c_vp]),
    "krb_rbicg_destroy": (c_int, [c_vp]),
    "krb_rbicg_start": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_dbl, c_dbl,
                                c_int, ctypes.POINTER(c_dbl), c_vp]),
    "krb_rbicg_set_counts": (c_int, [c_vp, c_i64, c_i64, c_vp]),
    "krb_rbicg_begin": (c_int, [c_vp, ctypes.POINTER(ctypes.c_int32), c_vp]),
    "krb_rbicg_run": (c_int, [c_vp, ctypes.POINTER(c_i64), c_vp]),
    "krb_rbicg_launch": (c_int, [c_vp, ctypes.POINTER(ctypes.c_int32), c_vp]),
    "krb_rbicg_wait": (c_int, [c_vp, ctypes.POINTER(c_i64), c_vp]),
    "krb_rbicg_views": (c_int, [c_vp] + [ctypes.POINTER(c_vp)] * 5),
    "krb_rbicg_rotate": (c_int, [c_vp, c_i64, c_vp]),
    "krb_rbicg_finish": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                 ctypes.POINTER(SolveResult),
                                 ctypes.POINTER(c_i64), ctypes.POINTER(c_dbl),
                                 c_vp]),
}

_lock = threading.Lock()
_lib = None


BUILD_INFO = os.path.join(_HERE, "build_info.json")


def build(force: bool = False) -> str:
    """Compile libkrb.so in-tree with nvcc for sm_100a (make in csrc/).
    ``force`` cleans first so every object is rebuilt from source; the
    compile commands, the nvcc version and a hash of the sources are written
    to build_info.json next to the library (evidence of a fresh build)."""
    import hashlib
    import json
    import time
    t0 = time.time()
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    dry = subprocess.run(["make", "-n", "-C", CSRC], check=True, capture_output=True,
                         text=True).stdout
    subprocess.run(["make", "-s", "-C", CSRC, "-j8"], check=True)
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cu", ".cuh")) or name == "Makefile":
            with open(os.path.join(CSRC, name), "rb") as f:
                h.update(name.encode() + f.read())
    nvcc = subprocess.run(["nvcc", "--version"], capture_output=True, text=True).stdout
    info = {"built_at": time.strftime("%Y-%m-%dT%H:%M:%S"), "clean": bool(force),
            "seconds": round(time.time() - t0, 1), "sources_sha256": h.hexdigest(),
            "nvcc": nvcc.strip().splitlines()[-1] if nvcc else None,
            "commands": [ln.strip() for ln in dry.splitlines() if "nvcc" in ln]}
    with open(BUILD_INFO, "w") as f:
        json.dump(info, f, indent=1)
    return LIB_PATH


def load(path: str | None = None):
    """Load libkrb.so and bind every exported symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise KrbError(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ "
                "as g; g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
        lib = ctypes.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = load().krb_last_error()
        raise KrbError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")


def call(name: str, *args):
    """Call an entry point and raise KrbError on a non-zero return."""
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc


# Python-side driver knobs (see tuning()): "graph_mode" = None (automatic),
# 0 host loop, 1 CUDA graph with a device WHILE node, 2 persistent kernel;
# "phase_prof" = per-phase device stamps of the persistent kernel.
# "kernel_times" = a zeroed (384,) int64 CUDA tensor that the graph /
# host-loop drivers accumulate live per-kernel device time into
# (krb_solve_config.d_kernel_times).
PY_TUNING = {"graph_mode": None, "phase_prof": False, "kernel_times": None}
_PY_DEFAULTS = dict(PY_TUNING)


class tuning:
    """Context manager (or plain call + reset_tuning()) setting driver /
    kernel-variant knobs for tests and profiling tools; every variant
    computes the same bits.  Python keys: graph_mode, phase_prof,
    kernel_times; native keys: see krb_set_tuning in include/krb.h."""

    def __init__(self, **knobs):
        for key, v in knobs.items():
            if key in PY_TUNING:
                PY_TUNING[key] = v
            else:
                call("krb_set_tuning", key.encode(), int(v))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        reset_tuning()


def reset_tuning():
    PY_TUNING.update(_PY_DEFAULTS)
    if _lib is not None:
        _lib.krb_reset_tuning()


def launch_count() -> int:
    return int(load().krb_launch_count())


def copy_d2d(dst_tensor, src_addr: int, count: int):
    """Device-to-device copy of `count` doubles from a raw device address
    (libkrb ring views) into a torch tensor, on the current stream."""
    if count <= 0:
        return
    from .device import stream_ptr
    call("krb_memcpy_d2d", ctypes.c_void_p(dst_tensor.data_ptr()),
         ctypes.c_void_p(src_addr), 8 * count, stream_ptr())


def fetch_f64(src_addr: int, count: int):
    """Copy `count` doubles from a raw device address to a host numpy array."""
    import numpy as np
    import torch
    if count <= 0:
        return np.zeros(0)
    out = torch.empty(count, dtype=torch.float64, device="cuda")
    copy_d2d(out, src_addr, count)
    return out.cpu().numpy()


def fetch_f64_many(parts):
    """Several (device address, count) ranges of doubles to host numpy arrays
    with ONE device->host read (one synchronisation)."""
    import numpy as np
    import torch
    total = sum(max(c, 0) for _, c in parts)
    if total == 0:
        return [np.zeros(0) for _ in parts]
    buf = torch.empty(total, dtype=torch.float64, device="cuda")
    off = 0
    for addr, c in parts:
        if c > 0:
            copy_d2d(buf[off:], addr, c)
            off += c
    host = buf.cpu().numpy()
    out, off = [], 0
    for _, c in parts:
        c = max(c, 0)
        out.append(host[off:off + c])
        off += c
    return out
