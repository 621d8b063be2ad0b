"""ctypes binding of the C ABI in include/pluq_b200.h (libpluq_b200.so, built in-tree).

The product path has no CPU fallback: if the shared library is missing or no CUDA
device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpluq_b200.so")

# Status codes (include/pluq_b200.h)
PLUQ_OK, PLUQ_EINVAL, PLUQ_EZERODIV, PLUQ_ECUDA, PLUQ_ENOMEM, PLUQ_EUNSUPPORTED = range(6)

_i64 = ctypes.c_int64
_p = ctypes.c_void_p
_pi64 = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes)
SIGNATURES = {
    "pluq_create": (ctypes.c_int, [ctypes.POINTER(_p), ctypes.c_int, _p]),
    "pluq_destroy": (ctypes.c_int, [_p]),
    "pluq_set_stream": (ctypes.c_int, [_p, _p]),
    "pluq_release_workspace": (ctypes.c_int, [_p]),
    "pluq_set_option": (ctypes.c_int, [_p, ctypes.c_char_p, _i64]),
    "pluq_get_option": (ctypes.c_int, [_p, ctypes.c_char_p, _pi64]),
    "pluq_check_residues": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _i64]),
    "pluq_last_error": (ctypes.c_char_p, [_p]),
    "pluq_last_stats": (ctypes.c_int, [_p, _pi64, _i64]),
    "pluq_measure_peaks": (ctypes.c_int, [_p, ctypes.POINTER(ctypes.c_double), _i64]),
    "pluq_nonzero": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _pi64]),
    "pluq_generic_counts": (ctypes.c_int, [_i64, _i64, _i64, _i64, _pi64]),
    "pluq_rank_profile_replay": (ctypes.c_int, [_i64, _i64, _i64, _i64, _pi64, _pi64, _pi64, _pi64, _pi64]),
    "pluq_factor": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _i64, _i64, _pi64, _pi64, _pi64, _pi64]),
    "pluq_factor_iterative": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _i64, _pi64, _pi64, _pi64, _pi64]),
    "pluq_factor_batched": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p]),
    "pluq_batched_max_elems": (_i64, [_p, _i64, _i64]),
    "pluq_factor_host_f64": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _i64, _pi64, _pi64, _pi64, _pi64]),
    "pluq_factor_host_i64": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _i64, _pi64, _pi64, _pi64, _pi64]),
    "pluq_factor_batched_host_f64": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _i64, _i64, _pi64, _pi64, _pi64]),
    "pluq_modgemm_sub": (ctypes.c_int, [_p, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _i64]),
    "pluq_modgemm_sub_tc": (ctypes.c_int, [_p, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _i64]),
    "pluq_trsm_llu": (ctypes.c_int, [_p, _p, _i64, _p, _i64, _i64, _i64, _i64]),
    "pluq_trsm_ru": (ctypes.c_int, [_p, _p, _i64, _p, _i64, _i64, _i64, _i64]),
    "pluq_permute_rows": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _pi64]),
    "pluq_permute_cols": (ctypes.c_int, [_p, _p, _i64, _i64, _i64, _pi64]),
}

_lib = None
_lock = threading.Lock()


def load_library():
    """Load libpluq_b200.so (no compute, no GPU needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the CUDA extension first "
                    "(python -c 'import __graft_entry__ as g; g.build()')"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class NativeError(RuntimeError):
    pass


def raise_for(status: int, ctx=None, what: str = "") -> None:
    if status == PLUQ_OK:
        return
    msg = what
    if ctx is not None and ctx.handle:
        detail = load_library().pluq_last_error(ctx.handle)
        if detail:
            msg = f"{what}: {detail.decode(errors='replace')}" if what else detail.decode(errors="replace")
    if status == PLUQ_EINVAL:
        raise ValueError(msg or "invalid argument")
    if status == PLUQ_EZERODIV:
        raise ZeroDivisionError(msg or "division by zero")
    if status == PLUQ_ENOMEM:
        raise MemoryError(msg or "out of device memory")
    if status == PLUQ_EUNSUPPORTED:
        raise NotImplementedError(msg or "unsupported shape")
    raise NativeError(msg or f"CUDA error (status {status})")


class Context:
    """One native context per (thread, device): stream, workspace, staging buffers."""

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1301_4438_b200 requires a CUDA device (no CPU fallback)")
        self.device = device
        self.lib = load_library()
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            torch.cuda.current_stream(device)  # make sure torch's context is live
            raise_for(self.lib.pluq_create(ctypes.byref(h), device, None), None, "pluq_create")
        self.handle = h

    def bind_stream(self):
        import torch

        s = torch.cuda.current_stream(self.device).cuda_stream
        self.lib.pluq_set_stream(self.handle, ctypes.c_void_p(s))

    def set_option(self, key: str, value: int) -> None:
        raise_for(self.lib.pluq_set_option(self.handle, key.encode(), int(value)), self, f"option {key}")

    def get_option(self, key: str) -> int:
        out = ctypes.c_int64()
        raise_for(self.lib.pluq_get_option(self.handle, key.encode(), ctypes.byref(out)), self, f"option {key}")
        return int(out.value)

    def stats(self) -> dict:
        buf = (ctypes.c_int64 * 19)()
        self.lib.pluq_last_stats(self.handle, buf, 19)
        keys = ["launches", "host_syncs", "nodes", "small_node_kernels", "basecase_kernels",
                "tc_gemms", "simt_gemms", "zero_skips", "generic_leaves", "speculative_ok",
                "speculative_fail", "t_generic_ns", "t_fallback_ns", "t_tc_mma_ns",
                "tc_timed_launches", "tc_timed_ns", "tc_timed_int8_ops", "spec_repairs", "early_chunks"]
        return dict(zip(keys, list(buf)))

    def measure_peaks(self) -> dict:
        """Microbenchmarked int8 tcgen05 and FP64 DMMA peaks of this device."""
        buf = (ctypes.c_double * 2)()
        raise_for(self.lib.pluq_measure_peaks(self.handle, buf, 2), self, "pluq_measure_peaks")
        return {"int8_tops": buf[0], "fp64_tflops": buf[1]}

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.pluq_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_tls = threading.local()


def context(device: int | None = None) -> Context:
    import torch

    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    ctx = cache.get(device)
    if ctx is None:
        ctx = cache[device] = Context(device)
    ctx.bind_stream()
    return ctx


def i64p(arr):
    """Pointer to a contiguous numpy int64 array (or NULL)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(_pi64)
