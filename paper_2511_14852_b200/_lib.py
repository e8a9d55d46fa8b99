"""ctypes binding of the C ABI (include/chebykan.h).

The library is built in-tree (``python -m paper_2511_14852_b200.build``) and
loaded from ``paper_2511_14852_b200/lib/libchebykan.so``.  There is no
fallback: if the library is missing or the device is not sm_100, calls fail
loudly.
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import threading

LIB_PATH = pathlib.Path(__file__).resolve().parent / "lib" / "libchebykan.so"
if os.environ.get("CK_LIB_PATH"):  # A/B experiments with a variant build (tools/build_variant.py)
    LIB_PATH = pathlib.Path(os.environ["CK_LIB_PATH"]).resolve()

# ck_status codes (include/chebykan.h)
CK_OK = 0
CK_INVALID_ARGUMENT = 1
CK_CUDA_ERROR = 2
CK_UNSUPPORTED = 3
CK_WORKSPACE_TOO_SMALL = 4

_c_int, _c_i64, _c_size, _c_p = ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
_c_dp = ctypes.POINTER(ctypes.c_double)
_c_fp = ctypes.POINTER(ctypes.c_float)

# name -> (restype, argtypes); must list every symbol in include/chebykan.h
SIGNATURES = {
    "ck_version": (_c_int, []),
    "ck_last_error": (ctypes.c_char_p, []),
    "ck_device_supported": (_c_int, [_c_int]),
    "ck_lut_build": (_c_int, [_c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_c_p)]),
    "ck_lut_create": (_c_int, [_c_int, _c_int, _c_int, _c_dp, _c_fp, _c_int, ctypes.POINTER(_c_p)]),
    "ck_basis_exact": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(_c_p)]),
    "ck_lut_destroy": (None, [_c_p]),
    "ck_lut_info": (_c_int, [_c_p, ctypes.POINTER(_c_int), ctypes.POINTER(_c_int), _c_dp]),
    "ck_lut_kind": (_c_int, [_c_p, ctypes.POINTER(_c_int), ctypes.POINTER(_c_int), ctypes.POINTER(_c_int)]),
    "ck_lut_read": (_c_int, [_c_p, _c_dp, _c_fp]),
    "ck_expand": (_c_int, [_c_p, _c_i64, _c_int, _c_p, _c_p, _c_p, _c_p]),
    "ck_basis_eval": (_c_int, [_c_p, _c_i64, _c_p, _c_p, _c_p, _c_p]),
    "ck_coeff_prep_bytes": (_c_size, [_c_int, _c_int, _c_int]),
    "ck_coeff_prepare": (_c_int, [_c_p, _c_int, _c_int, _c_int, _c_p, _c_size, _c_p]),
    "ck_forward_workspace_bytes": (_c_size, [_c_i64, _c_int, _c_int, _c_int]),
    "ck_basis_cache_bytes": (_c_size, [_c_i64, _c_int, _c_int, _c_int]),
    "ck_coeff_prep_check": (_c_int, [_c_p, _c_size, _c_int, _c_int, _c_int]),
    "ck_set_chunk_rows": (_c_i64, [_c_i64]),
    "ck_forward": (_c_int, [_c_p, _c_i64, _c_int, _c_int, _c_p, _c_p, _c_size, _c_p, _c_p, _c_p, _c_size, _c_p,
                            _c_size, _c_p]),
    "ck_backward_workspace_bytes": (_c_size, [_c_i64, _c_int, _c_int, _c_int]),
    "ck_backward": (_c_int, [_c_p, _c_p, _c_i64, _c_int, _c_int, _c_p, _c_p, _c_size, _c_int, _c_p, _c_p, _c_p,
                             _c_p, _c_size, _c_p, _c_size, _c_p, _c_p]),
    "ck_set_gemm_sm_reserve": (_c_int, [_c_int]),
    "ck_merge": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_int, _c_p]),
    "ck_forward_partial": (_c_int, [_c_p, _c_i64, _c_int, _c_int, _c_p, _c_p, _c_int, _c_int, _c_p, _c_p, _c_p]),
    "ck_combine": (_c_int, [_c_p, _c_i64, _c_int, _c_int, _c_int, _c_p, _c_p, _c_p]),
    "ck_adam_step": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_i64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, _c_i64, _c_p]),
    "ck_adam_begin": (_c_int, [_c_p, _c_p, ctypes.c_double, ctypes.c_double, _c_p]),
    "ck_adam_step_dev": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_i64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_double, _c_p, _c_p]),
    "ck_adam_step_multi": (_c_int, [_c_int, ctypes.POINTER(_c_p), ctypes.POINTER(_c_p), ctypes.POINTER(_c_p),
                                    ctypes.POINTER(_c_p), ctypes.POINTER(_c_i64), ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, _c_i64, _c_p, _c_p]),
    "ck_ipc_handle": (_c_int, [_c_p, _c_p, ctypes.POINTER(_c_i64)]),
    "ck_ipc_open": (_c_int, [_c_p, _c_i64, ctypes.POINTER(_c_p)]),
    "ck_ipc_close": (_c_int, [_c_p, _c_i64]),
    "ck_allreduce_peers": (_c_int, [ctypes.POINTER(_c_p), _c_int, _c_int, _c_i64, _c_p]),
    "ck_peer_flag_words": (_c_int, []),
    "ck_allreduce_peers_flags": (_c_int, [ctypes.POINTER(_c_p), ctypes.POINTER(_c_p), _c_int, _c_int, _c_i64, _c_i64,
                                          ctypes.c_uint64, _c_int, _c_p]),
    "ck_launch_count": (ctypes.c_longlong, []),
    "ck_timing_enable": (_c_int, [_c_int]),
    "ck_timing_collect": (_c_int, [_c_dp, ctypes.POINTER(ctypes.c_longlong), _c_int]),
    "ck_debug_gemm_trace": (_c_int, [ctypes.c_void_p, _c_int]),
    "ck_mse_workspace_bytes": (ctypes.c_size_t, [_c_i64]),
    "ck_mse_loss": (_c_int, [_c_p, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_p, ctypes.c_size_t, _c_p]),
}

KERNEL_CLASSES = ("gemm_fwd", "gemm_dx", "gemm_dc", "expand", "expand_t", "dx_combine", "split", "reduce", "lut",
                  "optim", "skinny")


def launch_count() -> int:
    return int(lib().ck_launch_count())


def timing_enable(on: bool) -> None:
    lib().ck_timing_enable(1 if on else 0)


def timing_collect() -> dict:
    """{class: (ms, launches)} since the last collect (waits for the events)."""
    n = len(KERNEL_CLASSES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_longlong * n)()
    check(lib().ck_timing_collect(ms, cnt, n), "ck_timing_collect")
    return {KERNEL_CLASSES[i]: (ms[i], int(cnt[i])) for i in range(n)}

_lib = None
_lock = threading.Lock()


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or the device is unsupported."""


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing; build it with `python -m paper_2511_14852_b200.build` "
                    "(there is no CPU fallback)")
            handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().ck_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    """Map a ck_status to the reference's exception types."""
    if rc == CK_OK:
        return
    msg = last_error()
    if rc == CK_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == CK_WORKSPACE_TOO_SMALL:
        raise RuntimeError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what} failed ({rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(device) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream
