"""ctypes binding of libxlmimo_b200.so (the C-ABI in include/xlmimo_b200.h).

There is no CPU fallback: if the shared library is missing, fails to load or
no CUDA device is visible, every compute entry point raises
:class:`BackendUnavailable`.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (ConfigurationError, DegenerateChannelError,
                     GeometryInfeasibleError, NotHpdError, SplittingError,
                     XlMimoError)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_native",
                        "libxlmimo_b200.so")

XL_C64, XL_C128 = 0, 1
XL_JACPCG, XL_CG, XL_DIRECT = 0, 1, 2
XL_JOR, XL_GS = 3, 4
XL_TEXTBOOK, XL_ALGORITHM = 0, 1
XL_SUCCESS, XL_ERR_CONFIG, XL_ERR_CUDA, XL_ERR_UNSUPPORTED, XL_ERR_WORKSPACE = 0, 1, 2, 3, 4
XL_STATUS_RANGE = 6

STATUS_EXCEPTIONS = {
    1: (NotHpdError, "nonpositive direction curvature encountered; P is not HPD"),
    2: (SplittingError, "preconditioner has zero diagonal entry"),
    3: (DegenerateChannelError, "tr(F^H F) = 0; channel block carries no energy"),
    4: (NotHpdError, "Cholesky breakdown: matrix is not positive definite"),
    5: (GeometryInfeasibleError, "no visible subarray after the retry budget"),
    6: (XlMimoError, "fp16-split range exceeded (re-run on the general path)"),
}


class BackendUnavailable(XlMimoError, RuntimeError):
    """The sm_100a shared library or a CUDA device is not available."""


class BackendError(XlMimoError, RuntimeError):
    """A CUDA launch or runtime error inside the library."""


_lib = None

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_f64 = ctypes.c_double
_sz = ctypes.c_size_t
_int = ctypes.c_int

_SIGNATURES = {
    "xl_abi_version": (_int, []),
    "xl_last_error": (ctypes.c_char_p, []),
    "xl_launch_count": (_u64, []),
    "xl_rzf_uses_tensor_cores": (_int, [_int, _int, _i32, _i32]),
    "xl_gram": (_int, [_int, _p, _i64, _i32, _i32, _f64, _p, _p, _p]),
    "xl_solve_workspace_bytes": (_sz, [_int, _i64, _i32, _i32]),
    "xl_solve": (_int, [_int, _int, _int, _p, _i64, _i32, _p, _i32, _p, _p, _i32,
                        _i32, _f64, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "xl_solve_stationary": (_int, [_int, _int, _p, _i64, _i32, _p, _i32, _p, _f64, _i32, _f64,
                                   _p, _p, _p, _p, _p, _p, _sz, _p]),
    "xl_rzf_workspace_bytes": (_sz, [_int, _int, _i64, _i32, _i32]),
    "xl_rzf": (_int, [_int, _int, _int, _p, _i64, _i32, _i32, _f64, _p, _f64, _i32,
                      _f64, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "xl_rzf_general_workspace_bytes": (_sz, [_int, _int, _i64, _i32, _i32]),
    "xl_rzf_general": (_int, [_int, _int, _int, _p, _i64, _i32, _i32, _f64, _p, _f64, _i32,
                              _f64, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "xl_rzf_traced": (_int, [_int, _int, _int, _p, _i64, _i32, _i32, _f64, _p, _f64, _i32,
                             _f64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "xl_debug_set_gram_out": (None, [_p]),
    "xl_debug_lk_trace": (None, [_p]),
    "xl_apply_precoder_workspace_bytes": (_sz, [_int, _i64, _i32, _i32]),
    "xl_apply_precoder": (_int, [_int, _p, _p, _i64, _i32, _i32, _f64, _f64, _p, _p, _p,
                                 _p, _p, _p, _p, _sz, _p]),
    "xl_sinr_workspace_bytes": (_sz, [_int, _i64, _i32]),
    "xl_sinr": (_int, [_int, _p, _p, _i64, _i32, _i32, _f64, _p, _p, _p, _p, _sz, _p]),
    "xl_channel_generate": (_int, [_int, _u64, _i64, _i64, _i32, _i32, _i32, _f64, _p,
                                   _f64, _f64, _f64, _p, _p, _p]),
    "xl_se_partials": (_int, [_p, _i64, _i64, _p, _p]),
    "xl_se_combine": (_int, [_p, _i64, _p, _p]),
    "xl_ber_errors": (_int, [_int, _p, _p, _p, _i64, _i32, _i32, _p, _p]),
}


def load_library():
    """Load the shared library (no device needed) and bind every symbol."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendUnavailable(
            f"{LIB_PATH} not built; run __graft_entry__.build() "
            "(python -m paper_2305_13925_b200.build_ext)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    """The library, only once a CUDA device is present (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise BackendUnavailable(
            "no CUDA device: the B200 precoding path has no CPU fallback")
    return load_library()


def check(rc: int, what: str = "") -> None:
    if rc == XL_SUCCESS:
        return
    msg = (_lib.xl_last_error() or b"").decode(errors="replace")
    if rc == XL_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == XL_ERR_UNSUPPORTED:
        raise ConfigurationError(f"unsupported shape: {msg}")
    raise BackendError(f"{what}: rc={rc}: {msg}")


def raise_status(status_host, what: str = "") -> None:
    """Raise the reference exception for the first failing realization."""
    import numpy as np
    st = np.asarray(status_host)
    bad = np.flatnonzero(st)
    if bad.size:
        code = int(st[bad[0]])
        exc, msg = STATUS_EXCEPTIONS.get(code, (XlMimoError, f"status {code}"))
        where = f" (realization {int(bad[0])}{' of ' + what if what else ''})"
        raise exc(msg + where)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
