"""ctypes binding of libw2l_criterion.so (the C-ABI in include/w2l_criterion.h).

The library is built in-tree (``paper_1812_07625_b200/lib``) by
``paper_1812_07625_b200._build``.  There is no fallback: if the library is
missing or fails to load, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

from ._build import LIB as _BUILT_LIB

# W2L_LIB selects another build of the same library (A/B timing in tools/ab.sh)
LIB = os.environ.get("W2L_LIB", _BUILT_LIB)
if not os.path.isabs(LIB):   # relative to the repo root (subprocesses change directory)
    LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), LIB)

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "w2l_criterion.h")

c_p = ctypes.c_void_p
c_i = ctypes.c_int
c_sz = ctypes.c_size_t
c_d_p = ctypes.POINTER(ctypes.c_double)
c_i32_p = ctypes.POINTER(ctypes.c_int32)

# name -> (restype, argtypes); mirrors include/w2l_criterion.h
SIGNATURES = {
    "w2l_asg_workspace_bytes": (c_sz, [c_i, c_i, c_i, c_i]),
    "w2l_asg_loss_grad": (c_i, [c_p, c_p, c_p, c_p, c_p, c_i, c_i, c_i, c_i, c_p, c_p, c_p, c_p,
                                c_p, c_p, c_sz, ctypes.c_uint, c_p]),
    "w2l_asg_workspace_bytes_f64": (c_sz, [c_i, c_i, c_i, c_i]),
    "w2l_asg_loss_grad_f64": (c_i, [c_p, c_p, c_p, c_p, c_p, c_i, c_i, c_i, c_i, c_p, c_p, c_p,
                                    c_p, c_p, c_p, c_sz, c_p]),
    "w2l_ctc_workspace_bytes": (c_sz, [c_i, c_i, c_i, c_i]),
    "w2l_ctc_loss_grad": (c_i, [c_p, c_p, c_p, c_p, c_i, c_i, c_i, c_i, c_i, c_p, c_p, c_p, c_p,
                                c_sz, ctypes.c_uint, c_p]),
    "w2l_ctc_workspace_bytes_f64": (c_sz, [c_i, c_i, c_i, c_i]),
    "w2l_ctc_loss_grad_f64": (c_i, [c_p, c_p, c_p, c_p, c_i, c_i, c_i, c_i, c_i, c_p, c_p, c_p,
                                    c_p, c_sz, c_p]),
    "w2l_viterbi_workspace_bytes": (c_sz, [c_i, c_i, c_i]),
    "w2l_viterbi": (c_i, [c_p, c_p, c_p, c_i, c_i, c_i, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "w2l_viterbi_f64": (c_i, [c_p, c_p, c_p, c_i, c_i, c_i, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "w2l_greedy_eval": (c_i, [c_p, c_p, c_i, c_i, c_i, c_i, c_p, c_p, c_i, c_i, c_p, c_p, c_p, c_p,
                              c_p, c_p, c_p]),
    "w2l_asg_loss_grad_traced": (c_i, [c_p, c_p, c_p, c_p, c_p, c_i, c_i, c_i, c_i, c_p, c_p,
                                       c_p, c_p, c_p, c_p, c_sz, ctypes.c_uint, c_p, c_p, c_p]),
    "w2l_ctc_loss_grad_traced": (c_i, [c_p, c_p, c_p, c_p, c_i, c_i, c_i, c_i, c_i, c_p, c_p,
                                       c_p, c_p, c_sz, ctypes.c_uint, c_p, c_p, c_p]),
    "w2l_stage_name": (ctypes.c_char_p, [c_i, c_i]),
    "w2l_status_first_error": (c_i, [c_p, c_i, c_i32_p, c_p]),
    "w2l_status_string": (ctypes.c_char_p, [c_i]),
    "w2l_version": (ctypes.c_char_p, []),
    "w2l_last_cuda_error": (ctypes.c_char_p, []),
    "w2l_probe_peaks": (c_i, [c_d_p, c_d_p, c_d_p]),
    "w2l_transitions_sgd_step": (c_i, [c_p, c_p, c_p, c_i, c_i, ctypes.c_float, ctypes.c_float,
                                       c_p]),
    "w2l_comm_available": (c_i, []),
    "w2l_comm_unique_id": (c_i, [c_p]),
    "w2l_comm_init": (c_i, [c_p, c_i, c_i, ctypes.POINTER(c_p)]),
    "w2l_comm_destroy": (c_i, [c_p]),
    "w2l_allreduce_grad_A": (c_i, [c_p, c_i, c_p, c_p]),
}

# C-ABI status codes (include/w2l_criterion.h)
OK, ERR_CONTRACT, ERR_NUMERIC, ERR_TARGET, ERR_INFEASIBLE, ERR_CUDA, ERR_COMM, ERR_PRECISION = \
    range(8)
FLAG_NO_FALLBACK = 1
FLAG_PHASE_CHAIN = 2
FLAG_PHASE_GRAD = 4
FLAG_LOSS_ONLY = 8
FLAG_CTC_LOGITS = 16
FLAG_FORCE_EXACT = 32
FLAG_NO_LOG_FALLBACK = 64
FLAG_NO_ROUTE = 128
FLAG_PHASE_VALIDATE = 256
FLAG_VALIDATED = 512
FLAG_STREAM_GRAD = 1024
MAX_TOKENS = 32
MAX_ASG_LABELS = 1024
MAX_CTC_LABELS = 511

_lib = None
_lock = threading.Lock()


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing or unusable; there is no CPU fallback."""


def header_symbols() -> list[str]:
    """Function names declared in include/w2l_criterion.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(w2l_[A-Za-z0-9_]+)\s*\(", text)))


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB):
                raise NativeLibraryError(
                    f"{LIB} is not built; run `python -m paper_1812_07625_b200._build` "
                    "(there is no CPU fallback)")
            handle = ctypes.CDLL(LIB)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def version() -> str:
    return lib().w2l_version().decode()


def probe_peaks() -> dict:
    m, d, f = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    rc = lib().w2l_probe_peaks(ctypes.byref(m), ctypes.byref(d), ctypes.byref(f))
    if rc != OK:
        raise NativeLibraryError(f"w2l_probe_peaks failed ({rc})")
    return {"mufu_ex2_per_s": m.value, "dadd_per_s": d.value, "ffma_per_s": f.value}
