"""ctypes binding of libevo.so (include/evo.h).

There is deliberately no fallback: if the library is missing or cannot be
loaded, every op raises ``NativeLibraryMissing``.  Status codes are mapped onto
the reference's exception classes (errors.py).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DimensionError, DomainError, KernelError, NativeLibraryMissing

LIB_PATH = os.environ.get("EVO_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libevo.so")

EVO_OK, EVO_ERR_SHAPE, EVO_ERR_DTYPE, EVO_ERR_ALIGN, EVO_ERR_CUDA, EVO_ERR_ARG, EVO_ERR_DOMAIN = range(7)
EVO_BF16, EVO_F32 = 0, 1

i64 = C.c_int64
vp = C.c_void_p
fp = C.POINTER(C.c_float)


class EvoAttnDesc(C.Structure):
    _fields_ = [("q", vp), ("k", vp), ("v", vp), ("g", vp),
                ("q_sb", i64), ("q_sl", i64), ("k_sb", i64), ("k_sl", i64),
                ("v_sb", i64), ("v_sl", i64), ("g_sb", i64), ("g_sl", i64),
                ("bias", vp), ("bias_s", i64 * 4),
                ("o_gated", vp), ("o_sb", i64), ("o_sl", i64),
                ("o_raw", vp), ("r_sb", i64), ("r_sl", i64),
                ("lse", vp),
                ("B", i64), ("L", i64),
                ("H", C.c_int), ("c", C.c_int),
                ("scale", C.c_float), ("flags", C.c_int)]


# EvoAttnDesc.flags (include/evo.h): per-call kernel-selection hints, 0 = automatic
EVO_ATTN_FORCE_WS, EVO_ATTN_FORCE_FLASH, EVO_ATTN_NO_BIAS_SMEM = 1, 2, 4


class EvoAttnBwdDesc(C.Structure):
    _fields_ = [("f", EvoAttnDesc),
                ("dout", vp), ("do_sb", i64), ("do_sl", i64),
                ("dq", vp), ("dk", vp), ("dv", vp), ("dg", vp),
                ("dq_sb", i64), ("dq_sl", i64), ("dk_sb", i64), ("dk_sl", i64),
                ("dv_sb", i64), ("dv_sl", i64), ("dg_sb", i64), ("dg_sl", i64),
                ("dbias", vp), ("dbias_s", i64 * 4),
                ("workspace", vp), ("workspace_bytes", i64)]


class EvoMat(C.Structure):
    _fields_ = [("ptr", vp), ("dtype", C.c_int), ("batch_stride", i64),
                ("split", i64 * 2), ("stride_hi", i64 * 2), ("stride_lo", i64 * 2)]


# name -> argtypes (restype is int for all compute entry points)
_SIGS = {
    "evo_device_info": [C.POINTER(C.c_int)] * 3,
    "evo_layernorm_fwd": [vp, C.c_int, i64, i64, vp, vp, vp, C.c_int, vp, vp, i64, i64, C.c_float, vp],
    "evo_layernorm_bwd": [vp, C.c_int, vp, C.c_int, i64, i64, vp, vp, vp, vp, C.c_int, vp, vp, vp, i64, i64, vp],
    "evo_layernorm_bwd_colsum": [vp, C.c_int, vp, C.c_int, i64, i64, vp, vp, vp, vp, C.c_int, vp, vp, vp, vp, i64, i64,
                                 vp],
    "evo_layernorm_rowdot_bwd": [vp, C.c_int, vp, vp, vp, C.c_int, vp, i64, vp, vp, vp, vp, vp, vp, vp, i64, i64,
                                 vp],
    "evo_layernorm_rowdot_fwd": [vp, C.c_int, vp, vp, vp, C.c_int, vp, C.c_int, i64, vp, vp, vp, i64, i64,
                                 C.c_float, vp],
    "evo_softmax_fwd": [vp, C.c_int, vp, C.c_int, C.POINTER(i64), vp, C.c_int, C.POINTER(i64), vp, C.c_int,
                        i64, i64, i64, i64, C.c_float, vp],
    "evo_softmax_bwd": [vp, C.c_int, vp, C.c_int, vp, C.c_int, i64, i64, C.c_float, vp],
    "evo_gated_attention_fwd": [C.POINTER(EvoAttnDesc), vp],
    "evo_gated_attention_bwd": [C.POINTER(EvoAttnBwdDesc), vp],
    "evo_residual_layernorm_fwd": [vp, vp, i64, vp, vp, i64, vp, vp, vp, vp, vp, vp, i64, i64, C.c_float, vp],
    "evo_gated_attention_bwd_workspace": [i64, i64, C.c_int, C.c_int, C.c_int],
    "evo_bgemm": [C.POINTER(EvoMat), C.POINTER(EvoMat), C.POINTER(EvoMat), i64, i64, i64, i64,
                  C.c_float, C.c_float, vp],
    "evo_bgemm_workspace": [i64, i64, i64, i64],
    "evo_bgemm_ws": [C.POINTER(EvoMat), C.POINTER(EvoMat), C.POINTER(EvoMat), i64, i64, i64, i64,
                     C.c_float, C.c_float, vp, i64, vp],
    "evo_wgrad_workspace": [i64, i64, i64],
    "evo_wgrad": [vp, i64, vp, i64, vp, i64, i64, i64, i64, vp, i64, vp],
    "evo_opm_fused_supported": [i64, i64, i64, i64, i64],
    "evo_opm_fused_fwd": [vp, vp, vp, vp, i64, vp, i64, i64, i64, i64, i64, C.c_float, vp],
    "evo_opm_bwd_supported": [i64, i64, i64, i64, i64],
    "evo_opm_bwd_workspace": [i64],
    "evo_opm_bwd_factor": [C.c_int, vp, i64, vp, vp, i64, i64, i64, i64, i64, C.c_float, vp, C.c_int, i64, i64, i64,
                           i64, vp, i64, vp],
    "evo_opm_transpose": [vp, i64, i64, i64, i64, i64, vp, vp, vp],
    "evo_tri_gate_fwd": [vp, i64, C.c_int, C.c_int, vp, vp, vp],
    "evo_tri_gate_bwd": [vp, vp, vp, C.c_int, i64, C.c_int, C.c_int, vp, vp, vp],
    "evo_gated_residual_fwd": [vp, vp, i64, vp, vp, i64, vp, C.c_int, i64, i64, vp],
    "evo_gated_residual_bwd": [vp, vp, i64, vp, vp, i64, vp, vp, i64, vp, vp, C.c_int, i64, i64, vp],
    "evo_bias_act_fwd": [vp, vp, i64, i64, C.c_int, C.c_int, vp],
    "evo_bias_act_bwd": [vp, vp, vp, vp, i64, i64, C.c_int, C.c_int, vp],
    "evo_count_nonfinite": [vp, C.c_int, i64, vp, vp],
    "evo_key_bias_grad_cols": [vp, i64, C.c_int, i64, vp, i64, i64, C.c_int, vp],
    "evo_colsum": [vp, C.c_int, i64, i64, i64, vp, vp],
    "evo_gate_mul_fwd": [vp, i64, C.c_int, vp, i64, vp, vp, i64, C.c_int, i64, i64, vp],
}

_lib = None
_lock = threading.Lock()


def exported_symbols():
    return ["evo_version", "evo_last_error_string", *_SIGS.keys()]


def load():
    """Load libevo.so once; raise NativeLibraryMissing if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not built; run `python -m paper_2203_00854_b200.build` "
                "(there is no CPU fallback)")
        try:
            lib = C.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
        lib.evo_version.restype = C.c_char_p
        lib.evo_last_error_string.restype = C.c_char_p
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int64 if name.endswith("_workspace") else C.c_int
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == EVO_OK:
        return
    msg = load().evo_last_error_string().decode(errors="replace")
    if rc == EVO_ERR_SHAPE:
        raise DimensionError(msg)
    if rc == EVO_ERR_DOMAIN:
        raise DomainError(msg)
    raise KernelError(f"libevo error {rc}: {msg}")


# kernels launched per C-ABI call (evo_gated_attention_bwd = prep + main + dq finish [+ dbias reduce])
LAUNCHES = {"evo_gated_attention_bwd": 3, "evo_bgemm_ws": 2, "evo_wgrad": 2, "evo_opm_bwd_factor": 2}


class Instrument:
    """Counts kernel launches per entry point and, for the entry points in ``timed``,
    brackets every call with CUDA events on the launching (current torch) stream so
    the average device duration can be read after a synchronize.  ``work`` carries
    the algorithmic (flops, bytes) of each timed call."""

    def __init__(self, timed=()):
        self.extra = 0
        self.counts: dict[str, int] = {}
        self.timed = set(timed)
        self.records: dict[str, list] = {}

    def launches(self) -> int:
        return sum(LAUNCHES.get(n, 1) * c for n, c in self.counts.items()) + self.extra

    def summary(self):
        out = {}
        for name, recs in self.records.items():
            ms = [a.elapsed_time(b) for a, b, _ in recs]
            fl = sum(w[0] for _, _, w in recs)
            by = sum(w[1] for _, _, w in recs)
            out[name] = {"launches": len(recs), "total_ms": sum(ms), "avg_ms": sum(ms) / max(len(ms), 1),
                         "flops": fl, "bytes": by}
        return out


INSTRUMENT: Instrument | None = None


def call(name: str, *args, work=None, launches=None) -> None:
    """launch a C-ABI entry point; ``launches`` = kernels it enqueues when not the
    static LAUNCHES default (used for the gpu_launches accounting)."""
    inst = INSTRUMENT
    if inst is None:
        check(getattr(load(), name)(*args))
        return
    inst.counts[name] = inst.counts.get(name, 0) + 1
    if launches is not None:
        inst.extra += launches - LAUNCHES.get(name, 1)
    if name in inst.timed:
        import torch
        st = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        check(getattr(load(), name)(*args))
        b.record(st)
        inst.records.setdefault(name, []).append((a, b, work or (0, 0)))
    else:
        check(getattr(load(), name)(*args))


def version() -> str:
    return load().evo_version().decode()
