"""ctypes binding of libbamg_sm100.so (the C ABI declared in include/bamg_sm100.h).

There is deliberately no fallback: if the library is missing, or no CUDA
device is visible, every entry point raises `BamgUnavailable`.  The product
path never computes on the host.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
import os as _os
LIB_PATH = Path(_os.environ.get("BAMG_LIB_PATH", str(_PKG / "libbamg_sm100.so")))


class BamgUnavailable(RuntimeError):
    """The sm_100a engine cannot run here (library not built or no GPU)."""


class BamgError(RuntimeError):
    """A CUDA or argument error reported by the engine."""


class CSR(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("rowptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p),
                ("packed", C.c_void_p), ("dict", C.c_void_p), ("pslice", C.c_void_p), ("pwords", C.c_int64),
                ("ptiles", C.c_void_p), ("st_w", C.c_int32), ("st_diag", C.c_int32),
                ("st_delta", C.c_int32 * 8), ("st_val", C.c_double * 8), ("st_d", C.c_double),
                ("st_rd", C.c_double), ("st_tiles", C.c_int64)]


P = C.c_void_p
PCSR = C.POINTER(CSR)
I32, I64, F64 = C.c_int32, C.c_int64, C.c_double
PI64 = C.POINTER(C.c_int64)
PINT = C.POINTER(C.c_int)
PF64 = C.POINTER(C.c_double)

# name -> argtypes (all return int unless listed in _RESTYPES)
_SIGS = {
    "bamg_ctx_create": [C.c_int, P, C.POINTER(P)],
    "bamg_ctx_destroy": [P],
    "bamg_last_error": [P],
    "bamg_version": [],
    "bamg_launch_count": [P],
    "bamg_sync_count": [P],
    "bamg_sync": [P],
    "bamg_prof_enable": [P, C.c_uint],
    "bamg_prof_read": [P, C.c_int, PF64, PI64, PF64],
    "bamg_fp64_peak": [P, C.c_int, PF64],
    "bamg_dgemm": [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, F64, P, C.c_int, P, C.c_int, F64, P, C.c_int],
    "bamg_trace_enable": [P, C.c_int],
    "bamg_trace_dump": [P, C.c_char_p, I64],
    "bamg_trace_timeline": [P, C.c_char_p, I64],
    "bamg_trace_position": [P],
    "bamg_spmv": [P, PCSR, P, P],
    "bamg_spmm": [P, PCSR, P, P, C.c_int],
    "bamg_csr_pack_plan": [P, PCSR, P, P, PINT, PI64],
    "bamg_csr_pack_fill": [P, PCSR, P, P, C.c_int, P],
    "bamg_csr_transpose": [P, PCSR, P, P, P],
    "bamg_sym_pattern_count": [P, PCSR, PCSR, P, PI64],
    "bamg_sym_pattern_fill": [P, PCSR, PCSR, P, P],
    "bamg_diag": [P, PCSR, P],
    "bamg_count_nonpositive": [P, P, I64, PI64],
    "bamg_chain_lattice_count": [P, C.c_int, C.c_int, F64, F64, F64, P, P, PI64],
    "bamg_chain_lattice_fill": [P, C.c_int, C.c_int, F64, F64, F64, P, P, P],
    "bamg_chain_planar_count": [P, P, I64, C.c_int, P, PI64],
    "bamg_uniform_draws": [P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, I64, P, P],
    "bamg_chain_planar_fill": [P, P, I64, C.c_int, P, P, P],
    "bamg_spgemm_count": [P, PCSR, PCSR, C.c_int, P, PI64],
    "bamg_spgemm_fill": [P, PCSR, PCSR, C.c_int, P, P, P],
    "bamg_spgemm_count_slot": [P, PCSR, PCSR, C.c_int, P, C.c_int],
    "bamg_spgemm_count_wait": [P, C.c_int, P, PI64],
    "bamg_spgemm_fill_slot": [P, PCSR, PCSR, C.c_int, P, P, P, C.c_int],
    "bamg_degenerate_rows": [P, PCSR, P, P],
    "bamg_jacobi": [P, PCSR, P, P, P, P, P, P, C.c_int, F64, P],
    "bamg_selftest_div": [P, I64, C.c_uint64, C.c_int, P],
    "bamg_col_norms": [P, P, I64, C.c_int, P],
    "bamg_col_dots": [P, P, P, I64, C.c_int, P],
    "bamg_col_scale_div": [P, P, I64, C.c_int, P],
    "bamg_col_fill": [P, P, I64, C.c_int, C.c_int, F64],
    "bamg_gather_rows": [P, P, P, I64, C.c_int, P],
    "bamg_smooth_block": [P, PCSR, PCSR, PCSR, PCSR, P, P, P, P, P, P, C.c_int, C.c_int, F64,
                          C.c_int, C.c_int, C.c_int],
    "bamg_refresh_sigmas": [P, PCSR, PCSR, PCSR, P, P, P, P, C.c_int],
    "bamg_test_weights": [P, PCSR, P, I64, C.c_int, C.c_int, P, P],
    "bamg_fit_set_row_range": [P, I64, I64],
    "bamg_csr_stencil": [P, PCSR, P, PCSR],
    "bamg_fit_rows": [P, PCSR, P, P, P, I64, C.c_int, C.c_int, C.c_int, F64, C.c_int, C.c_int,
                      F64, P, P, P, PI64],
    "bamg_fit_rows_csr": [P, PCSR, P, P, P, I64, C.c_int, C.c_int, C.c_int, F64, C.c_int, C.c_int,
                          F64, P, P, P, P, PI64, PI64],
    "bamg_fit_rows_csr_slot": [P, PCSR, P, P, P, I64, C.c_int, C.c_int, C.c_int, F64, C.c_int, C.c_int,
                               F64, P, P, P, P, C.c_int],
    "bamg_fit_rows_wait": [P, C.c_int, P, PI64, PI64],
    "bamg_rows_count": [P, P, P, I64, C.c_int, P, PI64],
    "bamg_rows_fill": [P, P, P, P, I64, C.c_int, P, P, P],
    "bamg_axis_ranks": [P, P, I64, P, PI64],
    "bamg_rerank": [P, P, P, I64, I64, P, PI64],
    "bamg_even_mask": [P, C.POINTER(P), C.c_int, I64, P],
    "bamg_split_from_mask": [P, P, I64, P, P, P, PI64],
    "bamg_cr_pass": [P, PCSR, PCSR, P, P, P, I64, C.c_int, F64, F64, C.c_int, PI64, PI64],
    "bamg_count_empty_rows": [P, PCSR, PI64],
    "bamg_permute_cols": [P, P, I64, C.c_int, C.POINTER(C.c_int32), P],
    "bamg_csr_to_dense": [P, PCSR, P, C.c_int, C.c_int],
    "bamg_dense_pinv": [P, P, C.c_int, F64, P],
    "bamg_fov_points": [P, P, C.c_int, C.c_int, F64, P, C.POINTER(C.c_int)],
    "bamg_eigvals": [P, P, C.c_int, P, P],
    "bamg_range_basis": [P, P, C.c_int, F64, P, P, C.POINTER(C.c_int)],
    "bamg_coarsest_triplets": [P, P, P, P, C.c_int, C.c_int, P, P, P],
    "bamg_coarsest_triplets_pinv": [P, P, P, P, C.c_int, C.c_int, P, P, P, P, P],
    "bamg_hier_create": [P, C.c_int, C.POINTER(P)],
    "bamg_hier_destroy": [P],
    "bamg_hier_set_level": [P, C.c_int, PCSR, P, P, PCSR, PCSR],
    "bamg_hier_set_coarsest": [P, P, C.c_int],
    "bamg_hier_set_coarsest_lu": [P, P, C.c_int],
    "bamg_coarsest_triplets_ex": [P, P, P, P, C.c_int, C.c_int, P, P, P, P, P, P],
    "bamg_coarse_lu_apply": [P, P, P, P],
    "bamg_coarse_lu_destroy": [P, P],
    "bamg_band_sweep_probe": [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, PF64],
    "bamg_coarsest_band": [P, PCSR, PCSR, PCSR, PCSR, C.c_int, P, P, P, P, P],
    "bamg_hier_set_smoother": [P, F64, C.c_int, C.c_int],
    "bamg_vcycle": [P, P, P, P],
    "bamg_gmres": [P, PCSR, P, P, P, P, C.c_int, C.c_int, F64, C.c_int, PINT, PF64, PINT],
    "bamg_dense_gemv": [P, P, C.c_int, P, P],
    "bamg_sign_fix_l1": [P, P, I64, C.c_int, P, C.c_int],
    "bamg_residual": [P, PCSR, P, P, P],
    "bamg_addmv": [P, PCSR, P, P, P],
    "bamg_jacobi_zero": [P, I64, P, P, P, F64, P],
    "bamg_dense_gemv_rows": [P, P, C.c_int, P, P],
    "bamg_mdot": [P, P, C.c_int, P, I64, P],
    "bamg_mupdate": [P, P, C.c_int, P, P, I64, P],
    "bamg_combine": [P, P, C.c_int, P, P, P, I64, P],
    "bamg_cgs_dots": [P, P, C.c_int, P, I64, P],
    "bamg_cgs_update": [P, P, C.c_int, P, P, P, P, P, F64, C.c_int, I64, P, P, P],
}
_RESTYPES = {"bamg_last_error": C.c_char_p, "bamg_launch_count": C.c_int64, "bamg_sync_count": C.c_int64,
             "bamg_trace_position": C.c_int64}

_lock = threading.Lock()
_lib = None
_gpu_lib = None  # set once a GPU was confirmed: the hot-path fast return of lib()
_ctx = {}


def exported_symbols():
    return list(_SIGS)


def load_library(require_gpu: bool = False):
    """dlopen the engine.  `require_gpu` additionally demands a CUDA device."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise BamgUnavailable(
                    f"{LIB_PATH} is not built; run `python -m paper_1402_4005_b200.build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
            missing = []
            for name, args in _SIGS.items():
                try:
                    fn = getattr(lib, name)
                except AttributeError:
                    missing.append(name)
                    continue
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, C.c_int)
            lib.missing_symbols = missing
            _lib = lib
    if require_gpu and not torch.cuda.is_available():
        raise BamgUnavailable("no CUDA device visible: the sm_100a engine has no CPU fallback")
    return _lib


def lib():
    global _gpu_lib
    if _gpu_lib is None:
        _gpu_lib = load_library(require_gpu=True)
    return _gpu_lib


def ctx(device: int | None = None):
    """Per-device engine context bound to torch's current stream at first use."""
    L = lib()
    dev = torch.cuda.current_device() if device is None else int(device)
    key = dev
    c = _ctx.get(key)
    if c is not None:
        return c
    if key not in _ctx:
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            out = P()
            rc = L.bamg_ctx_create(dev, P(stream), C.byref(out))
            if rc != 0:
                raise BamgError(f"bamg_ctx_create failed ({rc})")
            _ctx[key] = out
    return _ctx[key]


def check(rc: int, what: str, c=None):
    """Raise on negative codes (-2 argument errors as ValueError, like the
    reference); return the non-negative status otherwise."""
    if rc < 0:
        msg = lib().bamg_last_error(c if c is not None else ctx())
        text = f"{what}: {msg.decode() if msg else rc}"
        if rc == -2:
            raise ValueError(text)
        raise BamgError(text)
    return rc


# BAMG_SLOWCALL_MS=<ms>: report engine calls whose host wall time exceeds
# the threshold (development aid for host-side stalls)
_SLOW_MS = float(_os.environ.get("BAMG_SLOWCALL_MS", "0") or 0)


# BAMG_NVTX=1: one NVTX range per engine call (named after the C ABI entry),
# nested inside the per-level phase ranges bootstrap.py / solver.py push
# (tracing).  Off by default: the push/pop pair costs ~1 us per call.
NVTX = bool(int(_os.environ.get("BAMG_NVTX", "0") or 0))


def nvtx_push(name: str) -> None:
    if NVTX:
        torch.cuda.nvtx.range_push(name)


def nvtx_pop() -> None:
    if NVTX:
        torch.cuda.nvtx.range_pop()


def call(name: str, *args):
    c = ctx()
    if NVTX:
        torch.cuda.nvtx.range_push(name)
        try:
            return check(getattr(lib(), name)(c, *args), name, c)
        finally:
            torch.cuda.nvtx.range_pop()
    if _SLOW_MS > 0:
        import time
        t0 = time.perf_counter()
        rc = getattr(lib(), name)(c, *args)
        dt = (time.perf_counter() - t0) * 1e3
        if dt > _SLOW_MS:
            print(f"[bamg slow call] {name} {dt:.1f} ms", flush=True)
        return check(rc, name, c)
    rc = getattr(lib(), name)(c, *args)
    return check(rc, name, c)


def launches() -> int:
    return int(lib().bamg_launch_count(ctx()))


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return P(t.data_ptr())
