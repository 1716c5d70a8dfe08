"""ctypes binding of libklnmf.so (include/klnmf.h).

The library is the product: there is no CPU fallback.  If it is missing or
fails to load, every entry point raises ``RuntimeError`` (loudly), and any
CUDA failure inside a call is raised as ``RuntimeError`` carrying
``klnmf_last_error()``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libklnmf.so"

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
D = ctypes.c_double
INT = ctypes.c_int

# Every symbol include/klnmf.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "klnmf_abi_version",
    "klnmf_sizeof_solve_args",
    "klnmf_sizeof_side",
    "klnmf_last_error",
    "klnmf_event_record",
    "klnmf_event_create",
    "klnmf_event_destroy",
    "klnmf_stream_wait",
    "klnmf_ipc_export",
    "klnmf_ipc_open",
    "klnmf_ipc_close",
    "klnmf_chunk_order",
    "klnmf_chunk_perm4",
    "klnmf_sweep_range",
    "klnmf_sweep_range_passes",
    "klnmf_kkt_violation",
    "klnmf_mu_update_range",
    "klnmf_kl_data_term",
    "klnmf_row_sums",
    "klnmf_solve_exact",
    "klnmf_kkt_exact",
    "klnmf_mu_update_dev",
    "klnmf_solve_fast",
    "klnmf_prepare_fast",
    "klnmf_fast_kernel_count",
    "klnmf_fast_kernel_info",
    "klnmf_fast_kernel_fits",
    "klnmf_coop_info",
    "klnmf_solve_coop",
    "klnmf_row_sums_exact",
    "klnmf_row_sums_fast",
    "klnmf_chunk_masks",
    "klnmf_layout_to_device",
    "klnmf_layout_to_device_f32src",
    "klnmf_layout_from_device",
    "klnmf_layout_from_device_f32",
    "klnmf_transpose",
    "klnmf_coo_to_csc",
    "klnmf_bucketize",
    "klnmf_init_t",
    "klnmf_kl_data_term_dev",
    "klnmf_kl_data_term_t",
    "klnmf_kl_data_term_t_mapped",
    "klnmf_factor_stats",
    "klnmf_upload_i64_as_i32",
    "klnmf_upload_f64_as_f32",
    "klnmf_host_minmax_f64",
    "klnmf_upload_f64",
    "klnmf_download_f32_as_f64",
    "klnmf_download_f64",
    "klnmf_mm_header",
    "klnmf_mm_read",
    "klnmf_synth_build",
    "klnmf_synth_fetch",
)

STATS_LEN = 4
MM_FORMAT_ERROR = 2
ORDER_SHARED, ORDER_COUNTER = 0, 1
STAT_CAP_HITS, STAT_DEGENERATE, STAT_INNER_ITERS, STAT_PASSES = range(4)


class Side(ctypes.Structure):
    """klnmf_side_t"""

    _fields_ = [
        ("ptr", P),
        ("idx", P),
        ("val", P),
        ("n_fix", I64),
        ("n_mov", I64),
        ("nnz", I64),
    ]


class SolveArgs(ctypes.Structure):
    """klnmf_solve_args_t"""

    _fields_ = [
        ("side", Side),
        ("fixed", P),
        ("moving", P),
        ("sum_pos", P),
        ("perm_in", P),
        ("perm_out", P),
        ("nat_pos", P),
        ("items", P),
        ("n_items", I64),
        ("tmap", P),
        ("t_in", P),
        ("t_out", P),
        ("scratch", P),
        ("r", I32),
        ("rp", I32),
        ("alpha", D),
        ("beta", D),
        ("eps_grad", D),
        ("eps_x", D),
        ("eps_div", D),
        ("inner_cap", I64),
        ("stats", P),
        ("order_mode", I32),
        ("order_side", ctypes.c_uint32),
        ("order_seed", ctypes.c_uint64),
        ("order_iter", P),
        ("max_passes", I32),
        ("n_peers", I32),
        ("peer_moving", P),
        ("peer_t", P),
        ("t_scatter", I32),
        ("fixed_mask", P),
        ("slice_words", P),
    ]


_SIGS = {
    "klnmf_abi_version": ([], INT),
    "klnmf_sizeof_solve_args": ([], INT),
    "klnmf_sizeof_side": ([], INT),
    "klnmf_last_error": ([], ctypes.c_char_p),
    "klnmf_event_record": ([P, P, INT], INT),
    "klnmf_event_create": ([ctypes.POINTER(P)], INT),
    "klnmf_event_destroy": ([P], INT),
    "klnmf_stream_wait": ([P, P], INT),
    "klnmf_ipc_export": ([P, P, ctypes.POINTER(I64)], INT),
    "klnmf_ipc_open": ([P, ctypes.POINTER(P)], INT),
    "klnmf_ipc_close": ([P], INT),
    "klnmf_chunk_order": ([ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, I32, P], INT),
    "klnmf_chunk_perm4": ([ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, I32, P], INT),
    "klnmf_sweep_range": ([P, P, P, P, P, P, I64, I64, P, D, D, D, D, D, I64, I64, I64, I64, P], INT),
    "klnmf_sweep_range_passes": ([P, P, P, P, P, P, I64, I64, P, D, D, D, D, D, I64, I64, I64, I64, I64, P], INT),
    "klnmf_kkt_violation": ([P, P, P, P, P, P, D, D, D, D, D, I64, I64, I64, P], INT),
    "klnmf_mu_update_range": ([P, P, P, P, P, P, D, I64, I64, I64, I64, I64], INT),
    "klnmf_kl_data_term": ([P, P, P, P, P, D, I64, I64, I64, P], INT),
    "klnmf_row_sums": ([P, I64, I64, P], INT),
    "klnmf_solve_exact": ([ctypes.POINTER(SolveArgs), P], INT),
    "klnmf_kkt_exact": ([ctypes.POINTER(SolveArgs), P, P], INT),
    "klnmf_mu_update_dev": ([ctypes.POINTER(Side), P, P, P, I32, I32, D, P, I64, P, P], INT),
    "klnmf_solve_fast": ([ctypes.POINTER(SolveArgs), INT, P], INT),
    "klnmf_prepare_fast": ([I32], INT),
    "klnmf_fast_kernel_count": ([], INT),
    "klnmf_fast_kernel_info": ([INT, ctypes.POINTER(I64), ctypes.POINTER(I32), ctypes.POINTER(I32)], INT),
    "klnmf_fast_kernel_fits": ([INT, I32, ctypes.POINTER(I32)], INT),
    "klnmf_coop_info": ([I32, ctypes.POINTER(I64), ctypes.POINTER(I32), ctypes.POINTER(I64)], INT),
    "klnmf_solve_coop": ([ctypes.POINTER(SolveArgs), P, I32, I32, P, I64, P], INT),
    "klnmf_row_sums_exact": ([P, I64, I32, I32, P, P], INT),
    "klnmf_row_sums_fast": ([P, I64, I32, I32, P, P], INT),
    "klnmf_chunk_masks": ([P, I64, I32, I32, P, P], INT),
    "klnmf_layout_to_device": ([P, I64, I64, P, I32, P, INT, P], INT),
    "klnmf_layout_to_device_f32src": ([P, I64, I64, P, I32, P, P], INT),
    "klnmf_layout_from_device": ([P, I64, I64, P, I32, INT, P, P], INT),
    "klnmf_layout_from_device_f32": ([P, I64, I64, P, I32, P, P], INT),
    "klnmf_transpose": ([P, P, P, INT, I64, I64, I64, P, P, P, P, P, P], INT),
    "klnmf_coo_to_csc": ([P, P, P, INT, I64, I64, I64, P, P, P, P, P], INT),
    "klnmf_bucketize": ([P, I64, I64, P, INT, P, P, P], INT),
    "klnmf_init_t": ([ctypes.POINTER(Side), P, P, I32, P, P, I32, P, P], INT),
    "klnmf_kl_data_term_dev": ([ctypes.POINTER(Side), P, P, I32, P, P, I32, INT, D, P, P], INT),
    "klnmf_kl_data_term_t": ([P, P, I64, D, P, P], INT),
    "klnmf_kl_data_term_t_mapped": ([P, P, P, I64, D, P, P], INT),
    "klnmf_factor_stats": ([P, I64, I32, I32, INT, P, P], INT),
    "klnmf_upload_i64_as_i32": ([P, I64, P, P], INT),
    "klnmf_upload_f64_as_f32": ([P, I64, P, P], INT),
    "klnmf_host_minmax_f64": ([P, I64, P, P], INT),
    "klnmf_upload_f64": ([P, I64, P, P], INT),
    "klnmf_download_f32_as_f64": ([P, I64, P, P], INT),
    "klnmf_download_f64": ([P, I64, P, P], INT),
    "klnmf_mm_header": ([ctypes.c_char_p, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)], INT),
    "klnmf_mm_read": ([ctypes.c_char_p, I64, P, P, P], INT),
    "klnmf_synth_build": ([ctypes.c_uint64, I64, I64, I32, D, INT, D, D, INT, ctypes.POINTER(I64), P,
                           ctypes.POINTER(P), ctypes.POINTER(P), P], INT),
    "klnmf_synth_fetch": ([P, P, I64, INT, P, P, P], INT),
}

_lib = None


def load(path: Path | None = None):
    """Load libklnmf.so once; raises RuntimeError if it is absent or broken."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("KLNMF_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"libklnmf.so not found at {p}: build it with `python -m paper_1604_04026_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.klnmf_abi_version() != 1:
        raise RuntimeError("libklnmf.so ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().klnmf_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def coop_info(rp: int):
    """(entries per CTA, CTAs of the cooperative long-row kernel, sync bytes per row group)."""
    lib = load()
    e, n, b = I64(), I32(), I64()
    check(lib.klnmf_coop_info(int(rp), ctypes.byref(e), ctypes.byref(n), ctypes.byref(b)), "klnmf_coop_info")
    return e.value, n.value, b.value


def fast_kernels(rp: int | None = None):
    """[(kernel_id, capacity, lanes, npl)] of the fp32-mode bucket kernels
    (with rp: only those whose shared-memory layout fits at that padded rank;
    the long-row kernels always do)."""
    lib = load()
    out = []
    for k in range(lib.klnmf_fast_kernel_count()):
        if rp is not None:
            fits = I32()
            check(lib.klnmf_fast_kernel_fits(k, int(rp), ctypes.byref(fits)), "klnmf_fast_kernel_fits")
            if not fits.value:
                continue
        cap, lanes, npl = I64(), I32(), I32()
        check(lib.klnmf_fast_kernel_info(k, ctypes.byref(cap), ctypes.byref(lanes), ctypes.byref(npl)),
              "klnmf_fast_kernel_info")
        out.append((k, cap.value, lanes.value, npl.value))
    return out
