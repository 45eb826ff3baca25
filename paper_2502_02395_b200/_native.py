"""ctypes binding of libh2ulv_b200.so (the C ABI in include/h2ulv_b200.h).

There is deliberately no fallback: if the library cannot be loaded or no
CUDA device is present, `lib()` raises NativeUnavailableError.  Descriptor
arrays are numpy structured arrays whose layout mirrors the C structs
byte for byte (checked against the struct sizes at import).
"""

import ctypes
import os

import numpy as np

from .errors import NativeUnavailableError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("H2G_LIB_PATH") or os.path.join(HERE, "libh2ulv_b200.so")   # override: A/B builds

# --- descriptor layouts (must match include/h2ulv_b200.h) -------------------------------
GEMM_DT = np.dtype([("A", "<u8"), ("B", "<u8"), ("C", "<u8"), ("M", "<i4"), ("N", "<i4"), ("K", "<i4"),
                    ("lda", "<i4"), ("ldb", "<i4"), ("ldc", "<i4"), ("tile_start", "<i4"), ("flags", "<i4"),
                    ("alpha", "<f8"), ("beta", "<f8")])
GEMM_EXT_DT = np.dtype([("Cin", "<u8"), ("sgn", "<u8"), ("ldcin", "<i4"), ("remap_k", "<i4")])
CHOLP_DT = np.dtype([("H", "<u8"), ("Linv", "<u8"), ("ldh", "<i4"), ("ldl", "<i4"), ("n", "<i4"), ("p", "<i4"),
                     ("b", "<i4"), ("npd_slot", "<i4"), ("tile_start", "<i4"), ("pad_", "<i4")])
ROWS_DT = np.dtype([("Lb", "<u8"), ("Xin", "<u8"), ("Xout", "<u8"), ("Linv", "<u8"), ("pad0_", "<u8"),
                    ("rows", "<i4"), ("cols", "<i4"), ("q_begin", "<i4"), ("q_end", "<i4"), ("ldlb", "<i4"),
                    ("ldx", "<i4"), ("tile_start", "<i4"), ("pad1_", "<i4")])
COPY_DT = np.dtype([("src", "<u8"), ("dst", "<u8"), ("rows", "<i4"), ("cols", "<i4"), ("lds", "<i4"),
                    ("ldd", "<i4"), ("mode", "<i4"), ("tile_start", "<i4")])
GEMV_TERM_DT = np.dtype([("A", "<u8"), ("x", "<u8"), ("lda", "<i4"), ("trans", "<i4"), ("K", "<i4"),
                         ("pad_", "<i4")])
GEMV_OUT_DT = np.dtype([("y", "<u8"), ("y2", "<u8"), ("init", "<u8"), ("m", "<i4"), ("split", "<i4"),
                        ("term_begin", "<i4"), ("term_end", "<i4"), ("flags", "<i4"), ("chunk_start", "<i4")])
TRSV_DT = np.dtype([("L", "<u8"), ("Linv", "<u8"), ("x", "<u8"), ("n", "<i4"), ("ldl", "<i4")])
QRP_DT = np.dtype([("Z", "<u8"), ("V", "<u8"), ("tau", "<u8"), ("T", "<u8"), ("n", "<i4"), ("ldz", "<i4"),
                   ("p", "<i4"), ("b", "<i4")])
BASIS_DT = np.dtype([("Q", "<u8"), ("Z", "<u8"), ("qfull", "<u8"), ("frame", "<u8"), ("n", "<i4"), ("k", "<i4"),
                     ("ldz", "<i4"), ("pad_", "<i4")])
KBLOCK_DT = np.dtype([("rows", "<u8"), ("cols", "<u8"), ("out", "<u8"), ("m", "<i4"), ("n", "<i4"),
                      ("ldo", "<i4"), ("tile_start", "<i4")])
SYMCHECK_DT = np.dtype([("A", "<u8"), ("n", "<i4"), ("lda", "<i4")])
TRIINV_DT = np.dtype([("L", "<u8"), ("Linv", "<u8"), ("n", "<i4"), ("ldl", "<i4"), ("tile_start", "<i4"),
                      ("status_slot", "<i4")])
CHOLBOX_DT = np.dtype([("H", "<u8"), ("Linv", "<u8"), ("Q", "<u8"), ("R", "<u8"), ("n", "<i4"), ("r", "<i4"),
                       ("ldh", "<i4"), ("npd_slot", "<i4")])
XFORM_DT = np.dtype([("Q", "<u8"), ("x", "<u8"), ("y1", "<u8"), ("y2", "<u8"), ("n", "<i4"), ("split", "<i4"),
                     ("ldq", "<i4"), ("tile_start", "<i4")])
XFORMN_DT = np.dtype([("Q", "<u8"), ("xr", "<u8"), ("xs", "<u8"), ("out", "<u8"), ("n", "<i4"), ("r", "<i4"),
                      ("ldq", "<i4"), ("tile_start", "<i4")])
STEP_DT = np.dtype([("kind", "<i4"), ("count", "<i4"), ("grid", "<i4"), ("arg", "<i4"), ("descs", "<u8"),
                    ("map", "<u8"), ("npd", "<u8"), ("aux", "<u8"), ("d0", "<f8"), ("d1", "<f8"),
                    ("lane", "<i4"), ("wait_ev", "<i4"), ("rec_ev", "<i4"), ("pad_", "<i4")])

assert GEMM_DT.itemsize == 72 and GEMM_EXT_DT.itemsize == 24 and COPY_DT.itemsize == 40 and CHOLP_DT.itemsize == 48 and ROWS_DT.itemsize == 72
assert GEMV_TERM_DT.itemsize == 32 and GEMV_OUT_DT.itemsize == 48 and TRSV_DT.itemsize == 32
assert SYMCHECK_DT.itemsize == 16 and TRIINV_DT.itemsize == 32 and CHOLBOX_DT.itemsize == 48 and XFORM_DT.itemsize == 48 and XFORMN_DT.itemsize == 48
assert QRP_DT.itemsize == 48 and BASIS_DT.itemsize == 48 and KBLOCK_DT.itemsize == 40 and STEP_DT.itemsize == 80

NPD_STATUS_DT = np.dtype([("failed", "<i4"), ("pivot", "<i4"), ("level", "<i4"), ("box", "<i4")])
H2G_ENPD = 4
STEP = {"GEMM_NN": 0, "GEMM_NT": 1, "GEMM_TN": 2, "GEMM_TT": 3, "COPY": 5, "MEMCPY": 6,
        "QR_PANEL": 7, "BASIS": 8, "GEMV": 9, "TRSV": 10, "KBLOCK": 11, "NOP": 12, "CHOL_PANEL": 13, "TRSM_ROWS": 14,
        "SYMCHECK": 15, "TRIINV": 16, "CHOL_BOX": 17, "XFORM_T": 18, "XFORM_N": 19}
GEMM_LOWER = 1
GEMV_PLUS = 1
GEMV_SPLIT = 2
GEMM_TILE = {2: 64, 7: 64, 9: 32, 11: 64}  # tile edge per tile_cfg (gemm.cu: Cfg64b, Cfg64m3, Cfg32, Cfg64w8)
COPY_TILE = 64
PANEL_WIDTH = 64
GEMV_CHUNK = 64    # output rows per CTA of h2g_gemv_grouped (csrc/solve.cu GV_CHUNK)
QR_PANEL_WIDTH = 32

EXPORTS = ["h2g_gemm_tiles", "h2g_gemm_grouped", "h2g_gemm_grouped_ext", "h2g_gemm_grouped_split", "h2g_gemm_split_workspace", "h2g_chol_panel_tiles", "h2g_chol_panel", "h2g_chol_panel_sync", "h2g_chol_panel_fused_max", "h2g_trsm_rows", "h2g_copy_tiles", "h2g_block_copy",
           "h2g_gemv_grouped", "h2g_trsv_batched", "h2g_qr_panel", "h2g_basis_finish", "h2g_kernel_blocks",
           "h2g_run_program", "h2g_run_program_timed", "h2g_exec_ctx_create", "h2g_exec_ctx_destroy",
           "h2g_graph_capture", "h2g_graph_launch", "h2g_graph_destroy", "h2g_abi_version",
           "h2g_last_error", "h2g_device_sm_count", "h2g_sym_check", "h2g_tri_inv", "h2g_chol_box", "h2g_xform_t", "h2g_xform_n", "h2g_xform_n_rows",
           "h2g_session_create", "h2g_session_factor_async", "h2g_session_status", "h2g_session_destroy",
           "h2g_direct_matvec_workspace", "h2g_direct_matvec"]

_LIB = None


def load_library(path=LIB_PATH):
    """Load the shared library without touching the GPU (CPU-safe)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise NativeUnavailableError(
            f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i32 = ctypes.c_void_p, ctypes.c_int
    sig = {
        "h2g_gemm_tiles": (i32, [i32, i32, i32, i32]),
        "h2g_gemm_grouped": (i32, [i32, i32, i32, vp, vp, i32, vp]),
        "h2g_gemm_grouped_ext": (i32, [i32, i32, i32, vp, vp, vp, i32, vp]),
        "h2g_gemm_grouped_split": (i32, [i32, i32, i32, vp, vp, i32, i32, vp, vp]),
        "h2g_gemm_split_workspace": (ctypes.c_size_t, [i32, i32]),
        "h2g_chol_panel_tiles": (i32, [i32, i32, i32]),
        "h2g_chol_panel": (i32, [vp, i32, vp, i32, vp, vp]),
        "h2g_chol_panel_sync": (i32, [vp, i32, vp, i32, vp, vp, vp]),
        "h2g_chol_panel_fused_max": (i32, []),
        "h2g_trsm_rows": (i32, [vp, vp, i32, vp]),
        "h2g_copy_tiles": (i32, [i32, i32]),
        "h2g_block_copy": (i32, [vp, vp, i32, vp]),
        "h2g_gemv_grouped": (i32, [vp, i32, vp, vp, i32, i32, vp]),
        "h2g_trsv_batched": (i32, [vp, i32, i32, i32, vp]),
        "h2g_qr_panel": (i32, [vp, i32, i32, vp]),
        "h2g_basis_finish": (i32, [vp, i32, vp]),
        "h2g_kernel_blocks": (i32, [vp, vp, i32, vp, i32, ctypes.c_double, ctypes.c_double, vp, vp]),
        "h2g_run_program": (i32, [vp, i32, vp, vp]),
        "h2g_exec_ctx_create": (i32, [i32, ctypes.POINTER(vp)]),
        "h2g_exec_ctx_destroy": (i32, [vp]),
        "h2g_run_program_timed": (i32, [vp, i32, vp, vp]),
        "h2g_graph_capture": (i32, [vp, i32, vp, vp, ctypes.POINTER(vp)]),
        "h2g_graph_launch": (i32, [vp, vp]),
        "h2g_graph_destroy": (i32, [vp]),
        "h2g_abi_version": (i32, []),
        "h2g_last_error": (ctypes.c_char_p, []),
        "h2g_device_sm_count": (i32, []),
        "h2g_sym_check": (i32, [vp, i32, vp, vp]),
        "h2g_tri_inv": (i32, [vp, vp, i32, vp, vp]),
        "h2g_chol_box": (i32, [vp, i32, vp, vp]),
        "h2g_xform_t": (i32, [vp, vp, i32, i32, i32, vp]),
        "h2g_xform_n": (i32, [vp, vp, i32, i32, i32, i32, vp]),
        "h2g_xform_n_rows": (i32, []),
        "h2g_session_create": (i32, [vp, i32, i32, vp, i32, vp, vp, ctypes.POINTER(vp)]),
        "h2g_session_factor_async": (i32, [vp, vp]),
        "h2g_session_status": (i32, [vp, vp, vp]),
        "h2g_session_destroy": (i32, [vp]),
        "h2g_direct_matvec_workspace": (ctypes.c_int64, [ctypes.c_int64]),
        "h2g_direct_matvec": (i32, [vp, vp, vp, ctypes.c_int64, i32, i32, ctypes.c_double, ctypes.c_double, vp,
                                    ctypes.c_int64, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.h2g_abi_version() != 1:
        raise NativeUnavailableError("libh2ulv_b200.so ABI version mismatch")
    _LIB = lib
    return lib


def lib():
    """The library, after checking that a CUDA device is usable."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailableError("no CUDA device: the H2-ULV path runs only on the GPU (no CPU fallback)")
    return load_library()


def ctypes_void_p():
    return ctypes.c_void_p


def check(rc, what="h2g call"):
    if rc != 0:
        msg = load_library().h2g_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
