"""ctypes binding of the C ABI in include/phj.h (libphj.so, sm_100a).

The extension is built in-tree by ``__graft_entry__.build()`` into
``paper_1109_3577_b200/_lib/libphj.so``.  There is no fallback: if the library
is missing or no CUDA device is visible, compute entry points raise.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
# PHJ_LIB_PATH selects an alternative in-tree build (kernel variant A/B runs)
LIB_PATH = os.environ.get("PHJ_LIB_PATH") or os.path.join(HERE, "_lib", "libphj.so")
#: read back per-sweep diagnostics (active blocks per sweep) after each
#: launch -- extra device->host traffic, off unless PHJ_DIAG=1 or set here
DIAG = os.environ.get("PHJ_DIAG", "0") == "1"

PHJ_OK = 0
F64, F32 = 0, 1
RULE_REF, RULE_KRUZKOV = 0, 1
COST_NODE, COST_CTRL = 0, 1
LAB_FIXED, LAB_TARGET, LAB_HARD = -1, -2, -3

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
D = ctypes.c_double


class Grid(ctypes.Structure):
    _fields_ = [("dim", I32), ("periodic", I32 * 3), ("shape", I64 * 3), ("ext", I64 * 3),
                ("strides", I64 * 3), ("lo", D * 3), ("spacing", D * 3), ("ext_lo", D * 3),
                ("k", D)]


class Stencil(ctypes.Structure):
    _fields_ = [("dim", I32), ("n_classes", I32), ("n_controls", I32), ("cost_mode", I32),
                ("n_real", I32), ("pad_", I32),
                ("oct_start", P), ("ctrl", P), ("nzmask", P), ("weights", P), ("cost", P)]


def unroll(dim: int) -> int:
    """PHJ_UNROLL(dim) of the loaded build: octant groups are padded to a
    multiple of this (header default when the library is not built)."""
    try:
        return int(load().phj_unroll(int(dim)))
    except (PhjError, OSError):
        return 4 if dim == 2 else 2


class SolveArgs(ctypes.Structure):
    _fields_ = [("grid", Grid), ("st", Stencil), ("dtype", I32), ("rule", I32),
                ("v0", P), ("v1", P), ("lab", P), ("fmask", P), ("coef", P), ("coef0", D),
                ("n_patches", I32), ("max_sweeps", I32), ("mine", P), ("tol", D),
                ("workspace", P), ("patch_sweeps", P), ("maxch_hist", P), ("evals", P),
                ("info", P), ("ao3_fb", P), ("ao3_mask", P), ("ao3_count", P),
                ("ao3_words", I32), ("options", I32), ("act_tol", D), ("inner_sweeps", I32),
                ("patch_counts", P), ("band_list", P), ("band_off", P), ("n_band", I32),
                ("band_inner", I32), ("stream", P)]


SOLVE_NO_PRUNE = 1  # PHJ_SOLVE_NO_PRUNE
SOLVE_ASYNC = 2  # PHJ_SOLVE_ASYNC
TRANSPORT_ASYNC = 1  # PHJ_TRANSPORT_ASYNC
TRANSPORT_PAIRS = 2  # PHJ_TRANSPORT_PAIRS


class TransportArgs(ctypes.Structure):
    _fields_ = [("grid", Grid), ("st", Stencil), ("phi0", P), ("phi1", P), ("fb", P),
                ("kind", P), ("ent_scratch", P), ("n_colors", I32), ("tol", D), ("act_eps", D),
                ("max_sweeps", I32), ("workspace", P), ("maxch_hist", P), ("color_sweeps", P),
                ("info", P), ("updates", P), ("options", I32), ("inner_sweeps", I32), ("phi_dtype", I32),
                ("seed_flat", P), ("seed_col", P), ("n_seed", ctypes.c_int64),
                ("band_list", P), ("band_off", P), ("n_band", I32), ("stream", P)]


class Shapes(ctypes.Structure):
    _fields_ = [("n_balls", I32), ("balls", P), ("n_planes", I32), ("planes", P),
                ("n_obst_circles", I32), ("obst_circles", P), ("n_obst_boxes", I32),
                ("obst_boxes", P)]


class SpeedModel(ctypes.Structure):
    _fields_ = [("kind", I32), ("c0", D), ("amp", D), ("omega", D * 3), ("ctrl_norm", D),
                ("eps", D), ("speed", P)]


#: every symbol include/phj.h declares (checked by the CPU test suite)
EXPORTS = (
    "phj_solve_workspace_bytes", "phj_unroll", "phj_blocks_total", "phj_block_dims",
    "phj_band_scratch_bytes", "phj_band_count", "phj_band_fill", "phj_solve",
    "phj_fmask_from_labels",
    "phj_fmask_from_hard",
    "phj_feedback", "phj_feedback_allowed", "phj_feedback_slab", "phj_transport", "phj_lift", "phj_argmax_update",
    "phj_argmax_colors", "phj_argmax_colors_t", "phj_count_labels",
    "phj_interpolate_points",
    "phj_assemble_codes",
    "phj_assemble_repair", "phj_assemble_finish", "phj_classify", "phj_node_coef",
    "phj_init_field", "phj_to_kruzkov", "phj_from_kruzkov", "phj_sync_periodic",
    "phj_error_partials", "phj_peak_flops", "phj_last_error", "phj_num_sms",
    "phj_launch_count",
)

_lib: Optional[ctypes.CDLL] = None


class PhjError(RuntimeError):
    """A libphj call failed (message from phj_last_error)."""


def load() -> ctypes.CDLL:
    """Load libphj.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise PhjError(
            f"CUDA extension not built: {LIB_PATH} missing "
            "(run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "phj_solve_workspace_bytes": (I64, [P, I32, I32]),
        "phj_blocks_total": (I64, [P]),
        "phj_block_dims": (ctypes.c_int, [I32, P]),
        "phj_band_scratch_bytes": (I64, [P, I32, I32, I32]),
        "phj_band_count": (ctypes.c_int, [P, I32, I32, P, P, D, I32, I32, I32, P, P, P]),
        "phj_band_fill": (ctypes.c_int, [P, I32, I32, I32, I32, I32, I32, P, P, P, P]),
        "phj_unroll": (I32, [I32]),
        "phj_solve": (ctypes.c_int, [P]),
        "phj_fmask_from_labels": (ctypes.c_int, [P, P, P, P]),
        "phj_fmask_from_hard": (ctypes.c_int, [P, P, P, P]),
        "phj_feedback": (ctypes.c_int, [P, P, I32, I32, P, P, P, P, D, D, P, P, P]),
        "phj_feedback_allowed": (ctypes.c_int, [P, P, I32, I32, P, P, P, P, D, D, P, P, P, I32,
                                                P, P, P]),
        "phj_feedback_slab": (ctypes.c_int, [P, P, I32, I32, P, P, P, P, D, D, P, P, P, I32,
                                             P, P, I32, I32, P]),
        "phj_transport": (ctypes.c_int, [P]),
        "phj_lift": (ctypes.c_int, [P, P, I32, P, P, D, D, I32, P]),
        "phj_argmax_update": (ctypes.c_int, [P, P, I32, P, P, P]),
        "phj_argmax_colors": (ctypes.c_int, [P, P, I32, P, P, P]),
        "phj_argmax_colors_t": (ctypes.c_int, [P, P, I32, I32, D, P, P, P]),
        "phj_count_labels": (ctypes.c_int, [P, ctypes.c_int64, I32, P, P]),
        "phj_interpolate_points": (ctypes.c_int, [P, I32, P, P, ctypes.c_int64, D, D, I32, P, P,
                                                  P]),
        "phj_assemble_codes": (ctypes.c_int, [P, P, P, P, P, P, P]),
        "phj_assemble_repair": (ctypes.c_int, [P, P, P, I32, P, P]),
        "phj_assemble_finish": (ctypes.c_int, [P, P, P, P, P, P]),
        "phj_classify": (ctypes.c_int, [P, P, P, P, P]),
        "phj_node_coef": (ctypes.c_int, [P, P, P, I32, I32, P, P]),
        "phj_init_field": (ctypes.c_int, [P, I32, P, D, P, P]),
        "phj_to_kruzkov": (ctypes.c_int, [I64, I32, P, P, D, P]),
        "phj_from_kruzkov": (ctypes.c_int, [I64, I32, P, P, D, P]),
        "phj_sync_periodic": (ctypes.c_int, [P, I32, P, P]),
        "phj_error_partials": (ctypes.c_int, [I64, P, P, D, D, P, P]),
        "phj_peak_flops": (ctypes.c_int, [I32, I32, P, P]),
        "phj_last_error": (ctypes.c_char_p, []),
        "phj_num_sms": (ctypes.c_int, []),
        "phj_launch_count": (ctypes.c_ulonglong, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != PHJ_OK:
        msg = load().phj_last_error().decode(errors="replace")
        raise PhjError(f"{what}: {msg} (rc={rc})")


def ptr(t) -> Optional[int]:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream
