"""ctypes binding of ``libmeshplan_b200.so`` (the C ABI in include/meshplan_b200.h).

This is the only module that talks to the native library.  Loading is lazy
and loud: if the library is missing, every device entry point raises
``DeviceError`` -- there is no CPU fallback anywhere in the package.
Device arrays are passed as raw pointers taken from torch tensors, and the
CUDA stream as a ``void*`` (torch's current stream by default).
"""

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import DeviceError, raise_for_status

LIB_PATH = Path(os.environ.get("MESHPLAN_B200_LIB", Path(__file__).resolve().parent / "lib" / "libmeshplan_b200.so"))

MP_F64, MP_F32, MP_I64, MP_I32 = 0, 1, 2, 3
MP_AOS, MP_SOA = 0, 1
MP_SCHED_COLOUR, MP_SCHED_DATAFLOW, MP_SCHED_PULL = 0, 1, 4
OPS = {"flux": 0, "flux-noread": 1, "scatter8": 2, "face-flux": 3, "face-flux-heavy": 4}
#: per device op: (arity, indirect-read components consumed, direct components
#: consumed, increment components) -- the functor shapes of csrc/mp_ops.cuh
OP_SHAPES = {"flux": (2, 4, 1, 4), "flux-noread": (2, 0, 2, 4), "scatter8": (8, 0, 4, 3),
             "face-flux": (2, 5, 1, 5), "face-flux-heavy": (2, 7, 2, 5)}
DTYPES = {"f64": MP_F64, "f32": MP_F32, "i64": MP_I64, "i32": MP_I32}
LAYOUTS = {"aos": MP_AOS, "soa": MP_SOA}

c_i32, c_i64, c_u32, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p


class MpLoop(ctypes.Structure):
    _fields_ = [
        ("op", c_i32), ("unit", c_i32), ("dtype", c_i32), ("ind_layout", c_i32),
        ("n_elems", c_i64), ("n_points", c_i64),
        ("arity", c_i32), ("map_layout", c_i32),
        ("map", c_vp), ("ind_read", c_vp),
        ("ind_read_comps", c_i32), ("dir_comps", c_i32),
        ("dir_read", c_vp), ("inc", c_vp),
        ("inc_comps", c_i32), ("pad_", c_i32),
    ]


class MpHierPlan(ctypes.Structure):
    _fields_ = [
        ("num_blocks", c_i32), ("block_size", c_i32), ("stage_reads", c_i32), ("max_staged", c_i32),
        ("slot_bytes", c_i32), ("written_is_staged", c_i32),
        ("meta", c_vp), ("staged_ids", c_vp),
        ("written_offsets", c_vp), ("written_ids", c_vp), ("written_slots", c_vp),
        ("local_slots", c_vp), ("thread_colours", c_vp), ("colour_counts", c_vp),
        ("num_block_colours", c_i32), ("pad_", c_i32),
        ("colour_block_offsets_host", c_vp), ("blocks_by_colour", c_vp),
        ("order", c_vp), ("pred_offsets", c_vp), ("preds", c_vp), ("flags", c_vp), ("tickets", c_vp),
        ("pull_off", c_vp), ("pull_ref", c_vp),
        ("tdesc_colour", c_vp), ("tdesc_order", c_vp), ("elem_meta", c_vp), ("elem_meta_bytes", c_i32),
        ("pad2_", c_i32), ("tpred_offsets", c_vp), ("tpreds", c_vp), ("tpred_pad", c_vp), ("tblock_colour", c_vp),
    ]


_SIGNATURES = {
    "mp_last_error": (ctypes.c_char_p, []),
    "mp_version": (ctypes.c_char_p, []),
    "mp_device_sm_count": (c_i32, [c_i32]),
    "mp_exec_global": (c_i32, [ctypes.POINTER(MpLoop), c_vp, c_i32, c_i32, c_vp]),
    "mp_exec_hier": (c_i32, [ctypes.POINTER(MpLoop), ctypes.POINTER(MpHierPlan), c_i32, c_u32, c_vp]),
    "mp_exec_hier_pipelined": (c_i32, [ctypes.POINTER(MpLoop), ctypes.POINTER(MpHierPlan), c_i32, c_u32, c_vp]),
    "mp_exec_hier_stream": (c_i32, [ctypes.POINTER(MpLoop), ctypes.POINTER(MpHierPlan), c_i32, c_u32, c_vp]),
    "mp_exec_atomic": (c_i32, [ctypes.POINTER(MpLoop), c_vp]),
    "mp_exec_serial":(c_i32, [ctypes.POINTER(MpLoop), c_vp, c_vp, c_vp, c_vp]),
    "mp_race_check": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "mp_plan_block_points": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_i32, c_i32, c_u32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "mp_plan_local_slots": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_i32, c_i32, c_u32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mp_plan_thread_colours": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_i32, c_i32, c_u32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "mp_plan_gather_refs": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "mp_exec_hier_gather": (c_i32, [ctypes.POINTER(MpLoop), ctypes.POINTER(MpHierPlan), c_vp, c_vp, c_i32, c_vp]),
    "mp_plan_row_placement": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "mp_plan_block_colours": (c_i32, [c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "mp_greedy_colour_csr": (c_i32, [c_i64, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "mp_greedy_colour_adj": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "mp_smallest_last_order": (c_i32, [c_i64, c_vp, c_vp, c_vp]),
    "mp_bfs_levels": (c_i32, [c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "mp_bfs_levels_host": (c_i32, [c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "mp_pairs_from_segments": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mp_plan_block_dag": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_vp, c_i32, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "mp_heavy_edge_matching": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "mp_cut_weight": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "mp_refine_boundary_pass": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i32, c_vp]),
    "mp_heavy_edge_matching_device": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "mp_refine_boundary": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_vp]),
    "mp_rebalance": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i32]),
    "mp_initial_partition": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp]),
    "mp_halo_pack":(c_i32, [c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "mp_halo_unpack": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_vp]),
    "mp_halo_put": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "mp_halo_get": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_i64, c_vp, c_vp, c_i32, c_vp]),
    "mp_epoch_bump": (c_i32, [c_vp, c_vp]),
    "mp_halo_signal": (c_i32, [c_vp, c_vp, c_vp]),
    "mp_exec_hier_stream_export": (c_i32, [ctypes.POINTER(MpLoop), ctypes.POINTER(MpHierPlan), c_i32, c_vp, c_vp]),
    "mp_export_desc_bytes": (c_i32, []),
    "mp_mailbox_alloc": (c_i32, [c_i64, c_vp]),
    "mp_ipc_handle": (c_i32, [c_vp, c_vp]),
    "mp_ipc_open": (c_i32, [c_vp, c_vp]),
    "mp_ipc_close": (c_i32, [c_vp]),
    "mp_free": (None, [c_vp]),
}

_lib = None


def exported_symbols() -> tuple:
    return tuple(_SIGNATURES)


def load():
    """Load the library once; raises DeviceError when it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DeviceError(
            f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
            "(python -m paper_1802_03749_b200.build_native). There is no CPU fallback."
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    lib = load()
    status = getattr(lib, name)(*args)
    if status != 0:
        msg = lib.mp_last_error()
        raise_for_status(status, msg.decode() if msg else "")


# --- pointer helpers -------------------------------------------------------------


def ptr(t) -> int | None:
    """Raw address of a torch tensor (device or host) or numpy array; None -> NULL."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the engine runs only on the GPU (no CPU fallback)")
    load()
