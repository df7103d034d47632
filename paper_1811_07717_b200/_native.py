"""ctypes binding of libhfb200.so (the C ABI in include/hfb200.h).

The library is required: importing this module without it raises
ImportError, and every call needs a CUDA device.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libhfb200.so")

HF_COL_DONE, HF_COL_FAILED, HF_COL_ZERO, HF_COL_FROZEN = 2, 3, 4, 5
PCG_WIDTHS = (2, 4, 8, 16, 32, 64)


class HfCsr(C.Structure):
    _fields_ = [("n_rows", C.c_int32), ("n_cols", C.c_int32), ("nnz", C.c_int64),
                ("indptr", C.c_void_p), ("indices", C.c_void_p), ("val", C.c_void_p)]


class HfSegmentation(C.Structure):
    _fields_ = [("n_comp", C.c_int32), ("n_surf", C.c_int32), ("n_dir", C.c_int32),
                ("comp_surf", C.c_void_p), ("tri_off", C.c_void_p), ("box", C.c_void_p),
                ("rays", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `python paper_1811_07717_b200/build.py` (nvcc, sm_100a).  There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, D, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t
    pcsr = C.POINTER(HfCsr)
    sig = {
        "hf_version": (C.c_char_p, []),
        "hf_last_error": (C.c_char_p, []),
        "hf_device_sm_count": (C.c_int, [C.POINTER(I32)]),
        "hf_launch_count": (C.c_longlong, []),
        "hf_scan_workspace_bytes": (SZ, [I32]),
        "hf_exclusive_scan_i32": (C.c_int, [P, P, I32, P, P, SZ, P]),
        "hf_ldp": (C.c_int, [pcsr, P, P, C.POINTER(I32), P]),
        "hf_csr_bandwidth": (C.c_int, [pcsr, P, C.POINTER(I32), P]),
        "hf_csr_prune_workspace_bytes": (SZ, [I32]),
        "hf_csr_prune_count": (C.c_int, [pcsr, P, SZ, C.POINTER(I64), P]),
        "hf_csr_prune_fill": (C.c_int, [pcsr, P, SZ, P, P, P, P]),
        "hf_pcg_workspace_bytes": (SZ, [I32, I32, I64]),
        "hf_pcg_multi": (C.c_int, [pcsr, P, P, I32, I32, D, I32, P, P, P, P, P, P, P, P, SZ, P]),
        "hf_pcg_profile": (C.c_int, [pcsr, P, P, I32, I32, I32, P, P, C.POINTER(I32), P, SZ, P]),
        "hf_pcg_stream_workspace_bytes": (SZ, [I32, I32, I32]),
        "hf_pcg_stream": (C.c_int, [pcsr, P, P, I32, I32, I32, I32, D, I32, P, P, P, P, P, P, P, SZ, P]),
        "hf_p1_blocks": (C.c_int, [P, P, I32, P, I32, P, I32, D, P, P, C.POINTER(I32), P]),
        "hf_p1_assemble_workspace_bytes": (SZ, [I32, I32, I32]),
        "hf_p1_assemble_prepare": (C.c_int, [P, I32, I32, P, I32, I32, P, C.POINTER(I64), P, SZ, P]),
        "hf_p1_assemble_fill": (C.c_int, [P, I32, I32, P, P, P, I32, I32, P, P, P, P, SZ, P]),
        "hf_response_matrix": (C.c_int, [pcsr, P, I32, I32, I32, I32, P, P, P]),
        "hf_lf_tail": (C.c_int, [P, I32, I32, pcsr, P, I32, I32, P, P]),
        "hf_dense_lf": (C.c_int, [P, I32, I32, P, I32, I32, P, I32, P]),
        "hf_eit_sens_workspace_bytes": (SZ, [I64]),
        "hf_csr_dense": (C.c_int, [pcsr, P, I32, I32, P, I32, P]),
        "hf_eit_sens": (C.c_int, [P, P, P, P, I32, I32, P, I32, I32, P, I32, I32, P, P, SZ, P]),
        "hf_topology_workspace_bytes": (SZ, [I32, I32, I32]),
        "hf_boundary_faces": (C.c_int, [P, I32, I32, P, C.POINTER(I64), P, SZ, P]),
        "hf_whitney_gt": (C.c_int, [P, P, I32, I32, P, I32, P, P, P, P, C.POINTER(I64), P, SZ, P]),
        "hf_nearest_center": (C.c_int, [P, I32, P, I32, P, P, P]),
        "hf_triangle_centroids": (C.c_int, [P, P, I32, P, P]),
        "hf_tet_centroids": (C.c_int, [P, P, P, I32, P, P]),
        "hf_dof_partition_workspace_bytes": (SZ, [I32]),
        "hf_dof_partition": (C.c_int, [P, P, I32, I32, P, P, P, SZ, P]),
        "hf_ground_node_workspace_bytes": (SZ, [I32]),
        "hf_ground_node": (C.c_int, [P, I32, P, I32, I32, P, C.POINTER(I32), P]),
        "hf_locate": (C.c_int, [C.POINTER(HfSegmentation), P, I32, P, P]),
        "hf_grid_tets": (C.c_int, [P, P, P, I32, I32, I32, P, P, P]),
        "hf_mesh_compact_workspace_bytes": (SZ, [I32, I32]),
        "hf_mesh_compact": (C.c_int, [P, P, I32, P, P, P, I32, I32, I32, P, P, P, C.POINTER(I64),
                                      C.POINTER(I64), P, SZ, P]),
        "hf_apply_priorities": (C.c_int, [P, I32, P, P, P, P]),
        "hf_meg_workspace_bytes": (SZ, [I32, I32]),
        "hf_meg_rhs": (C.c_int, [P, P, P, I32, I32, I32, P, P, I32, P, I32, P, SZ, P]),
        "hf_meg_primary": (C.c_int, [P, P, I32, P, I32, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

# Every symbol include/hfb200.h declares (checked by tests/test_abi.py).
EXPORTED = ("hf_version", "hf_last_error", "hf_device_sm_count", "hf_launch_count", "hf_scan_workspace_bytes",
            "hf_exclusive_scan_i32", "hf_ldp", "hf_csr_bandwidth",
            "hf_csr_prune_workspace_bytes", "hf_csr_prune_count", "hf_csr_prune_fill",
            "hf_pcg_workspace_bytes", "hf_pcg_multi", "hf_pcg_profile", "hf_pcg_stream_workspace_bytes",
            "hf_pcg_stream", "hf_p1_blocks",
            "hf_p1_assemble_workspace_bytes", "hf_p1_assemble_prepare", "hf_p1_assemble_fill",
            "hf_response_matrix", "hf_lf_tail", "hf_dense_lf", "hf_csr_dense", "hf_eit_sens_workspace_bytes", "hf_eit_sens",
            "hf_topology_workspace_bytes", "hf_boundary_faces", "hf_whitney_gt",
            "hf_nearest_center", "hf_triangle_centroids", "hf_tet_centroids",
            "hf_dof_partition_workspace_bytes", "hf_dof_partition", "hf_ground_node_workspace_bytes",
            "hf_ground_node", "hf_locate", "hf_grid_tets", "hf_mesh_compact_workspace_bytes",
            "hf_mesh_compact", "hf_apply_priorities", "hf_meg_workspace_bytes", "hf_meg_rhs",
            "hf_meg_primary")


class NativeError(RuntimeError):
    """A libhfb200 call returned a non-zero hf_status."""

    def __init__(self, name, code):
        msg = lib.hf_last_error().decode(errors="replace")
        super().__init__(f"{name} failed (status {code}): {msg}")
        self.code = code


def check(name, code):
    if code != 0:
        raise NativeError(name, code)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1811_07717_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")


def ptr(t):
    """Device (or host) address of a tensor, or None."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def csr_struct(n_rows, n_cols, indptr, indices, val):
    return HfCsr(int(n_rows), int(n_cols), int(indices.numel()), indptr.data_ptr(),
                 indices.data_ptr(), val.data_ptr())
