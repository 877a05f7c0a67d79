"""ctypes binding of libpdx_b200.so (the C-ABI in include/pdx_b200.h).

The library is built in-tree (``make -C paper_2503_04422_b200/csrc``, or
``__graft_entry__.build()``) so it travels with the repository to the GPU
box.  There is no fallback: if the library or a CUDA device is missing,
every product entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libpdx_b200.so"
if os.environ.get("PDX_B200_LIB"):  # development: an alternative build of the same ABI (A/B runs)
    LIB_PATH = Path(os.environ["PDX_B200_LIB"])
CSRC = PKG / "csrc"

PDX_OK, PDX_EINVAL, PDX_ECUDA, PDX_ENOSUPPORT, PDX_EFORMAT, PDX_EIO = 0, 1, 2, 3, 4, 5
METRIC = {"l2": 0, "l1": 1, "ip": 2}
PRUNER = {"none": 0, "ads": 1, "bond": 2, "bsa": 3}
CRITERIA = {"sequential": 0, "decreasing": 1, "dmeans": 2, "zones": 3}
TILE = 64

# every symbol include/pdx_b200.h declares
EXPORTS = ("pdx_abi_version", "pdx_last_error", "pdx_device_info", "pdx_pack_tiles",
           "pdx_project", "pdx_select_buckets", "pdx_dimension_orders", "pdx_search_workspace",
           "pdx_search", "pdx_merge_topk", "pdx_segment_means", "pdx_ground_truth",
           "pdx_bsa_residuals", "pdx_file_probe", "pdx_file_load", "pdx_file_save",
           "pdx_index_create", "pdx_index_open", "pdx_index_destroy", "pdx_index_search",
           "pdx_k8_norms", "pdx_k8_margin", "pdx_k8_filter", "pdx_k8_rescore",
           "pdx_vertical_accumulate", "pdx_batch_profile", "pdx_row_norms",
           "pdx_kmeans_assign", "pdx_bucket_layout", "pdx_kmeans_update", "pdx_kmeans_shift",
           "pdx_kmeans_farthest", "pdx_gather_rows", "pdx_pack_rows", "pdx_k8_norms_ld",
           "pdx_k8_candidates", "pdx_k8_rescore_rows", "pdx_k8_candidates_bf16",
           "pdx_k8_to_bf16")


class PdxStore(C.Structure):
    _fields_ = [("d", C.c_int32), ("d_pad", C.c_int32), ("group", C.c_int32),
                ("nbuckets", C.c_int32), ("ntiles", C.c_int64), ("nblocks", C.c_int64),
                ("d_tiles", C.c_void_p), ("d_tile_ids", C.c_void_p),
                ("d_block_tile", C.c_void_p), ("d_block_m", C.c_void_p),
                ("d_bucket_block", C.c_void_p), ("max_bucket_blocks", C.c_int32),
                ("max_bucket_tiles", C.c_int32), ("d_tile_block", C.c_void_p),
                ("d_resid", C.c_void_p), ("resid_steps", C.c_int32),
                ("resid_initial_step", C.c_int32)]


class PdxSearchParams(C.Structure):
    _fields_ = [("k", C.c_int32), ("metric", C.c_int32), ("pruner", C.c_int32),
                ("initial_step", C.c_int32), ("selection_fraction", C.c_double),
                ("ads_d", C.c_int32), ("warps", C.c_int32), ("ads_epsilon0", C.c_double),
                ("tiles_per_warp", C.c_int32), ("ring_slots", C.c_int32),
                ("bsa_coef", C.c_void_p), ("splits", C.c_int32),
                ("batched", C.c_int32)]


class PdxFileInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("block_size", C.c_int32),
                ("nblocks", C.c_int64), ("flags", C.c_int32), ("nlist", C.c_int32),
                ("transform_seed", C.c_uint64), ("training_seed", C.c_uint64),
                ("ntiles", C.c_int64), ("max_block_bytes", C.c_int64)]


class PdxIndexDesc(C.Structure):
    _fields_ = [("store", C.c_void_p), ("d", C.c_int32), ("group", C.c_int32),
                ("nblocks", C.c_int64), ("blocks", C.c_void_p), ("block_m", C.c_void_p),
                ("block_mpad", C.c_void_p), ("ids", C.c_void_p), ("global_means", C.c_void_p),
                ("rotation", C.c_void_p), ("nlist", C.c_int32), ("centroids", C.c_void_p),
                ("bucket_offsets", C.c_void_p), ("bucket_means", C.c_void_p)]


class PdxQueryParams(C.Structure):
    _fields_ = [("k", C.c_int32), ("metric", C.c_int32), ("pruner", C.c_int32),
                ("criteria", C.c_int32), ("zone_width", C.c_int32), ("nprobe", C.c_int32),
                ("selection_fraction", C.c_double), ("initial_step", C.c_int32),
                ("rotate", C.c_int32), ("epsilon0", C.c_double), ("bsa_coef", C.c_void_p),
                ("queries_on_device", C.c_int32), ("outputs_on_device", C.c_int32),
                ("tensor_cores", C.c_int32)]


class PdxSearchOut(C.Structure):
    _fields_ = [("d_dist", C.c_void_p), ("d_ids", C.c_void_p), ("d_count", C.c_void_p),
                ("d_touched", C.c_void_p), ("d_total", C.c_void_p), ("d_trace", C.c_void_p),
                ("trace_cap", C.c_int64), ("d_trace_len", C.c_void_p), ("d_debug", C.c_void_p)]


def build(force: bool = False, quiet: bool = True) -> Path:
    """Compile libpdx_b200.so for sm_100a with nvcc (in-tree)."""
    srcs = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "pdx_b200.h"]
    newest = max(p.stat().st_mtime for p in srcs)
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < newest:
        cmd = ["make", "-C", str(CSRC), "-j8"]
        if quiet:
            subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
        else:
            subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def lib():
    """The loaded library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                               "`python -c 'import __graft_entry__ as g; g.build()'` "
                               "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.pdx_abi_version.restype = C.c_int
        L.pdx_last_error.argtypes = [C.c_char_p, C.c_size_t]
        L.pdx_device_info.argtypes = [vp, vp, vp, vp]
        L.pdx_pack_tiles.argtypes = [vp, i64, i32, vp, i64, i32, vp, vp, vp, vp]
        L.pdx_project.argtypes = [vp, i64, i32, vp, vp, vp]
        L.pdx_select_buckets.argtypes = [vp, i64, i32, vp, i32, i32, i32, vp, vp, vp]
        L.pdx_dimension_orders.argtypes = [vp, i32, i64, i32, vp, vp, i32, i32, i32, vp, vp]
        L.pdx_search_workspace.argtypes = [vp, i64, i32]
        L.pdx_search_workspace.restype = i64
        L.pdx_search.argtypes = [vp, vp, vp, i64, vp, i32, vp, i64, i64, vp, vp, i64, vp]
        L.pdx_merge_topk.argtypes = [vp, vp, i32, i64, i32, vp, vp, vp]
        L.pdx_segment_means.argtypes = [vp, i32, vp, vp, i32, vp, vp]
        L.pdx_ground_truth.argtypes = [vp, i64, i32, vp, i64, i32, i32, vp, vp, vp]
        L.pdx_bsa_residuals.argtypes = [vp, i32, vp, vp, vp]
        L.pdx_file_probe.argtypes = [C.c_char_p, vp]
        L.pdx_index_create.argtypes = [vp, vp]
        L.pdx_index_open.argtypes = [C.c_char_p, i32, vp]
        L.pdx_index_destroy.argtypes = [vp]
        L.pdx_index_search.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, vp]
        L.pdx_k8_norms.argtypes = [vp, i64, i32, vp, vp]
        L.pdx_k8_margin.argtypes = [i32, i32]
        L.pdx_k8_margin.restype = C.c_float
        L.pdx_k8_filter.argtypes = [vp, i64, i64, i32, i64, vp, vp, i32, i32, i32, vp, vp, vp,
                                    vp, i32, vp]
        L.pdx_k8_rescore.argtypes = [vp, i64, vp, i64, i32, i32, vp, vp, i32, vp, vp, vp]
        L.pdx_file_load.argtypes = [C.c_char_p, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pdx_file_save.argtypes = [C.c_char_p, vp, i32, vp, vp, vp, C.c_uint64, i32,
                                    C.c_uint64, vp, vp, vp, vp]
        L.pdx_vertical_accumulate.argtypes = [vp, i32, i32, vp, i32, i32, vp, vp, i32, i32, vp,
                                              vp]
        L.pdx_batch_profile.argtypes = [i32, vp, i32, vp]
        L.pdx_row_norms.argtypes = [vp, i64, i32, vp, vp]
        L.pdx_kmeans_assign.argtypes = [vp, vp, i64, i32, vp, vp, vp, i32, vp, vp, vp]
        L.pdx_bucket_layout.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, vp]
        L.pdx_kmeans_update.argtypes = [vp, vp, vp, i32, i32, vp, vp]
        L.pdx_kmeans_shift.argtypes = [vp, vp, i32, i32, vp, vp]
        L.pdx_kmeans_farthest.argtypes = [vp, i64, i32, vp, i32, vp, C.c_float, vp, vp]
        L.pdx_gather_rows.argtypes = [vp, i32, vp, i64, vp, vp]
        L.pdx_pack_rows.argtypes = [vp, i64, i32, vp, vp, vp, vp]
        L.pdx_k8_norms_ld.argtypes = [vp, i64, i32, i64, vp, vp]
        L.pdx_k8_candidates_bf16.argtypes = [vp, i64, i32, i64, vp, vp, vp, i64, i64, i32, i32,
                                             vp, vp, i32, vp, vp, vp]
        L.pdx_k8_to_bf16.argtypes = [vp, i64, i32, i64, i64, vp, vp]
        L.pdx_k8_rescore_rows.argtypes = [vp, i64, i32, vp, vp, i64, i32, i32, vp, vp, i32, i32,
                                           vp, vp, vp]
        L.pdx_k8_candidates.argtypes = [vp, i64, i32, i64, vp, vp, i64, i32, i32, vp, vp, i32,
                                        vp, vp, vp]
        for name in EXPORTS:
            getattr(L, name).restype = getattr(L, name).restype or C.c_int
        if L.pdx_abi_version() != 3:
            raise RuntimeError("libpdx_b200.so ABI version mismatch")
        _lib = L
    return _lib


def last_error() -> str:
    buf = C.create_string_buffer(1024)
    lib().pdx_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def check(rc: int):
    """Map an ABI status to the reference's exception types."""
    if rc == PDX_OK:
        return
    msg = last_error()
    if rc == PDX_EINVAL:
        raise ValueError(msg)
    if rc == PDX_ENOSUPPORT:
        raise NotImplementedError(msg)
    if rc == PDX_EFORMAT:
        from .storage import FormatError
        raise FormatError(msg)
    if rc == PDX_EIO:
        raise OSError(msg)
    raise RuntimeError(f"CUDA failure in libpdx_b200: {msg}")


def ptr(t) -> int | None:
    """Device (or host) address of a torch tensor / numpy array; None for None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_handle(stream=None) -> int | None:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream or None
