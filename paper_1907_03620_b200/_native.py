"""ctypes bindings of the in-tree native libraries.

The clustering library (libraster_b200.so, C-ABI include/raster_gpu.h) is the
only compute path: there is no Python or CPU fallback. If the library is
missing, importing a compute entry point raises NativeLibraryMissing.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .build import GEN_LIB, GPU_LIB

RG_OK, RG_ERR_CONFIG, RG_ERR_OOB, RG_ERR_CUDA, RG_ERR_OOM, RG_ERR_STATE, RG_ERR_ARG, RG_ERR_UNSUPPORTED = range(8)
RG_MEM_HOST, RG_MEM_DEVICE = 0, 1
RG_CLUSTER_WINDOW_FIX = 1


class NativeLibraryMissing(RuntimeError):
    pass


class rg_params(C.Structure):
    _fields_ = [
        ("precision", C.c_double),
        ("x_min", C.c_double), ("x_max", C.c_double),
        ("y_min", C.c_double), ("y_max", C.c_double),
        ("threshold", C.c_uint64),
        ("distance", C.c_int32),
        ("metric", C.c_int32),
        ("min_cluster_size", C.c_uint64),
        ("mode", C.c_int32),
        ("oob_policy", C.c_int32),
        ("dedupe_points", C.c_int32),
        ("reserved0", C.c_int32),
        ("capacity_hint", C.c_uint64),
    ]


class rg_stats(C.Structure):
    _fields_ = [
        ("n_points", C.c_uint64),
        ("n_ingested", C.c_uint64),
        ("n_skipped", C.c_uint64),
        ("peak_accumulator_entries", C.c_uint64),
        ("n_significant", C.c_uint64),
        ("n_components", C.c_uint64),
        ("n_clusters", C.c_uint64),
        ("table_capacity", C.c_uint64),
        ("table_grows", C.c_uint64),
        ("ms_contract", C.c_double),
        ("ms_prune", C.c_double),
        ("ms_agglomerate", C.c_double),
        ("ms_label", C.c_double),
    ]


class rg_device_view(C.Structure):
    _fields_ = [
        ("key", C.c_void_p),
        ("count", C.c_void_p),
        ("cluster_id", C.c_void_p),
        ("n_significant", C.c_uint64),
        ("n_clusters", C.c_uint64),
        ("origin_x", C.c_int64),
        ("origin_y", C.c_int64),
        ("key_bits_y", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


class rg_gen_spec(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("n_clusters", C.c_uint64),
        ("points_per_cluster", C.c_uint64),
        ("sigma", C.c_double),
        ("blob_points", C.c_uint64),
        ("blob_sigma", C.c_double),
        ("n_walks", C.c_uint64),
        ("walk_steps", C.c_uint64),
        ("points_per_step", C.c_uint64),
        ("step", C.c_double),
        ("n_noise", C.c_uint64),
        ("x_lo", C.c_double), ("x_hi", C.c_double),
        ("y_lo", C.c_double), ("y_hi", C.c_double),
    ]


P = C.c_void_p
U64 = C.c_uint64
I64 = C.c_int64
ST = C.c_int

# name -> (restype, argtypes); mirrors include/raster_gpu.h exactly.
GPU_SYMBOLS = {
    "rg_abi_version": (C.c_int, []),
    "rg_status_string": (C.c_char_p, [ST]),
    "rg_device_count": (C.c_int, []),
    "rg_params_default": (None, [C.POINTER(rg_params)]),
    "rg_params_validate": (ST, [C.POINTER(rg_params), C.c_char_p, C.c_size_t]),
    "rg_params_scale": (C.c_double, [C.POINTER(rg_params)]),
    "rg_params_min_column": (I64, [C.POINTER(rg_params)]),
    "rg_params_max_column": (I64, [C.POINTER(rg_params)]),
    "rg_params_tile_bound": (C.c_double, [C.POINTER(rg_params)]),
    "rg_create": (ST, [C.POINTER(rg_params), C.c_int, C.POINTER(P)]),
    "rg_destroy": (None, [P]),
    "rg_last_error": (C.c_char_p, [P]),
    "rg_set_stream": (ST, [P, P]),
    "rg_synchronize": (ST, [P]),
    "rg_reset": (ST, [P]),
    "rg_ingest": (ST, [P, P, U64, ST]),
    "rg_stream_begin": (ST, [P, U64]),
    "rg_stream_buffer": (ST, [P, P, P]),
    "rg_stream_submit": (ST, [P, U64]),
    "rg_stream_end": (ST, [P]),
    "rg_merge": (ST, [P, P]),
    "rg_clone": (ST, [P, C.POINTER(P)]),
    "rg_key_packing": (ST, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(C.c_uint32)]),
    "rg_export_entries": (ST, [P, P, P, U64, C.POINTER(U64), ST]),
    "rg_ingest_counts": (ST, [P, P, P, U64, ST]),
    "rg_entry_count": (ST, [P, C.POINTER(U64)]),
    "rg_total_ingested": (ST, [P, C.POINTER(U64)]),
    "rg_skipped": (ST, [P, C.POINTER(U64)]),
    "rg_count_of": (ST, [P, I64, I64, C.POINTER(U64)]),
    "rg_export_counts": (ST, [P, P, P, P, U64, C.POINTER(U64)]),
    "rg_prune": (ST, [P, C.POINTER(U64)]),
    "rg_window_fix": (ST, [P, C.POINTER(U64)]),
    "rg_load_significant": (ST, [P, P, P, P, U64, ST]),
    "rg_agglomerate": (ST, [P, C.POINTER(U64)]),
    "rg_cluster": (ST, [P, P, U64, ST, C.POINTER(rg_stats)]),
    "rg_cluster_ex": (ST, [P, P, U64, ST, C.c_uint32, C.POINTER(rg_stats)]),
    "rg_prune_agglomerate": (ST, [P, C.c_uint32, C.POINTER(rg_stats)]),
    "rg_route_pairs": (ST, [P, P, P, U64, I64, U64, P, C.c_uint32, P, P, P]),
    "rg_get_significant": (ST, [P, P, P, P, P, U64, ST]),
    "rg_get_clusters": (ST, [P, P, P, P, P, U64, ST]),
    "rg_device_result": (ST, [P, C.POINTER(rg_device_view)]),
    "rg_decode_key": (None, [C.POINTER(rg_device_view), U64, C.POINTER(I64), C.POINTER(I64)]),
    "rg_label_points": (ST, [P, P, U64, P, ST]),
    "rg_cluster_points": (ST, [P, P, U64, ST, C.POINTER(U64), C.POINTER(U64)]),
    "rg_get_cluster_points": (ST, [P, P, U64, P, ST]),
    "rg_get_stats": (ST, [P, C.POINTER(rg_stats)]),
    "rg_kernel_launches": (U64, [P]),
}

GEN_SYMBOLS = {
    "rg_gen_count": (U64, [C.POINTER(rg_gen_spec)]),
    "rg_generate": (C.c_int, [C.POINTER(rg_gen_spec), P, C.c_int]),
    "rg_shuffle": (C.c_int, [P, P, U64, U64, C.c_int]),
}

_gpu = None
_gen = None


def _bind(lib, table):
    for name, (res, args) in table.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def _load(path: Path, table, what: str):
    if not path.exists():
        raise NativeLibraryMissing(
            f"{what} not built: {path} is missing. Run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `python -m paper_1907_03620_b200.build`.")
    return _bind(C.CDLL(str(path)), table)


def gpu():
    """The sm_100a clustering library (product path)."""
    global _gpu
    if _gpu is None:
        import os

        override = os.environ.get("RASTER_B200_LIB")  # A/B experiments with variant builds
        _gpu = _load(Path(override) if override else GPU_LIB, GPU_SYMBOLS, "libraster_b200.so")
    return _gpu


def gen():
    global _gen
    if _gen is None:
        _gen = _load(GEN_LIB, GEN_SYMBOLS, "libraster_datagen.so")
    return _gen
