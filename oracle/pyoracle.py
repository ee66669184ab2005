"""ctypes bindings of the CPU checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm import this module; the product package never does.

    port() -> oracle/_build/liboracle.so   C restatement (raster_oracle.c)
    ref()  -> oracle/_ref/libraster_ref.so  the reference compiled from its
              own headers (ref_shim.cpp); None when it was never built
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_build" / "liboracle.so"
REF_LIB = HERE / "_ref" / "libraster_ref.so"


class orc_params(C.Structure):
    _fields_ = [
        ("precision", C.c_double),
        ("x_min", C.c_double), ("x_max", C.c_double),
        ("y_min", C.c_double), ("y_max", C.c_double),
        ("threshold", C.c_uint64),
        ("distance", C.c_int32),
        ("metric", C.c_int32),
        ("min_cluster_size", C.c_uint64),
    ]


class orc_result(C.Structure):
    _fields_ = [
        ("n_ingested", C.c_uint64),
        ("n_skipped", C.c_uint64),
        ("n_distinct", C.c_uint64),
        ("n_sig", C.c_uint64),
        ("tx", C.POINTER(C.c_int64)),
        ("ty", C.POINTER(C.c_int64)),
        ("count", C.POINTER(C.c_uint64)),
        ("cluster_id", C.POINTER(C.c_int64)),
        ("n_components", C.c_uint64),
        ("n_clusters", C.c_uint64),
    ]


@dataclass
class Result:
    """Canonical flat clustering (same form as FlatClustering)."""
    tx: np.ndarray
    ty: np.ndarray
    count: np.ndarray
    cluster_id: np.ndarray
    n_clusters: int
    n_ingested: int = 0
    n_skipped: int = 0
    n_distinct: int = 0
    n_components: int = 0


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        if not PORT_LIB.exists():
            raise RuntimeError(f"oracle not built: {PORT_LIB} (run oracle/build_ref.sh)")
        lib = C.CDLL(str(PORT_LIB))
        P = C.c_void_p
        lib.orc_cluster.argtypes = [P, C.c_uint64, C.POINTER(orc_params), C.POINTER(orc_result)]
        lib.orc_cluster_ex.argtypes = [P, C.c_uint64, C.POINTER(orc_params), C.c_int,
                                       C.POINTER(orc_result)]
        lib.orc_agglomerate.argtypes = [P, P, P, C.c_uint64, C.POINTER(orc_params),
                                        C.POINTER(orc_result)]
        lib.orc_label_points.argtypes = [P, C.c_uint64, C.POINTER(orc_params),
                                         C.POINTER(orc_result), P]
        lib.orc_free.argtypes = [C.POINTER(orc_result)]
        lib.orc_project.argtypes = [C.c_double, C.c_double, C.c_double,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        _port = lib
    return _port


def ref():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            return None
        lib = C.CDLL(str(REF_LIB))
        P = C.c_void_p
        lib.ref_cluster.argtypes = [P, C.c_uint64, C.POINTER(orc_params), C.c_uint,
                                    C.POINTER(orc_result), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
        lib.ref_time_pipeline.argtypes = [P, C.c_uint64, C.POINTER(orc_params), C.c_uint,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]
        lib.ref_time_pipeline.restype = C.c_double
        lib.ref_time_pipeline_mode.argtypes = [P, C.c_uint64, C.POINTER(orc_params), C.c_uint,
                                               C.c_int, C.POINTER(C.c_uint64),
                                               C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.ref_time_pipeline_mode.restype = C.c_double
        lib.ref_agglomerate.argtypes = [P, P, P, C.c_uint64, C.POINTER(orc_params),
                                        C.POINTER(orc_result)]
        lib.ref_cluster_flags.argtypes = [P, C.c_uint64, C.POINTER(orc_params), C.c_int,
                                          C.POINTER(orc_result)]
        lib.ref_prime_points_ex.argtypes = [P, C.c_uint64, C.POINTER(orc_params), C.c_int, P, P,
                                            P, C.c_uint64]
        lib.ref_prime_points_ex.restype = C.c_int64
        lib.ref_prime_points.argtypes = [P, C.c_uint64, C.POINTER(orc_params), P, P, P,
                                         C.c_uint64]
        lib.ref_prime_points.restype = C.c_int64
        lib.ref_strict_ingest.argtypes = [P, C.c_uint64, C.POINTER(orc_params), C.c_char_p,
                                          C.c_uint64, C.POINTER(C.c_uint64)]
        lib.ref_project.argtypes = [C.c_double, C.c_double, C.c_double,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.ref_free.argtypes = [C.POINTER(orc_result)]
        lib.ref_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


def make_params(gp) -> orc_params:
    """From a paper_1907_03620_b200.GridParams (or anything with its fields)."""
    p = orc_params()
    p.precision = float(gp.precision)
    p.x_min, p.x_max = float(gp.bounds.x_min), float(gp.bounds.x_max)
    p.y_min, p.y_max = float(gp.bounds.y_min), float(gp.bounds.y_max)
    p.threshold = int(gp.threshold)
    p.distance = int(gp.distance)
    p.metric = int(gp.metric)
    p.min_cluster_size = int(gp.min_cluster_size)
    return p


def _take(r: orc_result, free) -> Result:
    n = r.n_sig

    def arr(ptr, dt):
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True) if n else np.empty(0, dt)

    out = Result(arr(r.tx, np.int64), arr(r.ty, np.int64), arr(r.count, np.uint64),
                 arr(r.cluster_id, np.int64), int(r.n_clusters), int(r.n_ingested),
                 int(r.n_skipped), int(r.n_distinct), int(r.n_components))
    free(C.byref(r))
    return out


def _pts(points) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 2))
    return a


def _flags(window_fix: bool, dedupe: bool) -> int:
    return (1 if window_fix else 0) | (2 if dedupe else 0)


def port_cluster(points, gp, window_fix: bool = False, dedupe: bool = False) -> Result:
    """dedupe = Mode::retain_points with dedupe_points."""
    a = _pts(points)
    r = orc_result()
    lib = port()
    if lib.orc_cluster_ex(a.ctypes.data if a.size else None, a.shape[0],
                          C.byref(make_params(gp)), _flags(window_fix, dedupe), C.byref(r)) != 0:
        raise RuntimeError("oracle failed")
    return _take(r, lib.orc_free)


def port_agglomerate(tx, ty, count, gp) -> Result:
    tx = np.ascontiguousarray(tx, np.int64)
    ty = np.ascontiguousarray(ty, np.int64)
    cnt = np.ascontiguousarray(count, np.uint64)
    r = orc_result()
    lib = port()
    n = tx.shape[0]
    if lib.orc_agglomerate(tx.ctypes.data if n else None, ty.ctypes.data if n else None,
                           cnt.ctypes.data if n else None, n, C.byref(make_params(gp)),
                           C.byref(r)) != 0:
        raise RuntimeError("oracle failed")
    return _take(r, lib.orc_free)


def port_labels(points, gp, res: Result) -> np.ndarray:
    a = _pts(points)
    r = orc_result()
    r.n_sig = res.tx.shape[0]
    keep = [np.ascontiguousarray(res.tx, np.int64), np.ascontiguousarray(res.ty, np.int64),
            np.ascontiguousarray(res.count, np.uint64), np.ascontiguousarray(res.cluster_id, np.int64)]
    r.tx = keep[0].ctypes.data_as(C.POINTER(C.c_int64))
    r.ty = keep[1].ctypes.data_as(C.POINTER(C.c_int64))
    r.count = keep[2].ctypes.data_as(C.POINTER(C.c_uint64))
    r.cluster_id = keep[3].ctypes.data_as(C.POINTER(C.c_int64))
    out = np.empty(a.shape[0], np.int32)
    port().orc_label_points(a.ctypes.data if a.size else None, a.shape[0],
                            C.byref(make_params(gp)), C.byref(r),
                            out.ctypes.data if a.size else None)
    return out


def port_project(x: float, y: float, scale: float):
    tx, ty = C.c_int64(), C.c_int64()
    port().orc_project(x, y, scale, C.byref(tx), C.byref(ty))
    return tx.value, ty.value


def ref_cluster(points, gp, workers: int = 0) -> tuple[Result, float, float]:
    lib = ref()
    if lib is None:
        raise RuntimeError("reference build oracle/_ref missing")
    a = _pts(points)
    r = orc_result()
    tp, tc = C.c_double(), C.c_double()
    if lib.ref_cluster(a.ctypes.data if a.size else None, a.shape[0], C.byref(make_params(gp)),
                       workers, C.byref(r), C.byref(tp), C.byref(tc)) != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return _take(r, lib.ref_free), tp.value, tc.value


def ref_cluster_window_fix(points, gp) -> Result:
    return ref_cluster_flags(points, gp, window_fix=True)


def ref_cluster_flags(points, gp, window_fix: bool = False, dedupe: bool = False) -> Result:
    lib = ref()
    a = _pts(points)
    r = orc_result()
    if lib.ref_cluster_flags(a.ctypes.data if a.size else None, a.shape[0],
                             C.byref(make_params(gp)), _flags(window_fix, dedupe),
                             C.byref(r)) != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return _take(r, lib.ref_free)


def ref_agglomerate(tx, ty, count, gp) -> Result:
    lib = ref()
    tx = np.ascontiguousarray(tx, np.int64)
    ty = np.ascontiguousarray(ty, np.int64)
    cnt = np.ascontiguousarray(count, np.uint64)
    n = tx.shape[0]
    r = orc_result()
    if lib.ref_agglomerate(tx.ctypes.data if n else None, ty.ctypes.data if n else None,
                           cnt.ctypes.data if n else None, n, C.byref(make_params(gp)),
                           C.byref(r)) != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return _take(r, lib.ref_free)


def ref_time(points_ptr: int, n: int, gp, workers: int = 0):
    """Times the reference pipeline over a host buffer; returns
    (t_total, t_projection, t_clustering, n_clusters)."""
    lib = ref()
    nc = C.c_uint64()
    tp, tc = C.c_double(), C.c_double()
    t = lib.ref_time_pipeline(points_ptr, n, C.byref(make_params(gp)), workers, C.byref(nc),
                              C.byref(tp), C.byref(tc))
    if t < 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return t, tp.value, tc.value, nc.value


def ref_time_mode(points_ptr: int, n: int, gp, workers: int = 0, retain: bool = False):
    """ref_time with Mode::retain_points when `retain` (the reference's
    point-retaining pipeline); returns (t_total, t_projection, t_clustering,
    n_clusters)."""
    lib = ref()
    nc = C.c_uint64()
    tp, tc = C.c_double(), C.c_double()
    t = lib.ref_time_pipeline_mode(points_ptr, n, C.byref(make_params(gp)), workers, int(retain),
                                   C.byref(nc), C.byref(tp), C.byref(tc))
    if t < 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return t, tp.value, tc.value, nc.value


def ref_prime_points(points, gp, window_fix: bool = False, dedupe: bool = False):
    """Reference RASTER' output rows (cluster id, x, y) in output order."""
    lib = ref()
    a = _pts(points)
    p = make_params(gp)
    f = _flags(window_fix, dedupe)
    n = lib.ref_prime_points_ex(a.ctypes.data if a.size else None, a.shape[0], C.byref(p), f,
                                None, None, None, 0)
    if n < 0:
        raise RuntimeError(lib.ref_last_error().decode())
    cid = np.empty(n, np.int64)
    px = np.empty(n, np.float64)
    py = np.empty(n, np.float64)
    lib.ref_prime_points_ex(a.ctypes.data if a.size else None, a.shape[0], C.byref(p), f,
                            cid.ctypes.data, px.ctypes.data, py.ctypes.data, n)
    return cid, px, py


def ref_strict(points, gp):
    lib = ref()
    a = _pts(points)
    buf = C.create_string_buffer(512)
    ing = C.c_uint64()
    thrown = lib.ref_strict_ingest(a.ctypes.data if a.size else None, a.shape[0],
                                   C.byref(make_params(gp)), buf, 512, C.byref(ing))
    return bool(thrown), buf.value.decode(), ing.value


def ref_project(x: float, y: float, precision: float):
    tx, ty = C.c_int64(), C.c_int64()
    ref().ref_project(x, y, precision, C.byref(tx), C.byref(ty))
    return tx.value, ty.value
