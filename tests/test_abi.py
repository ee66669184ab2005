"""CPU-only checks of the C-ABI boundary: the sm_100a library loads without a
GPU, exports every symbol include/*.h declares, its host-side parameter
logic mirrors GridParams (core.hpp:84-132), and it refuses to run without a
usable device instead of falling back to the CPU."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_1907_03620_b200 import _native as N
from paper_1907_03620_b200.build import GEN_LIB, GPU_LIB
from paper_1907_03620_b200.raster import Bounds, ConfigError, GridParams

ROOT = Path(__file__).resolve().parents[1]


def declared(header: Path) -> set[str]:
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(rg_\w+)\s*\(", text)) - {"rg_status", "rg_memkind"}


@pytest.mark.parametrize("header,lib", [("raster_gpu.h", GPU_LIB), ("raster_datagen.h", GEN_LIB)])
def test_library_exports_every_declared_symbol(header, lib):
    names = declared(ROOT / "include" / header)
    assert names
    handle = C.CDLL(str(lib))
    missing = [n for n in sorted(names) if not hasattr(handle, n)]
    assert not missing, missing
    table = N.GPU_SYMBOLS if header == "raster_gpu.h" else N.GEN_SYMBOLS
    assert set(table) == names  # the ctypes mirror binds exactly the header


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(GPU_LIB)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def test_abi_version_and_defaults():
    lib = N.gpu()
    assert lib.rg_abi_version() == 1
    p = N.rg_params()
    lib.rg_params_default(C.byref(p))
    # GridParams{} core.hpp:84-93
    assert (p.precision, p.x_min, p.x_max, p.y_min, p.y_max) == (3.5, -180.0, 180.0, -90.0, 90.0)
    assert (p.threshold, p.distance, p.metric, p.min_cluster_size) == (5, 1, 0, 4)


def test_params_validation_mirrors_reference():
    GridParams().validate()
    for bad in (GridParams(threshold=0), GridParams(distance=0), GridParams(min_cluster_size=0),
                GridParams(bounds=Bounds(5.0, 5.0, -90.0, 90.0)),
                GridParams(bounds=Bounds(-180.0, 180.0, -90.0, float("inf"))),
                GridParams(precision=400.0)):
        with pytest.raises(ConfigError):
            bad.validate()


def test_params_host_facts(kat):
    c = kat["tile_bound"]
    gp = GridParams(precision=c["precision"], bounds=Bounds(*c["bounds"]))
    assert gp.tile_bound() == c["value"]
    assert GridParams(precision=3.5).scale() == kat["scale"]["value"]
    g3 = GridParams(precision=3.0)
    assert (g3.min_column(), g3.max_column()) == (-180000, 180000)


def test_gpu_key_limit_is_a_config_error():
    # 10^9 tiles per degree: columns * rows exceed a 63-bit packed key.
    with pytest.raises(ConfigError):
        GridParams(precision=9.0).validate()


def test_no_device_means_error_not_fallback():
    lib = N.gpu()
    if lib.rg_device_count() > 0:
        pytest.skip("a usable device is present")
    h = C.c_void_p()
    p = N.rg_params()
    lib.rg_params_default(C.byref(p))
    st = lib.rg_create(C.byref(p), -1, C.byref(h))
    assert st == N.RG_ERR_CUDA
    assert h.value is None
    assert lib.rg_last_error(None)


def test_stream_handle_mapping():
    """torch's legacy default stream reports handle 0, which the C-ABI reads
    as "the context's private stream"; the Python layer passes it as
    cudaStreamLegacy so work stays ordered with torch's producers."""
    from paper_1907_03620_b200.raster import stream_arg

    assert stream_arg(None) is None
    assert stream_arg(0) == 1
    assert stream_arg(0x7F00DEADBEEF) == 0x7F00DEADBEEF
