"""The C++ drop-in (include/raster_b200/gpu.hpp) against the reference
library, over the reference's own types (tests/cpp/adapter_parity.cpp; built
in the build container by tests/cpp/build.sh). Needs a B200."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "adapter_parity"


@pytest.mark.gpu
def test_cpp_adapter_matches_reference():
    if not BIN.exists():
        pytest.skip("adapter_parity not built (needs /root/reference headers at build time)")
    out = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK: 0 failure(s)" in out.stdout
