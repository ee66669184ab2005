"""Shared test setup. GPU tests are marked `gpu`; everything else runs on a
CPU-only box. The native libraries are built in-tree once per session."""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


@pytest.fixture(scope="session", autouse=True)
def _built_libraries():
    from paper_1907_03620_b200 import build

    build.build_gpu()
    build.build_datagen()
    # The oracle (test infrastructure) is rebuilt only if missing: on the GPU
    # box the reference tree is absent and the shipped oracle/_ref is kept.
    if not (ROOT / "oracle" / "_build" / "liboracle.so").exists():
        build.build_oracle()
    yield


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    z = np.load(ROOT / "tests" / "golden" / "ref_fixtures.npz")
    meta = json.loads(bytes(z["meta"]))
    return z, meta


@pytest.fixture(scope="session")
def kat():
    import json

    return json.loads((ROOT / "tests" / "golden" / "kat_reference.json").read_text())
