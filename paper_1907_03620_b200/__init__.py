"""B200-native (sm_100a) RASTER contraction + agglomeration.

The product is libraster_b200.so (C-ABI: include/raster_gpu.h; C++ drop-in:
include/raster_b200/gpu.hpp). This package builds it in-tree and exposes a
Python mirror of the reference API (raster.py) for tests and benchmarks.
"""
from .raster import (  # noqa: F401
    Bounds,
    Cluster,
    ClusterSet,
    ConfigError,
    Error,
    FlatClustering,
    GridParams,
    Metric,
    Mode,
    OobPolicy,
    OutOfBoundsError,
    Pipeline,
    PipelineStats,
    SignificantTiles,
    Tile,
    TileAccumulator,
    agglomerate,
    agglomerate_flat,
    cluster_flat,
    cluster_sequential,
    device_count,
    neighbor_offsets,
    window_fix,
)
