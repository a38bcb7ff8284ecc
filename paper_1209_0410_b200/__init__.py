"""B200-native Hypercurves / Multicurves approximate-kNN hot path.

The compute path is libhcg.so (hand-written sm_100a CUDA behind the C ABI in
include/hcg.h); this package is the host-side mirror of the reference's
interface (namespace hc, proj/include/hypercurves/*.hpp) over that ABI.
"""
from ._lib import HcgError, HcgInvalidArgument, HcgIOError, LIB_PATH, lib  # noqa: F401
from .multicurves import (  # noqa: F401
    HILBERT, LIFTED, RAW, ZORDER, MulticurvesIndex, Neighbor, ProjectionScheme, SearchParams, View,
    binomial_tail, default_scheme, gen_queries, gen_rows, make_lut, merge_packed, miss_bound, monte_carlo_miss,
    plan_depth, read_search_csv, read_vectors, recall_at, shard_probe_depth, write_search_csv,
    write_vectors,
)

__version__ = "0.1.0"
