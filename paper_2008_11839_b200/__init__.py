"""gconn-b200: the GConn connectivity design space (arXiv 2008.11839) on
NVIDIA B200 (sm_100a).

Drop-in for the reference ``connlab`` driver API: the names below mirror
connlab/__init__.py:12-82.  All connectivity work runs in libgconn.so
(hand-written CUDA, loaded through a C ABI declared in include/gconn.h);
there is no CPU fallback.
"""
from .api import (DeviceForest, ForestEdges, RunStats, StaticConnectivity, finish_phase, label_finalization,
                  spanning_forest, spanning_forest_device, static_connectivity,
                  static_connectivity_device)
from .dset import DisjointSets, union_edge_list
from .errors import ConfigError, MalformedInputError, NativeError, VerificationError
from .generators import (build_csr, clique_graph, disjoint_union, gen_rmat, gen_uniform_pairs,
                         grid3d_edges, grid_graph, path_graph, star_graph)
from .graph import EdgeList, Graph
from .graphio import (gen_ba, gnp_graph, graph_to_edge_list, is_binary_graph, load_graph, load_graph_binary,
                      save_graph_binary)
from .incremental import IncrementalConnectivity, Insert, Query, incremental
from .spec import (LT_VARIANTS, AlgorithmSpec, FindOp, FinishKind, KOutMode, LTVariant, SampleKind,
                   SpliceOp, UnionConfig, UnionOp, all_valid_configs, enumerate_specs, format_spec,
                   parse_spec, valid_combination)
from .validate import (canonical_labels, check_forest, oracle_components, oracle_components_unionfind,
                       partition_equal, sampling_stats)

__version__ = "0.1.0"

__all__ = [
    "AlgorithmSpec", "ConfigError", "DeviceForest", "EdgeList", "FindOp", "FinishKind",
    "ForestEdges", "Graph", "IncrementalConnectivity", "Insert", "KOutMode", "LTVariant",
    "LT_VARIANTS", "MalformedInputError", "NativeError", "Query", "RunStats", "SampleKind",
    "SpliceOp", "StaticConnectivity", "UnionConfig", "UnionOp", "VerificationError", "all_valid_configs", "build_csr",
    "clique_graph", "disjoint_union", "enumerate_specs", "finish_phase", "format_spec",
    "gen_rmat", "gen_uniform_pairs", "grid3d_edges", "grid_graph", "incremental",
    "label_finalization", "parse_spec", "path_graph", "spanning_forest", "spanning_forest_device",
    "star_graph", "static_connectivity", "static_connectivity_device", "valid_combination",
    "DisjointSets", "union_edge_list", "canonical_labels", "check_forest", "oracle_components",
    "oracle_components_unionfind", "partition_equal", "sampling_stats", "gen_ba", "gnp_graph",
    "graph_to_edge_list", "is_binary_graph", "load_graph", "load_graph_binary", "save_graph_binary",
]
