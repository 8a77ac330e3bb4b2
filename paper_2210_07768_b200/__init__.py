"""B200-native FeatureBox extraction engine (arXiv 2210.07768).

A drop-in for the reference package's per-record extraction path
(``featurebox.pipeline._extract_batch`` and the pipelined stage chain around
it): same config schema, operator specs, errors and report, executed as a
runtime-compiled fused CUDA kernel per plan on sm_100a.
"""

from .columns import (BadMagicError, ChecksumError, ColumnImage, FormatError, Kind,
                      TruncatedError, UnknownColumnError, UnsupportedVersionError, ViewImage,
                      open_view, read_view, schema_of, unwrap_u64, wrap_u64, write_view)
from .config import (BatchInvariantError, CleanConfigError, CleanPolicy, ConfigError,
                     EmitError, JsonExtraction, LayerExecutionError, MergeUniquenessError,
                     PipelineConfig, PoolExhausted, StageError, UnsupportedOnDevice,
                     ViewSource, config_from_dict, load_config, parse_filter)
from .corpus import gen_corpus, make_corpus
from .featureops import (DictTable, FeatureConfigError, FeatureSign, FunctionRef, OperatorSpec,
                         fnv1a64, hash_combine, load_dict_table, resolve_function,
                         split_string)
from .opgraph import (LayerPlan, OperatorDag, PlacementBudget, expand_call_graph,
                      layer_schedule, place_operators, plan_report)

__version__ = "0.1.0"


def __getattr__(name):
    # the engine imports torch lazily (the planner and codegen do not need it)
    if name in ("Engine", "prepare", "run_pipelined", "run_pipeline", "run_views",
                "RunReport", "DeviceView", "parse_report_block"):
        from . import engine
        return getattr(engine, name)
    if name == "run_sharded":
        from . import sharded
        return sharded.run_sharded
    raise AttributeError(name)
