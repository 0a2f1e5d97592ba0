"""B200-native batched Digital-Twin sweep (drop-in for the hot path of the
arXiv 2508.08343 reference `loratwin`). See DESIGN.md and include/loratwin_gpu.h."""
from .types import *  # noqa: F401,F403
from .types import (AdapterSpec, AdapterTemplate, Condition, ConfigError, DeviceError, FrontierPoint, GMode,
                    InternalError, LengthMode, LengthSpec, LoadSource, LoratwinError, MetricsSummary, Phase,
                    PlacementResult, Request, ServerConfig, SimOptions, SimulationError, SimulationResult,
                    SweepGrid, SweepOptions, UnsupportedError, ValidationError, WorkloadSpec, enumerate_conditions,
                    h100_like_config, instantiate_condition)
from .batch import ConditionBatch, WorkloadBatch
from .api import (Device, Plan, device_group, compute_metrics, condition_hash, device, encode_workload, generate_arrivals,
                  generate_dataset, ideal_throughput, load_library, run_scripted, run_simulation, sweep_conditions, sweep_optimal)

from .predictor import (DatasetRow, DecisionTree, ForestModel, ForestParams, PlacementModel, PredictTarget, TreeNode,
                        TreeParams, train_forest, train_placement_model, train_tree)

__version__ = "0.1.0"
