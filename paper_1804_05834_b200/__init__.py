"""paper_1804_05834_b200 -- B200-native (sm_100a) CytonRL / deepq learner.

Same public names as the reference package (deepq/__init__.py:9-32) for the
learner hot path -- replay (ring + sum tree), network, optimizer and
``learn_step`` -- and for the acting loop around it (Trainer, select_action,
evaluate, the desk environments and the frame pipeline).  Everything computes in libdqn_b200.so on the GPU; importing
fails if that library is missing and every constructor fails without a CUDA
device (there is no CPU fallback).
"""

from . import _lib  # noqa: F401  (loads libdqn_b200.so or raises ImportError)
from .agent import (TdResult, compute_target_double, compute_target_dqn,  # noqa: F401
                    learn_step)
from .checkpoint import (Checkpoint, load_checkpoint, load_params_into,  # noqa: F401
                         save_checkpoint)
from .config import PRESETS, RunConfig, resolve_config  # noqa: F401
from .envs import (Catch, Environment, EnvSpec, EnvStep, GridWorld, Preprocessor,  # noqa: F401
                   TabularChain, bilinear_resize, make_env, preprocess_frame)
from .metrics import MetricRecord, MetricsWriter, RecordCollector  # noqa: F401
from .errors import (ArchitectureMismatchError, CheckpointCRCError,  # noqa: F401
                     CheckpointError, CheckpointMagicError, CheckpointVersionError,
                     ConfigError, DeepQError, GeometryError, NonFiniteError, PhaseOrderError)
from .network import (ARCHITECTURES, LayerSpec, Network, build_network,  # noqa: F401
                      init_params, load_params, trunk_layers)
from .optim import RmsProp, clip_gradients, sync_target  # noqa: F401
from .replay import (PrioritizedReplay, PriorityConfig, ReplayMemory,  # noqa: F401
                     SampleBatch, SumTree, Transition, anneal_beta)
from .schedules import LinearSchedule  # noqa: F401
from .tensor import Params, Tensor  # noqa: F401
from .trainer import Trainer, evaluate, run_training, select_action  # noqa: F401

__version__ = "0.1.0"

__all__ = [
    "ARCHITECTURES", "ArchitectureMismatchError", "Catch", "Checkpoint", "CheckpointCRCError",
    "CheckpointError", "CheckpointMagicError", "CheckpointVersionError", "load_checkpoint",
    "load_params_into", "save_checkpoint", "ConfigError", "EnvSpec", "EnvStep", "Environment", "GridWorld",
    "MetricRecord", "MetricsWriter", "PRESETS", "Preprocessor", "RecordCollector", "TabularChain",
    "Trainer", "bilinear_resize", "evaluate", "make_env", "preprocess_frame", "resolve_config",
    "run_training", "select_action", "DeepQError", "GeometryError", "LayerSpec",
    "LinearSchedule", "Network", "NonFiniteError", "Params", "PhaseOrderError",
    "PrioritizedReplay", "PriorityConfig", "ReplayMemory", "RmsProp", "RunConfig",
    "SampleBatch", "SumTree", "TdResult", "Tensor", "Transition", "anneal_beta",
    "build_network", "clip_gradients", "compute_target_double", "compute_target_dqn",
    "init_params", "learn_step", "load_params", "sync_target", "trunk_layers",
]
