"""B200-native AMaze + PLR hot path (drop-in for autocurricula's env/level/scoring path).

Hand-written sm_100a CUDA kernels behind a C ABI (include/amaze_b200.h,
libamaze_b200.so), reached through ctypes; torch tensors carry data to and from the
policy.  See DESIGN.md.
"""

__version__ = "0.1.0"

from .amaze import (EnvMetrics, MazeEnv, check_levels, env_metrics, level_metrics, mutate_level, mutate_levels,
                    sample_levels, sample_random_level)
from .batch import HOME, RESAMPLE, AutoResetWrapper, VectorBatchEnv, batch_lift
from .core import BatchShape, StaticParams, StepResult
from .errors import (AutocurriculaError, ConfigError, ContractViolation, LevelError, LevelParseError, RunnerFault,
                     ShapeError)
from .gae import compute_gae, gae_and_scores, per_lane_episode_stats
from .host import pinned_empty
from .level import MazeLevel, decode_level, encode_level, pack_levels, unpack_levels
from .rng import RngStream
from .policy import GraphRollout, TorchPolicyActor, policy_head, rollout, sample_actions
from .rollout import RolloutCursor, TrajectoryBatch, random_actions, rollout_actions
from .scoring import lane_scores, score_maxmc, score_pvl
from .teacher import TeacherBatchEnv, TeacherEnv
