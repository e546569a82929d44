"""B200-native particle mover + charge deposition for the picmc/BIT1 hot path.

Public surface (mirrors the reference's names where it replaces them):
  backends / backend  -- `cuda` kernels with picmc.backends signatures
  run_simulation      -- step driver (pkg/src/picmc/harness.py:105)
  Engine              -- device-resident engine (one GPU's shard)
  CanonicalEngine     -- reference slot order + Monte Carlo collisions
  collisions          -- collision_phase / Roles / step_stream_key
  RunConfig, load_config, Grid1D, SpeciesDef, PhysicalConstants
"""

from . import backends
from .config import CollisionRates, CollisionSetup, RunConfig, config_from_dict, load_config
from .core import Grid1D, PhysicalConstants, SpeciesDef
from .engine import PHASE_KEYS, Engine, Partition, partition_cells, reduce_bins
from .errors import CflViolation, ConfigError, ContractViolation, EngineError, InitError
from .harness import CollisionTally, RunMetrics, run_simulation
from .canonical import CanonicalEngine
from . import cellstore, collisions, fields, mover

__version__ = "0.1.0"

__all__ = [
    "CanonicalEngine", "CflViolation", "CollisionRates", "CollisionSetup", "CollisionTally", "ConfigError",
    "ContractViolation", "Engine", "EngineError", "Grid1D", "InitError", "PHASE_KEYS",
    "Partition", "PhysicalConstants", "RunConfig", "RunMetrics", "SpeciesDef", "backends",
    "collisions", "config_from_dict", "load_config", "partition_cells", "reduce_bins", "run_simulation",
]
