"""B200-native expert-cache replay engine (FlashMoE, arXiv 2601.17063).

Drop-in for the reference simulator's hot path (moecache: simulate /
run_simulation / sweep / policy_factory -> SimReport), backed by hand-written
sm_100a CUDA kernels behind the C ABI of include/mcb.h (libmcb.so).
"""
from .engine import (
    POLICY_NAMES,
    CapacityTooSmallError,
    CostModel,
    EvictionRecord,
    HardwareBudget,
    SimReport,
    SimRun,
    SimulationError,
    cache_size_calc,
    eviction_quality_duel,
    policy_factory,
    refetch_rate,
    run_simulation,
    simulate,
    step_latency_s,
    sweep,
)
from .dataset import DEFAULT_DISTANCE_CAP, LayerDataset, build_training_data
from .distributed import replay_sharded, sweep_sharded
from .net import EvictionNet, NetError, ShapeMismatchError, load_net, save_net
from .policies import NoEvictableError, PolicyDecision, PolicyError, lecar_update
from .refgen import SyntheticWorkloadConfig, expert_popularity, generate_trace
from .trace import (
    AccessEvent,
    HeaderMismatchError,
    InsufficientTokensError,
    InvalidConfigError,
    PackedTrace,
    Phase,
    RoutingTrace,
    TraceError,
    TraceHeader,
    TraceParseError,
    pack_trace,
    packed_from_decode_ids,
    prefill_coverage,
)

from .train import (
    EmptyDatasetError,
    NonFiniteLossError,
    TrainConfig,
    TrainResult,
    masked_mse,
    train_eviction_net,
    train_eviction_nets,
)
from .tracefile import (
    load_packed,
    parse_trace,
    read_trace,
    read_trace_binary,
    trace_to_text,
    write_batch_binary,
    write_trace,
    write_trace_binary,
)

__version__ = "0.1.0"
