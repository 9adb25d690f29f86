"""ctypes binding of libmcb.so (include/mcb.h).

This is the only place the package touches the native library.  There is no
CPU fallback: if the library is missing or no CUDA device is present, the
engine raises ``EngineUnavailableError`` instead of computing anything on the
host.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libmcb.so")

MCB_OK = 0
MCB_ERR_INVALID = 1
MCB_ERR_CAPACITY = 2
MCB_ERR_NO_EVICTABLE = 3
MCB_ERR_CUDA = 4
MCB_ERR_UNSUPPORTED = 5
MCB_ERR_NOMEM = 6
MCB_ERR_SHAPE = 7

MCB_LRU, MCB_LFU, MCB_BELADY, MCB_ML, MCB_ML_NO_PREFILL, MCB_FIFO, MCB_ARC, MCB_LECAR = range(8)
ML_CODES = (MCB_ML, MCB_ML_NO_PREFILL)
MCB_TUNE_SOLO_MIN = 0
MCB_TUNE_SEG_EV = 1
MCB_TUNE_SEG_NW = 2
MCB_TUNE_SEG_PASSES = 3
MCB_TUNE_GROUP_LANES = 4
MCB_TUNE_SERIAL = 5
MCB_TUNE_K3_CTAS = 6
MCB_TUNE_ML_CHUNKS = 7
MCB_TUNE_OVERLAP = 8
MCB_TUNE_WIDE_MIN = 9
MCB_TUNE_SEG_TSPEC = 10
MCB_TUNE_SCRATCH_BYTES = 11
MCB_TUNE_K3_TC = 12
MCB_TUNE_K3_TAU_PPB = 13
MCB_TUNE_K3_GROUPS = 14
MCB_TUNE_UPLOAD_PIECES = 16
R_PH, R_PM, R_DH, R_DM, R_COMP, R_EVICT, R_REFETCH, R_STATUS = range(8)
R_N = 8
OUT_HIT, OUT_MISS = 0xFFFF, 0xFFFE

EXPORTED_SYMBOLS = (
    "mcb_abi_version", "mcb_ctx_create", "mcb_ctx_destroy", "mcb_last_error", "mcb_last_stats",
    "mcb_set_timing", "mcb_last_timings", "mcb_set_tuning", "mcb_read_stats",
    "mcb_pack_trace", "mcb_validate_trace", "mcb_packed_view", "mcb_packed_positions", "mcb_packed_free",
    "mcb_replay", "mcb_replay_host", "mcb_next_use", "mcb_score", "mcb_router_topk", "mcb_ar1_hidden", "mcb_gen_reference",
    "mcb_comm_unique_id", "mcb_comm_init", "mcb_comm_allreduce_i64", "mcb_comm_destroy",
    "mcb_gen_reference_batch", "mcb_score_tc_scores", "mcb_last_chunks",
    "mcb_training_data", "mcb_set_lecar", "mcb_lecar_random", "mcb_pack_decode_ids",
    "mcb_eviction_duel", "mcb_train_epoch", "mcb_train_eval",
)


class EngineUnavailableError(RuntimeError):
    """libmcb.so or a CUDA device is missing; the engine has no CPU fallback."""


class MCBTrainData(ctypes.Structure):
    _fields_ = [("num_nets", ctypes.c_int32), ("num_experts", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("num_samples", ctypes.c_int64), ("features", ctypes.c_void_p),
                ("targets", ctypes.c_void_p), ("masks", ctypes.c_void_p)]


class MCBTrainCfg(ctypes.Structure):
    _fields_ = [("learning_rate", ctypes.c_double), ("weight_decay", ctypes.c_double),
                ("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("eps", ctypes.c_double),
                ("batch_size", ctypes.c_int64), ("n_train", ctypes.c_int64)]


class MCBTrace(ctypes.Structure):
    _fields_ = [
        ("num_layers", ctypes.c_int32),
        ("num_experts", ctypes.c_int32),
        ("top_k", ctypes.c_int32),
        ("num_traces", ctypes.c_int32),
        ("uniform", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("events_per_chain", ctypes.c_int64),
        ("total_acc", ctypes.c_int64),
        ("total_events", ctypes.c_int64),
        ("acc", ctypes.c_void_p),
        ("chain_acc_off", ctypes.c_void_p),
        ("chain_ev_off", ctypes.c_void_p),
        ("chain_rt_off", ctypes.c_void_p),
        ("ev_info", ctypes.c_void_p),
        ("routed", ctypes.c_void_p),
    ]


class MCBCost(ctypes.Structure):
    _fields_ = [
        ("t_load_s", ctypes.c_double),
        ("t_compute_s", ctypes.c_double),
        ("ml_score_cost_s", ctypes.c_double),
        ("loads_serial", ctypes.c_int32),
        ("window", ctypes.c_int32),
    ]


class MCBNets(ctypes.Structure):
    _fields_ = [
        ("num_experts", ctypes.c_int32),
        ("hidden", ctypes.c_int32),
        ("num_nets", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("params", ctypes.c_void_p),
    ]


class MCBOutputs(ctypes.Structure):
    _fields_ = [
        ("reports", ctypes.c_void_p),
        ("latency", ctypes.c_void_p),
        ("chain_reports", ctypes.c_void_p),
        ("hashes", ctypes.c_void_p),
        ("outcomes", ctypes.c_void_p),
        ("chain_latency", ctypes.c_void_p),
    ]


_lock = threading.Lock()
_lib = None


def load_library():
    """Load libmcb.so (building it first if this is a source checkout)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise EngineUnavailableError(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        sig = {
            "mcb_abi_version": ([], ctypes.c_int),
            "mcb_ctx_create": ([ctypes.c_int, P], ctypes.c_int),
            "mcb_ctx_destroy": ([P], ctypes.c_int),
            "mcb_last_error": ([ctypes.c_char_p, ctypes.c_size_t], ctypes.c_int),
            "mcb_last_stats": ([P, P, P], ctypes.c_int),
            "mcb_pack_trace": ([i32, i32, i32, i64, P, P, P, P, P, P, P], ctypes.c_int),
            "mcb_validate_trace": ([i32, i32, i32, i64, P, P, P, P, P, P], ctypes.c_int),
            "mcb_packed_view": ([P, P, P, P, P, P], ctypes.c_int),
            "mcb_packed_positions": ([P, i64, P, P], ctypes.c_int),
            "mcb_packed_free": ([P], ctypes.c_int),
            "mcb_replay": ([P, P, P, i32, P, i32, P, P, P, P], ctypes.c_int),
            "mcb_replay_host": ([P, P, P, i32, P, i32, P, P, P, P], ctypes.c_int),
            "mcb_set_timing": ([P, i32], ctypes.c_int),
            "mcb_last_timings": ([P, P, i32], ctypes.c_int),
            "mcb_set_tuning": ([P, i32, i64], ctypes.c_int),
            "mcb_read_stats": ([P, P, i32], ctypes.c_int),
            "mcb_next_use": ([P, P, P, P], ctypes.c_int),
            "mcb_score": ([P, P, P, i32, P, P, P], ctypes.c_int),
            "mcb_router_topk": ([P, P, P, i64, i32, i32, i32, i32, P, P, P], ctypes.c_int),
            "mcb_ar1_hidden": ([P, i64, i32, i32, ctypes.c_double, ctypes.c_uint64, P, P], ctypes.c_int),
            "mcb_comm_unique_id": ([P, i32], ctypes.c_int),
            "mcb_comm_init": ([P, i32, i32, P], ctypes.c_int),
            "mcb_comm_allreduce_i64": ([P, P, i64, P], ctypes.c_int),
            "mcb_comm_destroy": ([P], ctypes.c_int),
            "mcb_training_data": ([P, P, i32, i32, i32, P, P, P, P], ctypes.c_int),
            "mcb_set_lecar": ([P, ctypes.c_double, ctypes.c_double, i64], ctypes.c_int),
            "mcb_lecar_random": ([i64, i64, P], ctypes.c_int),
            "mcb_pack_decode_ids": ([P, P, i64, i64, i32, i32, i32, P, P, P], ctypes.c_int),
            "mcb_eviction_duel": ([P, P, P, P, P, P, P], ctypes.c_int),
            "mcb_train_epoch": ([P, P, P, P, P, P, i64, i64, P, P, P], ctypes.c_int),
            "mcb_train_eval": ([P, P, P, i64, i64, P, P], ctypes.c_int),
            "mcb_gen_reference_batch": ([P, i32, i32, i32, i64, i64, i32, ctypes.c_double, P, P, P, P], i32),
            "mcb_score_tc_scores": ([P, P, P, P, P, P], i32),
            "mcb_last_chunks": ([P, P], i32),
            "mcb_gen_reference": ([P, i32, i32, i32, i64, i64, i64, i32, ctypes.c_double, P, P, P, P],
                                  ctypes.c_int),
        }
        for name, (argt, rest) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = argt
            fn.restype = rest
        _lib = lib
        return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load_library().mcb_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


_contexts: dict[int, ctypes.c_void_p] = {}


def context(device: int = 0) -> ctypes.c_void_p:
    """Per-device engine context (created lazily, lives for the process)."""
    with _lock:
        ctx = _contexts.get(device)
    if ctx is not None:
        return ctx
    lib = load_library()
    try:
        import torch
        if not torch.cuda.is_available():
            raise EngineUnavailableError("no CUDA device: the B200 engine has no CPU fallback")
    except ImportError:  # pragma: no cover - torch is part of the image
        pass
    h = ctypes.c_void_p()
    rc = lib.mcb_ctx_create(device, ctypes.byref(h))
    if rc != MCB_OK:
        raise EngineUnavailableError(f"mcb_ctx_create failed: {last_error()}")
    with _lock:
        _contexts[device] = h
    return h


def read_stats(device: int = 0) -> list:
    """Device counters of the last replay: [uncertain scorer events, segmented
    fix-up events, unconverged segments, segments walked, ...]."""
    out = (ctypes.c_int64 * 8)()
    check(load_library().mcb_read_stats(context(device), out, 8))
    return list(out)


def set_lecar(learning_rate: float, discount_base: float, seed: int, device: int = 0):
    """LeCaR parameters for the MCB_LECAR cells of the following replays."""
    check(load_library().mcb_set_lecar(context(device), float(learning_rate), float(discount_base), int(seed)))


def lecar_random(seed: int, n: int):
    """CPython random.Random(seed).random() x n, as the engine materialises it (host only)."""
    import numpy as np
    out = np.zeros(max(int(n), 1), dtype=np.float64)
    check(load_library().mcb_lecar_random(int(seed), int(n), out.ctypes.data))
    return out[:n]


def last_chunks(device: int = 0) -> int:
    """Trace ranges the last replay on this device's context was split into."""
    n = ctypes.c_int64()
    check(load_library().mcb_last_chunks(context(device), ctypes.byref(n)))
    return int(n.value)


def set_tuning(knob: int, value: int, device: int = 0):
    check(load_library().mcb_set_tuning(context(device), knob, value))


def check(rc: int, errors: dict | None = None):
    """Map a status code onto the reference's exception types."""
    if rc == MCB_OK:
        return
    msg = last_error()
    from .engine import CapacityTooSmallError, SimulationError
    from .policies import NoEvictableError
    from .trace import InvalidConfigError
    if rc == MCB_ERR_CAPACITY:
        raise CapacityTooSmallError(msg)
    if rc == MCB_ERR_NO_EVICTABLE:
        raise NoEvictableError(msg)
    if rc == MCB_ERR_SHAPE:
        raise ValueError(msg)
    if rc == MCB_ERR_INVALID:
        if errors and "invalid" in errors:
            raise errors["invalid"](msg)
        raise InvalidConfigError(msg)
    if rc == MCB_ERR_UNSUPPORTED:
        raise SimulationError(f"unsupported by the B200 engine: {msg}")
    if rc == MCB_ERR_CUDA:
        raise RuntimeError(f"CUDA failure in libmcb: {msg}")
    raise RuntimeError(f"libmcb error {rc}: {msg}")
