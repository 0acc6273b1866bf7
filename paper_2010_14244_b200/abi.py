"""ctypes mirror of include/gmaco.h (the C ABI of the engine).

Plain data only: struct layouts, enums and reference-default parameter
blocks (the defaults of PheromoneParams pheromone.hpp:23-42, SignalParams
signals.hpp:14-22, RoutingParams routing.hpp:14-23 and SimConfig
engine.hpp:29-50).  The engine library itself is loaded by
:mod:`paper_2010_14244_b200.engine`.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

PHASES = 8

# enum gmaco_algorithm (engine.hpp:17 + colony)
DIJKSTRA, ACO, MACO, MACO_P, COLONY = 0, 1, 2, 3, 4
ALGORITHMS = {"dijkstra": DIJKSTRA, "aco": ACO, "maco": MACO, "maco-p": MACO_P, "colony": COLONY}
# enum gmaco_controller (engine.hpp:18)
FIXED, ADAPTIVE, PREEMPTIVE = 0, 1, 2
CONTROLLERS = {"fixed": FIXED, "adaptive": ADAPTIVE, "preemptive": PREEMPTIVE}
ALL_AT_START, UNIFORM_WINDOW = 0, 1
OD_UNIFORM, OD_BLOCKS = 0, 1
DEV_GLOBAL, DEV_EDGE_OCCUPANCY = 0, 1
RNG_PHILOX, RNG_REFERENCE = 0, 1
DEPOSIT_COMPLETION, DEPOSIT_BEST_TOUR, DEPOSIT_NONE = 0, 1, 2
PENDING, AT_NODE, ON_EDGE, QUEUED, ARRIVED, RETIRED = range(6)
DIST_DENSE, DIST_GRID, DIST_TARGETS = 0, 1, 2

OK, EVALIDATION, ERUNTIME = 0, 1, 2


class PheromoneParams(C.Structure):
    _fields_ = [
        ("tau_init_lo", C.c_double), ("tau_init_hi", C.c_double),
        ("delta_inc", C.c_double), ("delta_dec", C.c_double),
        ("rho", C.c_double), ("tau_min", C.c_double), ("tau_max", C.c_double),
        ("aco_deposit_q", C.c_double),
        ("decrement_siblings_only", C.c_int32), ("_pad", C.c_int32),
    ]


class SignalParams(C.Structure):
    _fields_ = [
        ("th_max", C.c_int32), ("fixed_cycle_order", C.c_int32 * PHASES), ("_pad", C.c_int32),
        ("t_max", C.c_double), ("green_duration_s", C.c_double), ("saturation_flow", C.c_double),
    ]


class RoutingParams(C.Structure):
    _fields_ = [
        ("deviation_threshold", C.c_int64), ("deviation_mode", C.c_int32),
        ("progress_filter", C.c_int32), ("aco_alpha", C.c_double), ("aco_beta", C.c_double),
    ]


class ColonyParams(C.Structure):
    _fields_ = [
        ("ants", C.c_int32), ("hop_limit", C.c_int32), ("max_hops", C.c_int32), ("rng", C.c_int32),
        ("congestion", C.c_int32), ("deposit", C.c_int32), ("congestion_evaporation", C.c_int32),
        ("replan_all", C.c_int32),
    ]


# gmaco_option_bits: implementation switches, results bit-identical (gmaco.h)
(OPT_NO_QUEUE, OPT_NO_SCRATCH, OPT_NO_TT, OPT_NO_ORDER, OPT_NO_PREFETCH, OPT_NO_PDL, OPT_NO_SMEM, OPT_NO_BITS,
 OPT_NO_E1_WALK, OPT_NATURAL_ROWS, OPT_PROFILE_CREATE, OPT_REDZONES) = (1 << i for i in range(12))


class EngineOptions(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("_pad", C.c_int32), ("sssp_delta", C.c_double)]


class SimConfig(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int32), ("controller", C.c_int32), ("vehicle_count", C.c_int32),
        ("spawn", C.c_int32), ("spawn_window_steps", C.c_int32), ("od_pattern", C.c_int32),
        ("dt_s", C.c_double), ("max_steps", C.c_int64), ("seed", C.c_uint64),
        ("decision_latency_s", C.c_double), ("od_bias", C.c_double),
        ("od_block_a", C.POINTER(C.c_int32)), ("od_block_b", C.POINTER(C.c_int32)),
        ("od_block_a_len", C.c_int32), ("od_block_b_len", C.c_int32),
        ("speed_min_mps", C.c_double), ("speed_max_mps", C.c_double),
        ("pheromone", PheromoneParams), ("signal", SignalParams), ("routing", RoutingParams),
        ("colony", ColonyParams), ("options", EngineOptions),
    ]


class GraphDesc(C.Structure):
    _fields_ = [
        ("node_count", C.c_int32), ("edge_count", C.c_int32),
        ("signalized", C.POINTER(C.c_uint8)), ("edge_from", C.POINTER(C.c_int32)),
        ("edge_to", C.POINTER(C.c_int32)), ("edge_length_mm", C.POINTER(C.c_int64)),
        ("edge_lanes", C.POINTER(C.c_int32)),
    ]


class DistanceDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("grid_rows", C.c_int32), ("grid_cols", C.c_int32),
        ("dist_mm", C.POINTER(C.c_int64)), ("targets", C.POINTER(C.c_int32)),
        ("target_count", C.c_int32), ("_pad", C.c_int32),
    ]


class RunResult(C.Structure):
    _fields_ = [
        ("mean_travel_s", C.c_double), ("mean_wait_s", C.c_double), ("mean_queue_len", C.c_double),
        ("max_edge_occupancy", C.c_int32), ("completed_count", C.c_int32),
        ("retired_count", C.c_int32), ("_pad", C.c_int32),
        ("steps_executed", C.c_int64), ("wall_clock_ms", C.c_int64),
    ]


_VEHICLE_FIELDS = [
    ("origin", np.int32), ("dest", np.int32), ("speed_mps", np.float64), ("advance_mm", np.int64),
    ("state", np.uint8), ("at_node", np.int32), ("on_edge", np.int32), ("progress_mm", np.int64),
    ("overshoot_mm", np.int64), ("queued_phase", np.int32), ("queue_joined_step", np.int64),
    ("depart_step", np.int64), ("arrive_step", np.int64), ("latency_debt_us", np.int64),
    ("driving_steps", np.int64), ("queued_steps", np.int64), ("latency_steps", np.int64),
    ("decisions", np.int32), ("deviations", np.int32), ("path_length_mm", np.int64),
]
_CT = {np.int32: C.c_int32, np.int64: C.c_int64, np.float64: C.c_double, np.uint8: C.c_uint8}
VEHICLE_FIELDS = [name for name, _ in _VEHICLE_FIELDS]


class VehicleView(C.Structure):
    _fields_ = [(name, C.POINTER(_CT[dt])) for name, dt in _VEHICLE_FIELDS]


_SIGNAL_FIELDS_S = [
    ("node", np.int32), ("green", np.int32), ("cycle_cursor", np.int32), ("discharge_lanes", np.int32),
    ("green_elapsed_steps", np.int64), ("green_elapsed_s", np.float64),
]
_SIGNAL_FIELDS_P = [("queue_len", np.int32), ("head_wait_s", np.float64), ("service_remainder", np.float64)]


class SignalView(C.Structure):
    _fields_ = (
        [(name, C.POINTER(_CT[dt])) for name, dt in _SIGNAL_FIELDS_S]
        + [(name, C.POINTER(_CT[dt])) for name, dt in _SIGNAL_FIELDS_P]
        + [("queue_vid", C.POINTER(C.c_int32)), ("queue_enqueue_step", C.POINTER(C.c_int64))]
    )


class Counters(C.Structure):
    _fields_ = [
        ("ant_steps", C.c_int64), ("vehicle_routes", C.c_int64), ("decisions", C.c_int64),
        ("candidates", C.c_int64), ("degree_sum", C.c_int64), ("kernels_per_step", C.c_int64),
        ("walk_bytes", C.c_int64),
    ]


def ptr(a: np.ndarray, ctype):
    """Pointer to a contiguous numpy array (caller keeps the array alive)."""
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ctype))


def default_config(**kw) -> SimConfig:
    """SimConfig with the reference defaults (engine.hpp:29-50 and the param
    structs), then `kw` overrides for top-level scalar fields."""
    c = SimConfig()
    c.algorithm = DIJKSTRA
    c.controller = FIXED
    c.vehicle_count = 1
    c.spawn = ALL_AT_START
    c.spawn_window_steps = 1
    c.od_pattern = OD_UNIFORM
    c.dt_s = 1.0
    c.max_steps = 5000
    c.seed = 0
    c.decision_latency_s = 0.0
    c.od_bias = 0.8
    c.speed_min_mps = 50.0
    c.speed_max_mps = 80.0
    p = c.pheromone
    p.tau_init_lo, p.tau_init_hi = 1.0, 10.0
    p.delta_inc, p.delta_dec = 1.0, 0.05
    p.rho, p.tau_min, p.tau_max, p.aco_deposit_q = 0.1, 0.0, 100.0, 100.0
    p.decrement_siblings_only = 0
    s = c.signal
    s.th_max = 10
    for i in range(PHASES):
        s.fixed_cycle_order[i] = i
    s.t_max, s.green_duration_s, s.saturation_flow = 120.0, 10.0, 0.5
    r = c.routing
    r.deviation_threshold, r.deviation_mode, r.progress_filter = 1000, DEV_GLOBAL, 1
    r.aco_alpha, r.aco_beta = 1.0, 2.0
    k = c.colony
    k.ants, k.hop_limit, k.max_hops, k.rng = 1, 0, 0, RNG_PHILOX
    k.congestion, k.deposit, k.congestion_evaporation, k.replan_all = 0, DEPOSIT_COMPLETION, 0, 0
    for key, val in kw.items():
        if key == "algorithm" and isinstance(val, str):
            val = ALGORITHMS[val]
        if key == "controller" and isinstance(val, str):
            val = CONTROLLERS[val]
        setattr(c, key, val)
    if "controller" not in kw:  # harness.cpp:63-72: maco-p ⇒ preemptive, others fixed
        c.controller = PREEMPTIVE if c.algorithm == MACO_P else FIXED
    return c


def colony_anchor(c: SimConfig) -> SimConfig:
    """Colony settings that reduce exactly to the reference ACO run."""
    k = c.colony
    k.ants, k.hop_limit, k.max_hops, k.rng = 1, 1, 0, RNG_REFERENCE
    k.congestion, k.deposit, k.congestion_evaporation, k.replan_all = 0, DEPOSIT_COMPLETION, 0, 0
    return c


def colony_production(c: SimConfig, ants: int) -> SimConfig:
    """GMACO-P colony settings of the bench workload."""
    k = c.colony
    k.ants, k.hop_limit, k.max_hops, k.rng = ants, 0, 0, RNG_PHILOX
    k.congestion, k.deposit, k.congestion_evaporation, k.replan_all = 1, DEPOSIT_BEST_TOUR, 1, 1
    return c


class Blocks:
    """Keeps OD block arrays alive while a SimConfig points at them."""

    def __init__(self, cfg: SimConfig, a, b, bias=0.8):
        self.a = np.ascontiguousarray(a, dtype=np.int32)
        self.b = np.ascontiguousarray(b, dtype=np.int32)
        cfg.od_pattern = OD_BLOCKS
        cfg.od_bias = bias
        cfg.od_block_a = ptr(self.a, C.c_int32)
        cfg.od_block_b = ptr(self.b, C.c_int32)
        cfg.od_block_a_len = len(self.a)
        cfg.od_block_b_len = len(self.b)


def vehicle_arrays(n: int):
    arrs = {name: np.zeros(n, dtype=dt) for name, dt in _VEHICLE_FIELDS}
    view = VehicleView(**{name: ptr(arrs[name], _CT[dt]) for name, dt in _VEHICLE_FIELDS})
    return arrs, view


def signal_arrays(n_signals: int, queue_cap: int):
    arrs = {name: np.zeros(n_signals, dtype=dt) for name, dt in _SIGNAL_FIELDS_S}
    arrs.update({name: np.zeros(n_signals * PHASES, dtype=dt) for name, dt in _SIGNAL_FIELDS_P})
    arrs["queue_vid"] = np.zeros(max(queue_cap, 1), dtype=np.int32)
    arrs["queue_enqueue_step"] = np.zeros(max(queue_cap, 1), dtype=np.int64)
    view = SignalView(**{name: ptr(a, _CT[a.dtype.type]) for name, a in arrs.items()})
    return arrs, view
