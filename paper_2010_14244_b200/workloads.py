"""The five BASELINE.json configurations as engine workloads.

Each builder returns (network, SimConfig, DistanceDesc, keepalive).  The
keepalive holds arrays the descriptors point into.  C2 is the bench
metric's configuration; the others are exercised by `bench.py --config`
and the parity tests.  All are colony (GMACO-P) runs: preemptive signals,
Philox ants, congestion-modified roulette and tour cost, best-tour deposit,
congestion evaporation.
"""
from __future__ import annotations

import numpy as np

from . import abi, networks


def _colony(vehicles: int, ants: int, seed: int, max_steps: int, **kw) -> abi.SimConfig:
    cfg = abi.default_config(algorithm="colony", controller="preemptive", vehicle_count=vehicles,
                             seed=seed, max_steps=max_steps, **kw)
    return abi.colony_production(cfg, ants=ants)


def c1(seed=1, max_steps=100, vehicles=100):
    """10x10 grid, 100 vehicles, 20 ants/colony, 100 iterations, MACO-P preemption."""
    net = networks.grid(10, 10)
    return net, _colony(vehicles, 20, seed, max_steps), net.grid_distance(), None


def c2(seed=1, max_steps=200, vehicles=1000):
    """32x32 grid with signals at every intersection, 1,000 vehicles, 64 ants/colony."""
    net = networks.grid(32, 32, signals="all")
    return net, _colony(vehicles, 64, seed, max_steps), net.grid_distance(), None


def c3(seed=1, max_steps=200, vehicles=10000):
    """100x100 grid, 10,000 vehicles, 128 ants/colony, congestion-modified pheromone."""
    net = networks.grid(100, 100)
    return net, _colony(vehicles, 128, seed, max_steps), net.grid_distance(), None


def c4(seed=1, max_steps=50, vehicles=100000, nodes=1_000_000, targets=64, ants=16, max_hops=4096):
    """Random-geometric road graph, 1M nodes / ~4M directed edges, 100,000 vehicles.

    Distances: exact reverse-Dijkstra tables to a bounded destination set of
    `targets` nodes (GMACO_DIST_TARGETS); vehicles' destinations lie in it."""
    net = networks.random_geometric(nodes, k=3, seed=20250810, links=2 * nodes)
    rng = np.random.default_rng(seed)
    tgt = np.sort(rng.choice(nodes, size=targets, replace=False)).astype(np.int32)
    dist = abi.DistanceDesc(kind=abi.DIST_TARGETS, targets=abi.ptr(tgt, __import__("ctypes").c_int32),
                            target_count=targets)
    cfg = _colony(vehicles, ants, seed, max_steps)
    cfg.colony.max_hops = max_hops
    return net, cfg, dist, tgt


def c5(seed=1, max_steps=200, vehicles=50000, ants=64):
    """Preemption stress: 256x256 grid, every intersection signalized, rush-hour
    OD matrix (80% of trips between a hotspot block and the centre block)."""
    R = 256
    net = networks.grid(R, R, signals="all")
    cfg = _colony(vehicles, ants, seed, max_steps)
    r, c = np.meshgrid(np.arange(R), np.arange(R), indexing="ij")
    hot = ((r < 24) & (c < 24)).ravel()                       # residential corner
    centre = ((abs(r - R // 2) < 12) & (abs(c - R // 2) < 12)).ravel()  # CBD
    a = np.nonzero(hot)[0].astype(np.int32)
    b = np.nonzero(centre)[0].astype(np.int32)
    keep = abi.Blocks(cfg, a, b, bias=0.8)
    return net, cfg, net.grid_distance(), keep


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
DESCRIPTIONS = {k: v.__doc__.splitlines()[0] for k, v in CONFIGS.items()}
