"""Parity at the benchmarked shapes: the configurations behind the bench
lines (BASELINE.json configs, paper_2010_14244_b200/workloads.py) run on the
device exactly as benchmarked -- same walker, same table layouts, same
fleet/ant counts -- and compared with the oracle after each iteration:
pheromone field, occupancy, every vehicle field, every signal field, the
work counters and sampled best-of-K planned tours.

* C3 exactly: 100x100 grid, 10,000 vehicles, 128 ants (one-vehicle CTAs of
  the lattice walker, multi-word move bits).
* C5 exactly: 256x256 all-signalized grid, the rush-hour Blocks OD (bias
  0.8), 64 ants, the bench's 50,000-vehicle fleet.
* C4 exactly: the 1M-node / 4M-edge random-geometric graph, 64 targets,
  max_hops 4096, 16 ants, the bench's 100,000-vehicle fleet (per-target
  candidate rows, BFS row order, longest-band-first queue, ant-queue walker).
  The oracle plans the vehicles of a step on all host threads.
* alpha not in {0, 1}: tau^alpha comes from the exact glibc-pow table
  (DevWorld::taupow), so runs are bit-exact, not within-1-ulp.

Reference: R/src/routing.cpp:77-115, R/src/pheromone.cpp:61-90,
R/src/engine.cpp:352-400 (oracle/gmaco_oracle.c restates them).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks, workloads
from paper_2010_14244_b200.engine import Engine

pytestmark = pytest.mark.gpu

COUNTERS = ("ant_steps", "vehicle_routes", "decisions", "candidates", "degree_sum")


def same_world(gpu, cpu, where, route_stride):
    va, vb = gpu.vehicles(), cpu.vehicles()
    for f in abi.VEHICLE_FIELDS:
        assert np.array_equal(va[f], vb[f]), f"{where}: vehicle field {f}"
    sa, sb = gpu.signals(), cpu.signals()
    for f in sa:
        assert np.array_equal(sa[f], sb[f]), f"{where}: signal field {f}"
    assert np.array_equal(gpu.pheromone(), cpu.pheromone()), f"{where}: pheromone"
    assert np.array_equal(gpu.occupancy(), cpu.occupancy()), f"{where}: occupancy"
    a, b = gpu.counters(), cpu.counters()
    for f in COUNTERS:
        assert getattr(a, f) == getattr(b, f), f"{where}: counter {f}"
    V = len(va["state"])
    for vid in range(0, V, route_stride):
        assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), f"{where}: planned tour of {vid}"


def run_pair(net, cfg, dist, iters, route_stride, where):
    gpu = Engine(net, cfg, dist)
    cpu = O.PortWorld(net, cfg, dist)
    for it in range(iters):
        gpu.step(1)
        cpu.step(1)
        same_world(gpu, cpu, f"{where} iteration {it + 1}", route_stride)
    return gpu, cpu


def test_c3_exact_shape():
    net, cfg, dist, keep = workloads.c3(seed=1, max_steps=10)
    assert (net.node_count, cfg.vehicle_count, cfg.colony.ants) == (10_000, 10_000, 128)
    gpu, _ = run_pair(net, cfg, dist, 2, 97, "C3")
    assert gpu.counters().ant_steps > 10_000 * 128 * 50  # full-length walks happened
    del keep


def test_c5_exact_shape():
    net, cfg, dist, keep = workloads.c5(seed=1, max_steps=10)
    assert cfg.vehicle_count == 50_000
    assert net.node_count == 256 * 256 and cfg.od_pattern == abi.OD_BLOCKS and cfg.od_bias == 0.8
    assert cfg.colony.ants == 64
    run_pair(net, cfg, dist, 2, 499, "C5")
    del keep


def test_c4_exact_shape():
    net, cfg, dist, keep = workloads.c4(seed=1, max_steps=10)
    assert net.node_count == 1_000_000 and net.edge_count >= 4_000_000 and cfg.vehicle_count == 100_000
    assert cfg.colony.max_hops == 4096 and cfg.colony.ants == 16 and dist.target_count == 64
    gpu, _ = run_pair(net, cfg, dist, 2, 997, "C4")
    assert gpu.counters().ant_steps > 100_000 * 16 * 500


@pytest.mark.parametrize("alpha", [0.5, 2.0])
@pytest.mark.parametrize("alg", ["aco", "maco-p"])
def test_alpha_reference_algorithms_exact(alg, alpha):
    """ACO weights pow(tau, alpha) * pow(vis, beta) (routing.cpp:91-94) with
    alpha not in {0, 1}: whole runs identical to the oracle and to the
    compiled reference."""
    net = networks.grid(10, 10)
    for seed in (1, 2):
        cfg = abi.default_config(algorithm=alg, vehicle_count=100, seed=seed)
        cfg.routing.aco_alpha, cfg.routing.aco_beta = alpha, 1.5
        ref = O.PortWorld(net, cfg).run()
        got = Engine(net, cfg, net.grid_distance()).run()
        assert O.results_identical(got, ref), (alg, alpha, seed)
        if O.ref_available():
            assert O.results_identical(O.ref_run(net, cfg), ref)


@pytest.mark.parametrize("alpha", [0.5, 2.0])
def test_alpha_colony_exact(alpha):
    """GMACO-P colonies (congestion-penalised roulette) with alpha not in
    {0, 1}, on the lattice walker and on the general-graph queue walker."""
    net = networks.grid(16, 16, signals="all")
    cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive",
                                                   vehicle_count=300, seed=3, max_steps=40), ants=32)
    cfg.routing.aco_alpha = alpha
    run_pair(net, cfg, net.grid_distance(), 3, 3, f"lattice alpha={alpha}")
    rg = networks.random_geometric(2500, k=3, seed=41)
    tgt = np.sort(np.random.default_rng(41).choice(2500, size=10, replace=False)).astype(np.int32)
    import ctypes as C
    dist = abi.DistanceDesc(kind=abi.DIST_TARGETS, targets=abi.ptr(tgt, C.c_int32), target_count=10)
    cfg = abi.colony_production(abi.default_config(algorithm="colony", vehicle_count=250, seed=5,
                                                   max_steps=40), ants=16)
    cfg.routing.aco_alpha = alpha
    cfg.colony.max_hops = 512
    run_pair(rg, cfg, dist, 3, 5, f"rgg alpha={alpha}")
