"""The engine's own memcheck (compute-sanitizer is closed on the GPU pool):
worlds created with abi.OPT_REDZONES put 1 KiB guard bands of 0xA5 around
every device array (arena arrays: behind them); after running each kernel
family the guards must be intact, and the results must still equal the
oracle (the guards shift every arena array, so any layout-dependent
out-of-bounds READ would show up as a parity failure as well)."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks, sharding
from paper_2010_14244_b200.engine import Engine

pytestmark = pytest.mark.gpu


def checked(cfg, flags=0):
    cfg.options.flags = abi.OPT_REDZONES | flags
    return cfg


def guards_ok(e):
    bad, msg = e.check_redzones()
    assert bad == 0, msg
    assert "guards intact" in msg
    return int(msg.split()[0])


def same_as_oracle(gpu, cpu):
    assert np.array_equal(gpu.pheromone(), cpu.pheromone())
    va, vb = gpu.vehicles(), cpu.vehicles()
    for f in abi.VEHICLE_FIELDS:
        assert np.array_equal(va[f], vb[f]), f


@pytest.mark.parametrize("alg", ["dijkstra", "aco", "maco", "maco-p"])
def test_reference_algorithms_guarded(alg):
    net = networks.grid(10, 10)
    cfg = checked(abi.default_config(algorithm=alg, vehicle_count=100, seed=1))
    ref = O.PortWorld(net, cfg).run()
    for dist in (net.grid_distance(), abi.DistanceDesc(kind=abi.DIST_DENSE)):  # closed form / device SSSP
        e = Engine(net, cfg, dist)
        assert O.results_identical(e.run(), ref)
        assert guards_ok(e) > 20


def test_lattice_colony_and_snapshots_guarded():
    net = networks.grid(32, 32, signals="all")
    cfg = checked(abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive",
                                                           vehicle_count=1000, seed=1, max_steps=80), ants=64))
    gpu, cpu = Engine(net, cfg, net.grid_distance()), O.PortWorld(net, cfg, net.grid_distance())
    V = cfg.vehicle_count
    bufs = [np.zeros(V, np.int64) for _ in range(2)]
    for k in range(60):  # direct launches, then the captured snapshot graphs
        gpu.step_snapshot(abi.VehicleView(progress_mm=abi.ptr(bufs[k & 1], C.c_int64)), k & 1)
        if k:
            gpu.vehicles_wait((k - 1) & 1, abi.VehicleView(progress_mm=abi.ptr(bufs[(k - 1) & 1], C.c_int64)))
    gpu.vehicles_wait(1, abi.VehicleView(progress_mm=abi.ptr(bufs[1], C.c_int64)))
    cpu.step(60)
    same_as_oracle(gpu, cpu)
    gpu.signals()
    guards_ok(gpu)


def _rgg(nodes, targets, seed):
    net = networks.random_geometric(nodes, k=3, seed=seed)
    tgt = np.sort(np.random.default_rng(seed).choice(nodes, size=targets, replace=False)).astype(np.int32)
    return net, tgt


@pytest.mark.parametrize("flags", [0, abi.OPT_NO_TT, abi.OPT_NO_QUEUE, abi.OPT_NO_SCRATCH])
def test_general_graph_walkers_guarded(flags):
    """Per-target queue walker (k_tt_*, k_colony_pro/qt/epi), shared-record
    queue walker, block walker and replay mode, with the device SSSP."""
    net, tgt = _rgg(3000, 12, 77)
    dist = abi.DistanceDesc(kind=abi.DIST_TARGETS, targets=abi.ptr(tgt, C.c_int32), target_count=len(tgt))
    cfg = checked(abi.colony_production(abi.default_config(algorithm="colony", vehicle_count=400, seed=5,
                                                           max_steps=30), ants=16), flags)
    cfg.colony.max_hops = 512
    gpu, cpu = Engine(net, cfg, dist), O.PortWorld(net, cfg, dist)
    gpu.step(6)
    cpu.step(6)
    same_as_oracle(gpu, cpu)
    for vid in range(0, 400, 13):
        assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True))
    guards_ok(gpu)


def test_generic_walker_and_queries_guarded():
    from test_gpu_parity import _hub_graph
    net = _hub_graph(20)
    cfg = checked(abi.colony_production(abi.default_config(algorithm="colony", vehicle_count=200, seed=3,
                                                           max_steps=30), ants=32))
    gpu, cpu = Engine(net, cfg), O.PortWorld(net, cfg)
    gpu.step(5)
    cpu.step(5)
    same_as_oracle(gpu, cpu)
    rng = np.random.default_rng(2)
    cur = rng.integers(0, net.node_count, 300)
    dst = (cur + 1 + rng.integers(0, net.node_count - 2, 300)) % net.node_count
    for alg in (abi.DIJKSTRA, abi.ACO, abi.MACO):
        a = gpu.next_node(alg, cur, dst, None, None, 7)
        b = cpu.next_node(alg, cur, dst, None, None, 7)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    gpu.set_pheromone(cpu.pheromone())
    guards_ok(gpu)


def test_sharded_maco_p_guarded():
    net = networks.grid(12, 12, signals="all")
    cfg = checked(abi.default_config(algorithm="maco-p", vehicle_count=301, seed=5, max_steps=60))
    shards = []
    for r in range(2):
        e = Engine(net, cfg, net.grid_distance())
        e.set_shard(*sharding.shard_bounds(301, 2, r))
        shards.append(e)
    step = sharding.local_transport(shards)
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    for _ in range(30):
        step()
        cpu.step(1)
    for e in shards:
        same_as_oracle(e, cpu)
        guards_ok(e)


def _digest(e):
    import hashlib
    h = hashlib.sha256()
    v = e.vehicles()
    for f in abi.VEHICLE_FIELDS:
        h.update(np.ascontiguousarray(v[f]).tobytes())
    h.update(e.pheromone().tobytes())
    h.update(e.occupancy().tobytes())
    s = e.signals()
    for f in sorted(s):
        h.update(np.ascontiguousarray(s[f]).tobytes())
    return h.hexdigest()


def test_repeated_runs_bit_identical():
    """Race evidence without racecheck: the kernels with dynamic scheduling
    (ant queue with atomic fetch, atomicMin argmins, atomic deposits, the
    concurrent signal CTAs, last-block finalization, PDL tails) give the same
    bits on every repetition."""
    net = networks.grid(32, 32, signals="all")
    cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive",
                                                   vehicle_count=1000, seed=2, max_steps=100), ants=64)
    rg, tgt = _rgg(3000, 12, 5)
    dist = abi.DistanceDesc(kind=abi.DIST_TARGETS, targets=abi.ptr(tgt, C.c_int32), target_count=len(tgt))
    cfg2 = abi.colony_production(abi.default_config(algorithm="colony", vehicle_count=600, seed=4, max_steps=40),
                                 ants=16)
    cfg2.colony.max_hops = 512
    for make, steps in ((lambda: Engine(net, cfg, net.grid_distance()), 40), (lambda: Engine(rg, cfg2, dist), 12)):
        ds = set()
        for _ in range(5):
            e = make()
            e.step(steps)
            ds.add(_digest(e))
            e.close()
        assert len(ds) == 1
