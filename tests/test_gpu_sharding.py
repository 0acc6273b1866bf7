"""Sharded colonies on the device: engines that each plan one vehicle shard
and exchange decision records + deposits must reproduce the unsharded
world bit for bit — through the host-mediated exchange (several engines on
one GPU, stepping in lockstep, so no kernel waits on another) and through
the engine's own NCCL exchange (world size 1 on the single available GPU)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks, sharding
from paper_2010_14244_b200.engine import Engine

pytestmark = pytest.mark.gpu


def world(V=301, ants=16, rows=12):
    net = networks.grid(rows, rows, signals="all")
    cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive",
                                                   vehicle_count=V, seed=5, max_steps=80), ants=ants)
    return net, cfg


def same(a, b):
    va, vb = a.vehicles(), b.vehicles()
    for f in abi.VEHICLE_FIELDS:
        if not np.array_equal(va[f], vb[f]):
            return f
    sa, sb = a.signals(), b.signals()
    for f in sa:
        if not np.array_equal(sa[f], sb[f]):
            return f
    if not np.array_equal(a.pheromone(), b.pheromone()):
        return "pheromone"
    if not np.array_equal(a.occupancy(), b.occupancy()):
        return "occupancy"
    return None


@pytest.mark.parametrize("nshards", [2, 3])
def test_host_mediated_shards_equal_unsharded(nshards):
    net, cfg = world()
    single = Engine(net, cfg, net.grid_distance())
    shards = []
    for r in range(nshards):
        e = Engine(net, cfg, net.grid_distance())
        e.set_shard(*sharding.shard_bounds(cfg.vehicle_count, nshards, r))
        shards.append(e)
    step = sharding.local_transport(shards)
    for k in range(10):
        step()
        single.step(1)
        for e in shards:
            assert same(e, single) is None, (k, same(e, single))
    assert sum(e.counters().ant_steps for e in shards) == single.counters().ant_steps
    # run to completion: every rank must agree on the step count and on
    # finished() (the NCCL path relies on it: no rank may stop early)
    while not single.finished():
        step()
        single.step(1)
        for e in shards:
            assert e.current_step() == single.current_step()
            assert e.finished() == single.finished()
        assert sum(e.counters().decisions for e in shards) == single.counters().decisions
    assert O.results_identical(shards[0].collect(), single.collect())


def test_mixed_engine_and_oracle_shards():
    """A GPU shard and an oracle shard exchanging records (edge ids at the
    boundary) still equal the unsharded oracle world."""
    net, cfg = world(V=200)
    cpu_single = O.PortWorld(net, cfg, net.grid_distance())
    g = Engine(net, cfg, net.grid_distance())
    g.set_shard(*sharding.shard_bounds(200, 2, 0))
    c = O.PortWorld(net, cfg, net.grid_distance())
    c.set_shard(*sharding.shard_bounds(200, 2, 1))
    step = sharding.local_transport([g, c])
    for _ in range(8):
        step()
        cpu_single.step(1)
    assert same(g, cpu_single) is None
    assert same(c, cpu_single) is None


def test_nccl_exchange_world1_equals_unsharded():
    from paper_2010_14244_b200 import engine
    import ctypes as C
    net, cfg = world(V=1000, ants=64, rows=32)
    uid = C.create_string_buffer(128)
    assert engine.load().gmaco_nccl_unique_id(uid) == 0
    e = Engine(net, cfg, net.grid_distance())
    e.attach_comm(0, 1, uid.raw)
    single = Engine(net, cfg, net.grid_distance())
    e.step(6)
    single.step(6)
    assert same(e, single) is None
    assert e.counters().ant_steps == single.counters().ant_steps


def _walker_world(kind):
    """(net, cfg, dist factory) per stage-B walker kind."""
    from test_gpu_parity import _hub_graph, _rgg_targets
    prod = lambda V, ants, steps: abi.colony_production(abi.default_config(
        algorithm="colony", controller="preemptive", vehicle_count=V, seed=9, max_steps=steps), ants=ants)
    if kind == "lattice-multiword":
        net = networks.grid(40, 40, signals="interior")
        return net, prod(240, 64, 30), net.grid_distance
    if kind in ("queue", "block"):
        net, _, tgt = _rgg_targets(3000, 12, 77)
        cfg = prod(300, 16, 30)
        cfg.colony.max_hops = 512
        cfg.options.flags = abi.OPT_NO_QUEUE if kind == "block" else 0
        make = lambda: abi.DistanceDesc(kind=abi.DIST_TARGETS, targets=abi.ptr(tgt, __import__("ctypes").c_int32),
                                        target_count=len(tgt))
        return net, cfg, make, tgt
    if kind == "generic":
        net = _hub_graph(20)
        return net, prod(200, 32, 30), lambda: abi.DistanceDesc(kind=abi.DIST_DENSE)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["lattice-multiword", "queue", "block", "generic"])
def test_host_mediated_shards_every_walker(kind):
    """Sharded stage B on each walker (prologue / queue / epilogue decision
    records included) equals the unsharded engine, step by step."""
    spec = _walker_world(kind)
    net, cfg, dist = spec[:3]
    keep = spec[3:]  # target arrays referenced by the descriptors
    single = Engine(net, cfg, dist())
    shards = []
    for r in range(3):
        e = Engine(net, cfg, dist())
        e.set_shard(*sharding.shard_bounds(cfg.vehicle_count, 3, r))
        shards.append(e)
    step = sharding.local_transport(shards)
    for k in range(6):
        step()
        single.step(1)
        for e in shards:
            assert same(e, single) is None, (kind, k, same(e, single))
    assert sum(e.counters().ant_steps for e in shards) == single.counters().ant_steps
    del keep


def test_nccl_communicator_shared_by_engines_of_a_job():
    """Engines attaching with the same (rank, world, id) reuse one
    communicator (the first attach creates it; a unique id is single-use for
    ncclCommInitRank), one live engine at a time: a second attach while the
    holder is alive is refused (status 1), since two engines capturing
    collectives on one communicator could interleave them differently on
    different ranks.  After the holder is closed the next engine reuses it and
    still equals the unsharded engine."""
    from paper_2010_14244_b200 import engine
    import ctypes as C
    net, cfg = world(V=300, ants=32, rows=16)
    uid = C.create_string_buffer(128)
    assert engine.load().gmaco_nccl_unique_id(uid) == 0
    single = Engine(net, cfg, net.grid_distance())
    single.step(5)
    first = Engine(net, cfg, net.grid_distance())
    first.attach_comm(0, 1, uid.raw)
    first.step(5)
    assert same(first, single) is None
    second = Engine(net, cfg, net.grid_distance())
    with pytest.raises(engine.EngineError) as ei:
        second.attach_comm(0, 1, uid.raw)
    assert ei.value.code == 1 and "held by another live engine" in str(ei.value)
    first.close()
    second.attach_comm(0, 1, uid.raw)  # reuses the job's communicator
    second.step(5)
    assert same(second, single) is None


def ref_world(alg, V=301):
    net = networks.grid(12, 12, signals="all")
    cfg = abi.default_config(algorithm=alg.replace("-scoped", ""), vehicle_count=V, seed=5, max_steps=120)
    cfg.routing.deviation_threshold = 150  # MACO deviations happen early on
    cfg.pheromone.decrement_siblings_only = int(alg == "maco-scoped")
    return net, cfg


@pytest.mark.parametrize("alg", ["maco-p", "maco", "maco-scoped", "aco", "dijkstra"])
def test_reference_algorithms_shard(alg):
    """The reference's own algorithms sharded over 3 engines (k_decide over
    the shard, decision records with the deviation flag exchanged,
    k_apply_remote, replicated cooperative tail with the in-kernel position
    scan over every rank's decisions) equal the unsharded engine step by
    step and the unsharded oracle at the end."""
    net, cfg = ref_world(alg)
    single = Engine(net, cfg, net.grid_distance())
    shards = []
    for r in range(3):
        e = Engine(net, cfg, net.grid_distance())
        e.set_shard(*sharding.shard_bounds(cfg.vehicle_count, 3, r))
        shards.append(e)
    step = sharding.local_transport(shards)
    for k in range(25):
        step()
        single.step(1)
        for e in shards:
            assert same(e, single) is None, (alg, k, same(e, single))
    while not single.finished():
        step()
        single.step(1)
    for e in shards:
        assert e.finished() and e.current_step() == single.current_step()
    assert sum(e.counters().decisions for e in shards) == single.counters().decisions
    ref = O.PortWorld(net, cfg, net.grid_distance()).run()
    assert O.results_identical(shards[1].collect(), ref)
    if alg.startswith("maco"):
        assert single.vehicles()["deviations"].sum() > 0


def test_maco_p_mixed_engine_and_oracle_shards():
    """Edge-id records (deviation flag included) cross the boundary between
    a GPU shard and an oracle shard."""
    net, cfg = ref_world("maco-p", V=200)
    cpu_single = O.PortWorld(net, cfg, net.grid_distance())
    g = Engine(net, cfg, net.grid_distance())
    g.set_shard(*sharding.shard_bounds(200, 2, 0))
    c = O.PortWorld(net, cfg, net.grid_distance())
    c.set_shard(*sharding.shard_bounds(200, 2, 1))
    step = sharding.local_transport([g, c])
    for _ in range(20):
        step()
        cpu_single.step(1)
    assert same(g, cpu_single) is None
    assert same(c, cpu_single) is None


def test_maco_p_nccl_exchange_world1_equals_unsharded():
    from paper_2010_14244_b200 import engine
    import ctypes as C
    net = networks.grid(32, 32, signals="all")
    cfg = abi.default_config(algorithm="maco-p", vehicle_count=1000, seed=3, max_steps=200)
    uid = C.create_string_buffer(128)
    assert engine.load().gmaco_nccl_unique_id(uid) == 0
    e = Engine(net, cfg, net.grid_distance())
    e.attach_comm(0, 1, uid.raw)
    single = Engine(net, cfg, net.grid_distance())
    e.step(40)
    single.step(40)
    assert same(e, single) is None
    assert O.results_identical(e.run(), single.run())


def _c4_like(V=500, seed=11):
    from test_gpu_parity import _rgg_targets
    net, dist, tgt = _rgg_targets(3000, 12, seed)
    cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive",
                                                   vehicle_count=V, seed=seed, max_steps=40), ants=16)
    cfg.colony.max_hops = 512
    return net, cfg, dist, tgt


@pytest.mark.parametrize("nshards", [2, 3])
def test_by_target_shards_equal_unsharded(nshards):
    """C4's path sharded by destination target (each shard refreshes and
    walks only its own targets' tables, destination-major order kept):
    every shard equals the unsharded engine step by step, the shards
    partition the fleet, and the refreshed tables partition the targets."""
    net, cfg, dist, tgt = _c4_like()
    single = Engine(net, cfg, dist)
    shards = []
    for r in range(nshards):
        e = Engine(net, cfg, dist)
        e.shard_by_target(r, nshards)
        shards.append(e)
    owned = np.sort(np.concatenate([e.owned for e in shards]))
    assert np.array_equal(owned, np.arange(cfg.vehicle_count))
    dest = single.vehicles()["dest"]
    tsets = [set(dest[e.owned].tolist()) for e in shards]
    for a in range(nshards):
        for b in range(a + 1, nshards):
            assert not (tsets[a] & tsets[b]), "a target is planned on two shards"
    step = sharding.local_transport_owned(shards)
    for k in range(8):
        step()
        single.step(1)
        for e in shards:
            assert same(e, single) is None, (k, same(e, single))
    assert sum(e.counters().ant_steps for e in shards) == single.counters().ant_steps
    for e in shards:  # planned tours live on the vehicle's own shard
        for vid in e.owned[::5]:
            assert np.array_equal(e.route(int(vid), True), single.route(int(vid), True))


def test_by_target_nccl_world1_equals_unsharded():
    """The by-target NCCL exchange (records packed in planning order,
    allgather, unpacked to vehicles) at world size 1."""
    from paper_2010_14244_b200 import engine
    import ctypes as C
    net, cfg, dist, tgt = _c4_like(V=400, seed=3)
    uid = C.create_string_buffer(128)
    assert engine.load().gmaco_nccl_unique_id(uid) == 0
    e = Engine(net, cfg, dist)
    e.attach_comm(0, 1, uid.raw)
    single = Engine(net, cfg, dist)
    e.step(10)
    single.step(10)
    assert same(e, single) is None
    assert O.results_identical(e.run(), single.run())
