"""Multi-rank protocol on CPU: world_size-2 gloo runs of the sharded world
(oracle shards exchanging decision records and deposits through
torch.distributed) must equal the unsharded world bit for bit -- for GMACO-P
colonies and for the reference's own algorithms, whose network-wide MACO
fold is replicated on every rank from the exchanged decisions in global vid
order (commit_pheromone, parallel.cpp:195-258)."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks, sharding

STEPS = 12


ALGS = ["colony", "maco-p", "maco", "maco-scoped", "aco", "dijkstra"]


def make_world(alg="colony"):
    net = networks.grid(12, 12, signals="all")
    if alg == "colony":
        cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive",
                                                       vehicle_count=301, seed=5, max_steps=80), ants=16)
    else:
        cfg = abi.default_config(algorithm=alg.replace("-scoped", ""), vehicle_count=301, seed=5, max_steps=80)
        cfg.routing.deviation_threshold = 150  # MACO deviations happen (n_t > threshold early on)
        cfg.pheromone.decrement_siblings_only = int(alg == "maco-scoped")
    return net, cfg


def digest(w):
    h = hashlib.sha256()
    v = w.vehicles()
    for f in abi.VEHICLE_FIELDS:
        h.update(np.ascontiguousarray(v[f]).tobytes())
    s = w.signals()
    for f in sorted(s):
        h.update(np.ascontiguousarray(s[f]).tobytes())
    h.update(w.pheromone().tobytes())
    h.update(w.occupancy().tobytes())
    return h.hexdigest()


def _worker(rank, world, port, q, alg):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    net, cfg = make_world(alg)
    w = O.PortWorld(net, cfg, net.grid_distance())
    w.world_size = world
    w.set_shard(*sharding.shard_bounds(cfg.vehicle_count, world, rank))

    def allgather(a):
        t = torch.from_numpy(a)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return torch.cat(out).numpy()

    def allreduce_sum(a):
        t = torch.from_numpy(a.copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy()

    for _ in range(STEPS):
        sharding.sharded_step(w, allgather, allreduce_sum)
    c = w.counters()
    q.put((rank, digest(w), w.current_step(), c.ant_steps, c.vehicle_routes))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("alg", ["colony", "maco-p"])
def test_gloo_two_rank_sharded_world_equals_single_world(alg):
    net, cfg = make_world(alg)
    single = O.PortWorld(net, cfg, net.grid_distance())
    single.step(STEPS)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, alg)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    ref = digest(single)
    for rank, d, step, _, _ in out:
        assert step == STEPS
        assert d == ref, f"rank {rank} state differs from the unsharded world"
    c = single.counters()
    assert sum(o[3] for o in out) == c.ant_steps
    assert sum(o[4] for o in out) == c.vehicle_routes


@pytest.mark.parametrize("alg", ALGS)
def test_in_process_three_shards_equal_single_world(alg):
    net, cfg = make_world(alg)
    single = O.PortWorld(net, cfg, net.grid_distance())
    shards = []
    for r in range(3):
        w = O.PortWorld(net, cfg, net.grid_distance())
        w.set_shard(*sharding.shard_bounds(cfg.vehicle_count, 3, r))
        shards.append(w)
    step = sharding.local_transport(shards)
    for _ in range(STEPS):
        step()
        single.step(1)
        ref = digest(single)
        assert all(digest(w) == ref for w in shards)
    assert sum(w.counters().ant_steps for w in shards) == single.counters().ant_steps
    if alg.startswith("maco"):
        assert single.vehicles()["deviations"].sum() > 0  # deviated records crossed the exchange
