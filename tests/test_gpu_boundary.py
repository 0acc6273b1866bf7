"""C-ABI contract edges (include/gmaco.h): snapshot field sets, mid-run
pheromone uploads on congestion colonies, engine teardown with work in
flight.  Engine results are compared with the oracle bit for bit."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks
from paper_2010_14244_b200.engine import Engine, EngineError

pytestmark = pytest.mark.gpu


def _colony(V=200, seed=4, steps=40, ants=32):
    cfg = abi.default_config(algorithm="colony", controller="preemptive", vehicle_count=V, seed=seed,
                             max_steps=steps)
    return abi.colony_production(cfg, ants=ants)


def test_vehicles_wait_rejects_a_different_field_set():
    """A snapshot of progress_mm (8 B/vehicle) must not be waited into a view
    asking for state (1 B/vehicle): same field COUNT, different fields."""
    net = networks.grid(10, 10, signals="all")
    cfg = _colony(V=150)
    gpu = Engine(net, cfg, net.grid_distance())
    V = cfg.vehicle_count
    prog = np.zeros(V, np.int64)
    st = np.zeros(V + 64, np.uint8)  # guard tail: must stay untouched
    gpu.step(2)
    gpu.vehicles_enqueue(abi.VehicleView(progress_mm=abi.ptr(prog, C.c_int64)), 0)
    with pytest.raises(EngineError) as ei:
        gpu.vehicles_wait(0, abi.VehicleView(state=abi.ptr(st, C.c_uint8)))
    assert ei.value.code == 1
    assert not st.any()
    gpu.vehicles_wait(0, abi.VehicleView(progress_mm=abi.ptr(prog, C.c_int64)))
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    cpu.step(2)
    assert np.array_equal(prog, cpu.vehicles()["progress_mm"])


@pytest.mark.parametrize("congestion", [1, 0])
def test_set_pheromone_mid_run_matches_oracle(congestion):
    """gmaco_set_pheromone on a congestion colony (the bench workload's
    shape): the next walk's weights carry the edge load exactly as stage F+G
    would have computed them (oracle refresh_edge_terms)."""
    net = networks.grid(12, 12, signals="all")
    cfg = _colony(V=300, seed=9)
    cfg.colony.congestion = congestion
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    gpu.step(4)
    cpu.step(4)
    rng = np.random.default_rng(5)
    lo, hi = int(cfg.pheromone.tau_min * 1e6), int(cfg.pheromone.tau_max * 1e6)
    tau = rng.integers(lo, hi // 10, net.edge_count).astype(np.int64)
    gpu.set_pheromone(tau)
    cpu.set_pheromone(tau)
    for k in (1, 3):
        gpu.step(k)
        cpu.step(k)
        assert np.array_equal(gpu.pheromone(), cpu.pheromone())
        va, vb = gpu.vehicles(), cpu.vehicles()
        for f in abi.VEHICLE_FIELDS:
            assert np.array_equal(va[f], vb[f]), f
        for vid in range(0, cfg.vehicle_count, 3):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid


def test_set_pheromone_rejects_values_outside_the_clamp_range():
    net = networks.grid(6, 6)
    cfg = abi.default_config(algorithm="aco", vehicle_count=30, seed=1)
    gpu = Engine(net, cfg)
    tau = np.full(net.edge_count, int(cfg.pheromone.tau_max * 1e6) + 1, np.int64)
    with pytest.raises(EngineError) as ei:
        gpu.set_pheromone(tau)
    assert ei.value.code == 1 and "outside [tau_min, tau_max]" in str(ei.value)


def test_destroy_with_snapshot_in_flight_then_reuse_pool():
    """Destroying an engine whose snapshot gather was never waited for must
    settle its stream before the pinned slots go back to the pool; a new
    engine that takes them reads correct snapshots."""
    net = networks.grid(10, 10, signals="all")
    cfg = _colony(V=150)
    V = cfg.vehicle_count
    for _ in range(3):
        e = Engine(net, cfg, net.grid_distance())
        bufs = [np.zeros(V, np.int64) for _ in range(2)]
        for k in range(6):
            e.step_snapshot(abi.VehicleView(progress_mm=abi.ptr(bufs[k & 1], C.c_int64)), k & 1)
        e.close()  # two snapshots never waited for
    e = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    out = np.zeros(V, np.int64)
    view = abi.VehicleView(progress_mm=abi.ptr(out, C.c_int64))
    for k in range(5):
        e.step_snapshot(view, 0)
        e.vehicles_wait(0, view)
        cpu.step(1)
        assert np.array_equal(out, cpu.vehicles()["progress_mm"]), k


@pytest.mark.parametrize("alg", ["colony", "maco-p"])
def test_step_snapshot_past_finished_keeps_the_final_state(alg):
    """gmaco_step_snapshot on a small world gathers in the step's finalizing
    tail block; a step past finished() is a no-op, and its snapshot must
    still hold the (final) state -- on both readback slots."""
    net = networks.grid(8, 8, signals="all")
    if alg == "colony":
        cfg = _colony(V=60, seed=3, steps=12, ants=16)
    else:
        cfg = abi.default_config(algorithm="maco-p", vehicle_count=60, seed=3, max_steps=12)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    V = cfg.vehicle_count
    bufs = [np.zeros(V, np.int64) for _ in range(2)]
    views = [abi.VehicleView(progress_mm=abi.ptr(b, C.c_int64)) for b in bufs]
    for k in range(20):  # 12 real steps, then 8 no-ops
        gpu.step_snapshot(views[k & 1], k & 1)
        gpu.vehicles_wait(k & 1, views[k & 1])
        cpu.step(1)
        assert np.array_equal(bufs[k & 1], cpu.vehicles()["progress_mm"]), k
    assert gpu.finished() and cpu.finished()
