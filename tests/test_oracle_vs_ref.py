"""The oracle port against the compiled, unmodified reference (oracle/_ref).

This is what pins the oracle: RunResult::identical_to (engine.cpp:34-40) on
the BASELINE configs and a matrix of variants, full world snapshots per
step, and the per-function entry points (next_node_*, fold_maco_edge,
spawn_vehicles, init_random, select_phase_*, discharge).  CPU only; skipped
when the reference library is not built (no /root/reference).
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference library not built")

ALGS = ["dijkstra", "aco", "maco", "maco-p"]


def cfg_of(alg, V, seed, **kw):
    c = abi.default_config(algorithm=alg, vehicle_count=V, seed=seed)
    for k, v in kw.items():
        if k == "siblings":
            c.pheromone.decrement_siblings_only = v
        elif k == "edge_occupancy":
            c.routing.deviation_mode = abi.DEV_EDGE_OCCUPANCY
            c.routing.deviation_threshold = v
        elif k == "progress_filter":
            c.routing.progress_filter = v
        elif k == "alpha_beta":
            c.routing.aco_alpha, c.routing.aco_beta = v
        elif k == "tau_min":
            c.pheromone.tau_min = v
            c.pheromone.tau_init_lo = max(v, c.pheromone.tau_init_lo)
        else:
            setattr(c, k, v)
    return c


@pytest.mark.parametrize("alg", ALGS)
def test_c1_identical_and_parallel_run(alg):
    """Config 1 (10x10, 100 vehicles): port == run() == parallel_run(w)."""
    net = networks.grid(10, 10)
    for seed in (1, 2, 3, 4, 5):
        cfg = cfg_of(alg, 100, seed)
        ref = O.ref_run(net, cfg)
        assert O.results_identical(O.PortWorld(net, cfg).run(), ref)
        assert O.results_identical(O.PortWorld(net, cfg, net.grid_distance()).run(), ref)
        if seed == 1:
            for workers in (2, 4, 8):
                assert O.results_identical(O.ref_run(net, cfg, workers), ref)


VARIANTS = [
    {}, dict(siblings=1), dict(edge_occupancy=1), dict(decision_latency_s=1.5),
    dict(spawn=abi.UNIFORM_WINDOW, spawn_window_steps=30), dict(controller=abi.ADAPTIVE),
    dict(progress_filter=0, max_steps=300), dict(alpha_beta=(0.0, 0.0)), dict(alpha_beta=(1.0, 1.0)),
    dict(dt_s=0.7, max_steps=800), dict(tau_min=1.0), dict(max_steps=0), dict(max_steps=9),
    dict(alpha_beta=(0.5, 1.0)), dict(alpha_beta=(2.0, 1.5)),
]


@pytest.mark.parametrize("variant", range(len(VARIANTS)))
def test_variant_matrix(variant):
    nets = [networks.grid(6, 9, 137.5, 2, "all"), O.ref_city(52, 64)]
    for net in nets:
        for alg in ALGS:
            cfg = cfg_of(alg, 150, 7, **VARIANTS[variant])
            assert O.results_identical(O.PortWorld(net, cfg).run(), O.ref_run(net, cfg)), (alg, net.node_count)


def test_blocks_od():
    net = networks.grid(8, 8)
    for alg in ALGS:
        cfg = cfg_of(alg, 200, 11)
        keep = abi.Blocks(cfg, np.arange(0, 6), np.arange(58, 64), bias=0.7)
        assert O.results_identical(O.PortWorld(net, cfg).run(), O.ref_run(net, cfg))
        del keep


@pytest.mark.parametrize("alg", ALGS)
def test_c2_stepwise_world_state(alg):
    """Config 2 (32x32 all-signalized, 1k vehicles): full world per step."""
    net = networks.grid(32, 32, signals="all")
    cfg = cfg_of(alg, 1000, 3, max_steps=120)
    port = O.PortWorld(net, cfg, net.grid_distance())
    ref = O.RefWorld(net, cfg)
    for k in (1, 2, 5, 20, 40):
        assert port.step(k) == ref.step(k)
        pv, rv = port.vehicles(), ref.vehicles()
        for f in abi.VEHICLE_FIELDS:
            assert np.array_equal(pv[f], rv[f]), f
        ps, rs = port.signals(), ref.signals()
        for f in ps:
            assert np.array_equal(ps[f], rs[f]), f
        assert np.array_equal(port.pheromone(), ref.pheromone())
        assert np.array_equal(port.occupancy(), ref.occupancy())
    assert O.results_identical(port.run(), ref.run())
    for vid in range(0, 1000, 97):
        assert np.array_equal(port.route(vid), ref.route(vid))


def test_next_node_against_reference():
    net = O.ref_city(52, 64)
    cfg = cfg_of("maco", 200, 4, max_steps=30)
    port, ref = O.PortWorld(net, cfg), O.RefWorld(net, cfg)
    port.step(15)
    ref.step(15)
    rng = np.random.default_rng(1)
    cur = rng.integers(0, 52, 4000)
    dst = rng.integers(0, 52, 4000)
    keep = cur != dst
    cur, dst = cur[keep], dst[keep]
    ent = rng.integers(0, 1 << 60, len(cur), dtype=np.uint64)
    stp = rng.integers(0, 1 << 20, len(cur), dtype=np.uint64)
    for alg in (abi.DIJKSTRA, abi.ACO, abi.MACO):
        for n_t in (0, 10 ** 6):
            a = port.next_node(alg, cur, dst, ent, stp, n_t)
            b = ref.next_node(alg, cur, dst, ent, stp, n_t)
            for x, y in zip(a, b):
                assert np.array_equal(x, y)


def test_fold_matches_reference_fold_and_literal():
    R, P = O.ref_lib(), O.port_lib()
    rng = np.random.default_rng(3)
    p = abi.default_config().pheromone
    p.tau_max, p.tau_min, p.tau_init_lo = 20.0, 0.5, 0.5
    for _ in range(2000):
        D = int(rng.integers(0, 50))
        pos = np.sort(rng.choice(max(D, 1), size=int(rng.integers(0, max(D, 1) + 1)), replace=False)).astype(np.int32)
        pos = pos[pos < D]
        t = int(rng.integers(0, 25_000_000))
        a = R.ref_fold_maco_edge(t, abi.ptr(pos, C.c_int32), len(pos), D, C.byref(p))
        b = P.og_fold_maco_edge(t, abi.ptr(pos, C.c_int32), len(pos), D, C.byref(p))
        assert a == b
    # literal apply_maco_update of the reference on a small field
    tau = np.array([3_000_000, 19_900_000, 600_000, 0], dtype=np.int64)
    lit = tau.copy()
    choices = [1, 1, 0, 3, 1]
    for ch in choices:
        assert R.ref_apply_maco_update(abi.ptr(lit, C.c_int64), 4, ch, C.byref(p)) == 0
    for e in range(4):
        pos = np.array([i for i, ch in enumerate(choices) if ch == e], dtype=np.int32)
        assert P.og_fold_maco_edge(int(tau[e]), abi.ptr(pos, C.c_int32), len(pos), len(choices), C.byref(p)) == lit[e]


def test_scalar_ops_match_reference():
    R, P = O.ref_lib(), O.port_lib()
    rng = np.random.default_rng(5)
    for rho in (0.0, 0.1, 0.37, 0.999):
        p = abi.default_config().pheromone
        p.rho = rho
        for t in rng.integers(0, 10 ** 9, 2000):
            assert R.ref_evaporate_one(int(t), C.byref(p)) == P.og_evaporate_one(int(t), C.byref(p))
    p = abi.default_config().pheromone
    for length in list(rng.integers(1, 10 ** 9, 2000)) + [1, 999, 10 ** 6]:
        assert R.ref_deposit_amount(int(length), C.byref(p)) == P.og_deposit_amount(int(length), C.byref(p))
    for seed in range(50):
        for a in range(20):
            assert R.ref_draw(seed, a, a * 7, a * 13) == P.og_draw(seed, a, a * 7, a * 13)


def test_signal_ops_match_reference():
    R, P = O.ref_lib(), O.port_lib()
    s = abi.default_config().signal
    rng = np.random.default_rng(9)
    for i in range(20000):
        q = (C.c_int32 * 8)(*rng.integers(0, 26, 8).tolist())
        hw = (C.c_double * 8)(*rng.uniform(0, 240, 8).tolist())
        cur = int(rng.integers(0, 8))
        kind = int(rng.integers(0, 3))
        assert R.ref_select_phase(kind, q, hw, cur, C.byref(s)) == P.og_select_phase(kind, q, hw, cur, C.byref(s))
    for sat in (0.3, 0.5, 0.7, 1.3):
        s.saturation_flow = sat
        r1, r2 = C.c_double(0.0), C.c_double(0.0)
        for k in range(300):
            q = int(rng.integers(0, 6))
            lanes = int(rng.integers(1, 4))
            assert R.ref_discharge(q, C.byref(r1), 1.0, lanes, C.byref(s)) == \
                P.og_discharge(q, C.byref(r2), 1.0, lanes, C.byref(s))
            assert r1.value == r2.value


def test_spawn_and_init_match_reference():
    R = O.ref_lib()
    for net in (networks.grid(12, 7), O.ref_city(52, 64)):
        for spawn in (abi.ALL_AT_START, abi.UNIFORM_WINDOW):
            cfg = cfg_of("aco", 500, 13, spawn=spawn, spawn_window_steps=40)
            V = 500
            o, d = np.zeros(V, np.int32), np.zeros(V, np.int32)
            sp, adv, dep = np.zeros(V), np.zeros(V, np.int64), np.zeros(V, np.int64)
            assert R.ref_spawn(C.byref(net.desc()), C.byref(cfg), abi.ptr(o, C.c_int32), abi.ptr(d, C.c_int32),
                               abi.ptr(sp, C.c_double), abi.ptr(adv, C.c_int64), abi.ptr(dep, C.c_int64)) == 0
            v = O.PortWorld(net, cfg).vehicles()
            assert np.array_equal(v["origin"], o) and np.array_equal(v["dest"], d)
            assert np.array_equal(v["speed_mps"], sp) and np.array_equal(v["advance_mm"], adv)
            assert np.array_equal(v["depart_step"], dep)
            tau = np.zeros(net.edge_count, np.int64)
            assert R.ref_init_random(C.byref(net.desc()), C.byref(cfg.pheromone), 13, abi.ptr(tau, C.c_int64)) == 0
            assert np.array_equal(O.PortWorld(net, cfg).pheromone(), tau)


def test_generators_match_reference():
    for r, c in [(2, 2), (3, 3), (10, 10), (4, 7), (32, 32)]:
        a, b = networks.grid(r, c), O.ref_grid(r, c)
        for f in ("signalized", "edge_from", "edge_to", "edge_length_mm", "edge_lanes"):
            assert np.array_equal(getattr(a, f), getattr(b, f))


def test_validation_errors_match_reference():
    R = O.ref_lib()
    net = networks.grid(3, 3)
    bad = [
        dict(vehicle_count=0), dict(dt_s=0.0), dict(max_steps=-1), dict(decision_latency_s=-1.0),
        dict(speed_min_mps=0.0), dict(speed_min_mps=90.0),
    ]
    for kw in bad:
        cfg = abi.default_config(**kw)
        with pytest.raises(O.OracleError) as e1:
            O.PortWorld(net, cfg)
        with pytest.raises(O.OracleError) as e2:
            O.RefWorld(net, cfg)
        assert str(e1.value) == str(e2.value)
    for field, val in [("rho", 1.0), ("delta_inc", 0.0), ("tau_min", -1.0), ("tau_init_hi", 200.0)]:
        cfg = abi.default_config()
        setattr(cfg.pheromone, field, val)
        with pytest.raises(O.OracleError) as e1:
            O.PortWorld(net, cfg)
        with pytest.raises(O.OracleError) as e2:
            O.RefWorld(net, cfg)
        assert str(e1.value) == str(e2.value)
    cfg = abi.default_config()
    cfg.signal.fixed_cycle_order[3] = 0
    with pytest.raises(O.OracleError) as e1:
        O.PortWorld(net, cfg)
    with pytest.raises(O.OracleError) as e2:
        O.RefWorld(net, cfg)
    assert str(e1.value) == str(e2.value)
    assert R  # keep lib alive
