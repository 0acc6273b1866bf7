"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle.

Bar: bit-exact for every integer / index / state field and every double the
reference produces (RunResult::identical_to, engine.cpp:34-40), on the same
seeded inputs.  The oracle (oracle/_build, pinned against the compiled
reference by tests/test_oracle_vs_ref.py) is the checker; where the compiled
reference itself is present (oracle/_ref) it is compared too.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks
from paper_2010_14244_b200.engine import Engine

pytestmark = pytest.mark.gpu

ALGS = ["dijkstra", "aco", "maco", "maco-p"]


def _cfg(alg, V, seed, **kw):
    cfg = abi.default_config(algorithm=alg, vehicle_count=V, seed=seed)
    for k, v in kw.items():
        if k == "siblings":
            cfg.pheromone.decrement_siblings_only = v
        elif k == "edge_occupancy":
            cfg.routing.deviation_mode = abi.DEV_EDGE_OCCUPANCY
            cfg.routing.deviation_threshold = v
        elif k == "progress_filter":
            cfg.routing.progress_filter = v
        elif k == "alpha_beta":
            cfg.routing.aco_alpha, cfg.routing.aco_beta = v
        elif k == "tau_min":
            cfg.pheromone.tau_min = v
            cfg.pheromone.tau_init_lo = max(v, cfg.pheromone.tau_init_lo)
        elif k == "threshold":
            cfg.routing.deviation_threshold = v
        else:
            setattr(cfg, k, v)
    return cfg


def _same_snapshot(a, b, where=""):
    va, vb = a.vehicles(), b.vehicles()
    for f in abi.VEHICLE_FIELDS:
        assert np.array_equal(va[f], vb[f]), f"{where} vehicle field {f}"
    sa, sb = a.signals(), b.signals()
    for f in sa:
        assert np.array_equal(sa[f], sb[f]), f"{where} signal field {f}"
    assert np.array_equal(a.pheromone(), b.pheromone()), f"{where} pheromone"
    assert np.array_equal(a.occupancy(), b.occupancy()), f"{where} occupancy"


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c1_run_identical(alg, seed):
    """BASELINE config 1: 10x10 grid, 100 vehicles."""
    net = networks.grid(10, 10)
    cfg = _cfg(alg, 100, seed)
    ref = O.PortWorld(net, cfg).run()
    for dist in (abi.DistanceDesc(kind=abi.DIST_DENSE), net.grid_distance()):
        got = Engine(net, cfg, dist).run()
        assert O.results_identical(got, ref), (alg, seed, dist.kind)
    if O.ref_available():
        assert O.results_identical(O.ref_run(net, cfg), ref)


VARIANTS = [
    dict(siblings=1),
    dict(edge_occupancy=1),
    dict(decision_latency_s=1.5),
    dict(spawn=abi.UNIFORM_WINDOW, spawn_window_steps=30),
    dict(controller=abi.ADAPTIVE),
    dict(progress_filter=0, max_steps=300),
    dict(alpha_beta=(0.0, 0.0)),
    dict(dt_s=0.7, max_steps=800),
    dict(tau_min=1.0),
    dict(threshold=50),
    dict(max_steps=0),
    dict(max_steps=7),
]


@pytest.mark.parametrize("variant", range(len(VARIANTS)))
@pytest.mark.parametrize("alg", ALGS)
def test_variants_identical(alg, variant):
    net = networks.grid(6, 9, 137.5, 2, "all")
    cfg = _cfg(alg, 150, 7, **VARIANTS[variant])
    ref = O.PortWorld(net, cfg).run()
    got = Engine(net, cfg).run()
    assert O.results_identical(got, ref)


@pytest.mark.parametrize("alg", ALGS)
def test_city_graph_identical(alg):
    """Irregular graph: the reference's own generate_city(52, 64) network."""
    if not O.ref_available():
        pytest.skip("reference library not built")
    net = O.ref_city(52, 64)
    for seed in (1, 5):
        cfg = _cfg(alg, 200, seed)
        ref = O.ref_run(net, cfg)
        got = Engine(net, cfg).run()
        assert O.results_identical(got, ref), seed


def test_blocks_od_identical():
    net = networks.grid(8, 8)
    for alg in ALGS:
        cfg = _cfg(alg, 200, 11)
        keep = abi.Blocks(cfg, np.arange(0, 6), np.arange(58, 64))
        ref = O.PortWorld(net, cfg).run()
        got = Engine(net, cfg, net.grid_distance()).run()
        assert O.results_identical(got, ref), alg
        del keep


@pytest.mark.parametrize("alg", ALGS)
def test_c2_stepwise_state(alg):
    """BASELINE config 2 (32x32, signals at every intersection, 1k vehicles):
    full world state after every few steps."""
    net = networks.grid(32, 32, signals="all")
    cfg = _cfg(alg, 1000, 3, max_steps=200)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    for k in (1, 1, 3, 10, 25, 60):
        assert gpu.step(k) == cpu.step(k)
        _same_snapshot(gpu, cpu, f"{alg} step {cpu.current_step()}")
    assert O.results_identical(gpu.run(), cpu.run())


def test_next_node_batch():
    """Per-vehicle route query next_node_* (routing.hpp:52-73) on random pairs."""
    net = networks.grid(16, 16)
    cfg = _cfg("maco", 300, 4, max_steps=40)
    gpu = Engine(net, cfg)
    cpu = O.PortWorld(net, cfg)
    gpu.step(20)
    cpu.step(20)
    rng = np.random.default_rng(0)
    n = 5000
    cur = rng.integers(0, net.node_count, n)
    dst = rng.integers(0, net.node_count, n)
    keep = cur != dst
    cur, dst = cur[keep], dst[keep]
    ent = rng.integers(0, 1 << 62, len(cur), dtype=np.uint64)
    stp = rng.integers(0, 1 << 20, len(cur), dtype=np.uint64)
    for alg in (abi.DIJKSTRA, abi.ACO, abi.MACO):
        for n_t in (0, 5000):
            a = gpu.next_node(alg, cur, dst, ent, stp, n_t)
            b = cpu.next_node(alg, cur, dst, ent, stp, n_t)
            for x, y in zip(a, b):
                assert np.array_equal(x, y), (alg, n_t)


def test_colony_anchor_equals_reference_aco():
    """K=1, 1-hop walk, reference RNG key ⇒ identical to Algorithm::Aco."""
    net = networks.grid(10, 10)
    for seed in (1, 2, 3):
        aco = _cfg("aco", 100, seed)
        col = abi.colony_anchor(_cfg("colony", 100, seed))
        ref = O.PortWorld(net, aco).run()
        got = Engine(net, col, net.grid_distance()).run()
        assert O.results_identical(got, ref), seed
        if O.ref_available():
            assert O.results_identical(O.ref_run(net, aco), ref)


@pytest.mark.parametrize("ants", [1, 20, 64, 100])
def test_colony_production_stepwise(ants):
    """GMACO-P colonies (Philox, congestion, best-tour deposit): planned
    tours, pheromone and counters bit-exact against the oracle port."""
    net = networks.grid(12, 12, signals="all")
    cfg = abi.colony_production(_cfg("colony", 300, 9, max_steps=60), ants=ants)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    for k in (1, 2, 5, 12):
        assert gpu.step(k) == cpu.step(k)
        _same_snapshot(gpu, cpu, f"colony step {cpu.current_step()}")
        for vid in range(cfg.vehicle_count):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid
    a, b = gpu.counters(), cpu.counters()
    for f in ("ant_steps", "vehicle_routes", "decisions", "candidates", "degree_sum"):
        assert getattr(a, f) == getattr(b, f), f
    assert O.results_identical(gpu.run(), cpu.run())


def test_colony_dense_queues_stepwise():
    """Congested lattice colony (800 vehicles on a 5x5 all-signalized grid):
    many arrivals join one queue in one step, so the tail's per-queue E3
    (one thread per signal queue) appends long arrival chains in ascending
    vid (commit_enqueue, engine.cpp:297-301).  Every step's full state is
    compared with the oracle, and the run must have produced such chains."""
    net = networks.grid(5, 5, signals="all")
    cfg = abi.colony_production(_cfg("colony", 800, 21, max_steps=80, controller=abi.PREEMPTIVE), ants=32)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    prev = gpu.signals()["queue_len"].astype(np.int64)
    most = 0
    for _ in range(40):
        assert gpu.step(1) == cpu.step(1)
        _same_snapshot(gpu, cpu, f"dense colony step {cpu.current_step()}")
        cur = gpu.signals()["queue_len"].astype(np.int64)
        most = max(most, int((cur - prev).max()))
        prev = cur
    assert most >= 3, f"no queue took 3 or more arrivals in one step (max {most})"
    assert O.results_identical(gpu.run(), cpu.run())


def test_colony_no_filter_tabu():
    """Progress filter off: tabu tenure + hop cap (cycles possible)."""
    net = networks.grid(8, 8)
    cfg = abi.colony_production(_cfg("colony", 120, 5, max_steps=40, progress_filter=0), ants=16)
    cfg.colony.max_hops = 40
    gpu = Engine(net, cfg)
    cpu = O.PortWorld(net, cfg)
    for k in (1, 4, 10):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, "colony-nofilter")
        for vid in range(cfg.vehicle_count):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid


def test_colony_reference_rng_multi_ant():
    net = networks.grid(9, 9)
    cfg = abi.colony_production(_cfg("colony", 150, 3, max_steps=50), ants=8)
    cfg.colony.rng = abi.RNG_REFERENCE
    cfg.colony.deposit = abi.DEPOSIT_COMPLETION
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    assert O.results_identical(gpu.run(), cpu.run())
    assert np.array_equal(gpu.pheromone(), cpu.pheromone())


def test_realized_paths():
    net = networks.grid(10, 10)
    cfg = _cfg("aco", 100, 4)
    gpu = Engine(net, cfg)
    cpu = O.PortWorld(net, cfg)
    gpu.run()
    cpu.run()
    for vid in range(100):
        assert np.array_equal(gpu.route(vid), cpu.route(vid)), vid


def test_colony_bench_workload_c2():
    """The bench workload itself (C2: 32x32 all-signalized, 1000 vehicles,
    64 ants, preemptive): a few iterations bit-exact against the oracle."""
    import bench
    net = networks.grid(32, 32, signals="all")
    cfg = bench.workload_config(1, 400)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    for k in (1, 2, 3):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, "bench workload")
    for vid in range(0, 1000, 37):
        assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid
    a, b = gpu.counters(), cpu.counters()
    assert (a.ant_steps, a.candidates, a.degree_sum) == (b.ant_steps, b.candidates, b.degree_sum)


@pytest.mark.parametrize("dist_kind", ["dense", "grid"])
def test_colony_ell4_table_and_grid(dist_kind):
    """Fast ELL-4 walk with dense-table distances (DK=0) and closed form (DK=1)."""
    net = networks.grid(10, 11, signals="all")
    cfg = abi.colony_production(_cfg("colony", 200, 13, max_steps=80, controller=abi.PREEMPTIVE), ants=32)
    dist = net.grid_distance() if dist_kind == "grid" else abi.DistanceDesc(kind=abi.DIST_DENSE)
    gpu = Engine(net, cfg, dist)
    cpu = O.PortWorld(net, cfg, dist)
    for k in (1, 3, 9):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, dist_kind)
    assert O.results_identical(gpu.run(), cpu.run())


def test_colony_city_generic_path():
    """Irregular graph (ELL-8 rows, generic walk kernel, dense distances)."""
    if not O.ref_available():
        pytest.skip("reference library not built")
    net = O.ref_city(52, 64)
    cfg = abi.colony_production(_cfg("colony", 200, 3, max_steps=120), ants=24)
    gpu = Engine(net, cfg)
    cpu = O.PortWorld(net, cfg)
    for k in (1, 5, 20):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, "city colony")
        for vid in range(200):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid
    assert O.results_identical(gpu.run(), cpu.run())


def test_colony_replay_mode_large_ants():
    """ants=512 on a 24x24 grid exceeds nothing but exercises the generic
    kernel (ants > 256) with scratch tours."""
    net = networks.grid(24, 24)
    cfg = abi.colony_production(_cfg("colony", 40, 21, max_steps=30), ants=512)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    gpu.step(4)
    cpu.step(4)
    _same_snapshot(gpu, cpu, "ants=512")
    for vid in range(40):
        assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid


def _rgg_targets(nodes, targets, seed):
    net = networks.random_geometric(nodes, k=3, seed=seed)
    rng = np.random.default_rng(seed)
    tgt = np.sort(rng.choice(nodes, size=targets, replace=False)).astype(np.int32)
    dist = abi.DistanceDesc(kind=abi.DIST_TARGETS, targets=abi.ptr(tgt, __import__("ctypes").c_int32),
                            target_count=targets)
    return net, dist, tgt


@pytest.mark.parametrize("mode", ["queue", "block", "replay"])
def test_colony_rgg_targets_csr_walker(mode):
    """C4's path at small scale: random-geometric graph (CSR rows, degree up
    to ~9 -> the MAXD=16 general walker), TARGETS distance tables, long
    multi-hop tours.  queue = persistent ant-queue walker (the default in
    scratch mode), block = one-CTA-per-vehicles walker with scratch tours,
    replay = winner replay; all bit-exact."""
    net, dist, tgt = _rgg_targets(3000, 12, 77)
    cfg = abi.colony_production(_cfg("colony", 400, 5, max_steps=40), ants=16)
    cfg.options.flags = {"queue": 0, "block": abi.OPT_NO_QUEUE, "replay": abi.OPT_NO_SCRATCH}[mode]
    cfg.colony.max_hops = 512
    gpu = Engine(net, cfg, dist)
    cpu = O.PortWorld(net, cfg, dist)
    for k in (1, 3, 8):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, f"rgg {mode}")
        for vid in range(0, 400, 7):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid
    a, b = gpu.counters(), cpu.counters()
    for f in ("ant_steps", "vehicle_routes", "decisions", "candidates", "degree_sum"):
        assert getattr(a, f) == getattr(b, f), f
    assert O.results_identical(gpu.run(), cpu.run())


@pytest.mark.parametrize("variant", ["bitmap_queue", "odd_ants", "cost_over_int32", "length_over_int32"])
def test_colony_rgg_targets_walker_variants(variant):
    """Paths around the per-target-row walker (k_colony_qt), all bit-exact:
    bitmap_queue = the shared-row queue walker (OPT_NO_TT); odd_ants = 12
    ants (lanes fetch single ants, no 16-lane groups); cost_over_int32 =
    edge costs len*(1+load) beyond 2^31 (the int32 record cost's -1 escape to
    the int64 table); length_over_int32 = edge lengths beyond 2^31 mm (no
    {slot, length} epilogue map)."""
    net, dist, tgt = _rgg_targets(2500, 10, 19)
    ants = 16
    flags = 0
    if variant == "bitmap_queue":
        flags = abi.OPT_NO_TT
    elif variant == "odd_ants":
        ants = 12
    elif variant == "cost_over_int32":
        net.edge_length_mm = net.edge_length_mm * 20000  # ~1e9 mm: cost >= 2^31 once load >= 2
    elif variant == "length_over_int32":
        net.edge_length_mm = net.edge_length_mm * 60000  # some lengths >= 2^31 mm
        assert net.edge_length_mm.max() >= 2 ** 31
    cfg = abi.colony_production(_cfg("colony", 600, 9, max_steps=30), ants=ants)
    cfg.options.flags = flags
    cfg.colony.max_hops = 400
    gpu = Engine(net, cfg, dist)
    cpu = O.PortWorld(net, cfg, dist)
    for k in (1, 2, 6):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, f"rgg {variant}")
        for vid in range(0, 600, 11):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid
    a, b = gpu.counters(), cpu.counters()
    for f in ("ant_steps", "vehicle_routes", "decisions", "candidates", "degree_sum"):
        assert getattr(a, f) == getattr(b, f), f
    assert O.results_identical(gpu.run(), cpu.run())


def test_colony_rgg_max_hops_cap():
    """Hop cap shorter than many tours: capped ants fail (cost = inf), and
    vehicles whose every ant failed keep their previous plan state."""
    net, dist, tgt = _rgg_targets(2000, 6, 3)
    cfg = abi.colony_production(_cfg("colony", 200, 8, max_steps=25), ants=32)
    cfg.colony.max_hops = 20
    gpu = Engine(net, cfg, dist)
    cpu = O.PortWorld(net, cfg, dist)
    for k in (1, 4, 12):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, "rgg max_hops")
    assert O.results_identical(gpu.run(), cpu.run())


def test_async_step_then_read_equals_oracle():
    """gmaco_step with executed == NULL only enqueues; the batched
    gmaco_get_vehicles read (which also refreshes the control block) is
    ordered after it.  Stepping past finished() stays a no-op."""
    net = networks.grid(10, 10, signals="all")
    cfg = abi.colony_production(_cfg("colony", 150, 4, max_steps=30), ants=32)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    for _ in range(12):
        assert gpu.step(1, count=False) is None
        cpu.step(1)
        _same_snapshot(gpu, cpu, "async step")
    assert gpu.current_step() == cpu.current_step()
    for _ in range(40):  # runs past max_steps: extra enqueued steps are no-ops
        gpu.step(1, count=False)
    cpu.step(40)
    assert gpu.finished() and cpu.finished()
    assert gpu.current_step() == cpu.current_step()
    assert O.results_identical(gpu.collect(), cpu.collect())


@pytest.mark.parametrize("shape,ants", [((40, 40), 64), ((40, 40), 20), ((70, 72), 64)])
def test_colony_lattice_multiword_move_bits(shape, ants):
    """Lattice walks longer than 64 hops keep one move bit per hop in several
    64-hop SMEM words (2 words at 40x40, 3 at 70x72); the winner's tour is
    rebuilt from prefix popcounts across words (warp epilogue for K % 32 == 0,
    serial otherwise).  Planned tours, pheromone and state bit-exact."""
    R, Cc = shape
    net = networks.grid(R, Cc, signals="interior")
    cfg = abi.colony_production(_cfg("colony", 250, 17, max_steps=40), ants=ants)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    for k in (1, 2, 6):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, f"multiword {shape} K={ants}")
        for vid in range(0, 250, 5):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid
    a, b = gpu.counters(), cpu.counters()
    for f in ("ant_steps", "vehicle_routes", "decisions", "candidates", "degree_sum"):
        assert getattr(a, f) == getattr(b, f), f


def _hub_graph(hub_degree, seed=5):
    """12x12 grid plus hubs whose out-degree is raised to `hub_degree` by
    bidirectional shortcut edges (shorter than the grid path, so the progress
    filter keeps them as candidates)."""
    base = networks.grid(12, 12, signals="interior")
    rng = np.random.default_rng(seed)
    n = base.node_count
    src, dst = list(base.edge_from), list(base.edge_to)
    ln, la = list(base.edge_length_mm), list(base.edge_lanes)
    have = set(zip(src, dst))
    deg = np.bincount(np.asarray(src), minlength=n)
    for hub in (13, 40, 77, 101, 130):
        others = [v for v in rng.permutation(n) if v != hub]
        for v in others:
            if deg[hub] >= hub_degree:
                break
            if (hub, v) in have or (v, hub) in have:
                continue
            for a, b in ((hub, v), (v, hub)):
                src.append(a); dst.append(b)
                ln.append(int(rng.integers(150_000, 900_000))); la.append(2)
                have.add((a, b)); deg[a] += 1
    return networks.Network(node_count=n, signalized=base.signalized.copy(),
                            edge_from=np.asarray(src, np.int32), edge_to=np.asarray(dst, np.int32),
                            edge_length_mm=np.asarray(ln, np.int64), edge_lanes=np.asarray(la, np.int32))


@pytest.mark.parametrize("hub_degree,mode", [(14, "queue"), (14, "block"), (14, "replay"), (20, "generic")])
def test_colony_wide_rows(hub_degree, mode):
    """Rows wider than the queue walker's 8-slot register window (span 16 on
    the 4-aligned CSR layout) and, at degree 20, beyond the CSR walkers'
    16-slot bound (generic kernel); dense distance tables."""
    net = _hub_graph(hub_degree)
    maxdeg = np.bincount(net.edge_from).max()
    assert (8 < maxdeg <= 16) if hub_degree <= 16 else maxdeg > 16
    cfg = abi.colony_production(_cfg("colony", 300, 23, max_steps=40), ants=32)
    cfg.options.flags = {"replay": abi.OPT_NO_SCRATCH, "block": abi.OPT_NO_QUEUE}.get(mode, 0)
    gpu = Engine(net, cfg)
    cpu = O.PortWorld(net, cfg)
    for k in (1, 3, 8):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, f"hubs {hub_degree} {mode}")
        for vid in range(0, 300, 3):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid
    a, b = gpu.counters(), cpu.counters()
    for f in ("ant_steps", "vehicle_routes", "decisions", "candidates", "degree_sum"):
        assert getattr(a, f) == getattr(b, f), f
    assert O.results_identical(gpu.run(), cpu.run())


@pytest.mark.parametrize("fused", [False, True])
def test_double_buffered_readback_every_step(fused):
    """gmaco_vehicles_enqueue / _wait (or gmaco_step_snapshot / _wait): each
    step's snapshot (taken while the next step is already enqueued) equals the
    oracle's state at that step."""
    import ctypes as C
    net = networks.grid(10, 10, signals="all")
    cfg = abi.colony_production(_cfg("colony", 150, 4, max_steps=30), ants=32)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    V = cfg.vehicle_count
    bufs = [dict(state=np.zeros(V, np.uint8), on_edge=np.zeros(V, np.int32), progress_mm=np.zeros(V, np.int64),
                 decisions=np.zeros(V, np.int32)) for _ in range(2)]
    views = [abi.VehicleView(state=abi.ptr(b["state"], C.c_uint8), on_edge=abi.ptr(b["on_edge"], C.c_int32),
                             progress_mm=abi.ptr(b["progress_mm"], C.c_int64),
                             decisions=abi.ptr(b["decisions"], C.c_int32)) for b in bufs]
    for k in range(14):
        if fused:  # gmaco_step_snapshot: step + gather in one graph launch
            gpu.step_snapshot(views[k % 2], k % 2)
        else:
            gpu.step(1, count=False)
            gpu.vehicles_enqueue(views[k % 2], k % 2)
        if k:
            gpu.vehicles_wait((k - 1) % 2, views[(k - 1) % 2])
            cpu.step(1)
            ref = cpu.vehicles()
            for f, arr in bufs[(k - 1) % 2].items():
                assert np.array_equal(arr, ref[f]), (k, f)
    gpu.vehicles_wait(13 % 2, views[13 % 2])
    cpu.step(1)
    ref = cpu.vehicles()
    for f, arr in bufs[13 % 2].items():
        assert np.array_equal(arr, ref[f]), f


COLONY_OPTIONS = [
    dict(congestion=0, deposit=abi.DEPOSIT_BEST_TOUR, congestion_evaporation=0, replan_all=0),
    dict(congestion=1, deposit=abi.DEPOSIT_COMPLETION, congestion_evaporation=1, replan_all=1),
    dict(congestion=1, deposit=abi.DEPOSIT_BEST_TOUR, congestion_evaporation=0, replan_all=1, hop_limit=5),
    dict(congestion=0, deposit=abi.DEPOSIT_BEST_TOUR, congestion_evaporation=1, replan_all=0, hop_limit=3),
    dict(congestion=1, deposit=abi.DEPOSIT_NONE, congestion_evaporation=1, replan_all=1),
]


@pytest.mark.parametrize("opts", range(len(COLONY_OPTIONS)))
@pytest.mark.parametrize("graph", ["lattice", "rgg"])
def test_colony_option_matrix(graph, opts):
    """Colony switches (congestion, deposit kind, congestion evaporation,
    replan_all, hop_limit) on the lattice walker and the ant-queue walker."""
    if graph == "lattice":
        net = networks.grid(14, 14, signals="all")
        dist_factory = net.grid_distance
        keep = None
    else:
        net, dist, keep = _rgg_targets(2500, 10, 41)
        dist_factory = lambda: dist
    cfg = abi.colony_production(_cfg("colony", 250, 31, max_steps=45), ants=32)
    for kk, vv in COLONY_OPTIONS[opts].items():
        setattr(cfg.colony, kk, vv)
    cfg.colony.max_hops = 512
    gpu = Engine(net, cfg, dist_factory())
    cpu = O.PortWorld(net, cfg, dist_factory())
    for k in (1, 4, 9):
        gpu.step(k)
        cpu.step(k)
        _same_snapshot(gpu, cpu, f"{graph} opts {opts}")
        for vid in range(0, 250, 4):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), vid
    assert O.results_identical(gpu.run(), cpu.run())
    del keep
