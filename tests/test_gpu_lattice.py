"""The lattice walker's roulette as an integer compare (LatRec,
paper_2010_14244_b200/csrc/device.cuh): for candidate weights (wa, wb) the
device tabulates thr with "first candidate iff k < thr", k the draw's top 53
bits.  It must equal the reference's sequential roulette
(R/src/routing.cpp:100-113) for every k:

* total = wa + wb positive and finite: first iff fl(fl(k * 2^-53) * total) < wa;
* otherwise the uniform pick: first iff (int)(u * 2) == 0, i.e. k < 2^52.

Checked here on the exact boundary (thr - 1 picks first, thr does not) for
random weights over the whole double range and for the edge cases a weight
table can hold (zero, subnormal, equal, overflowing, non-finite).  Whole-run
parity of the lattice walker against the oracle is in test_gpu_parity.py and
test_gpu_shapes.py."""
import numpy as np
import pytest

from paper_2010_14244_b200 import abi, networks
from paper_2010_14244_b200.engine import Engine

pytestmark = pytest.mark.gpu

K_END = 1 << 53


def first(k, wa, wb):
    """routing.cpp:100-113 for two candidates with u = k * 2^-53."""
    total = np.float64(wa) + np.float64(wb)
    u = np.float64(k) * np.float64(2.0 ** -53)
    if not (total > 0.0 and np.isfinite(total)):
        return int(u * 2.0) == 0
    return bool(u * total < np.float64(wa))


@pytest.fixture(scope="module")
def engine():
    net = networks.grid(4, 4)
    return Engine(net, abi.default_config(algorithm="aco", vehicle_count=4, seed=1), net.grid_distance())


def check(engine, wa, wb):
    thr = engine.roulette_threshold(wa, wb)
    rng = np.random.default_rng(7)
    with np.errstate(over="ignore", invalid="ignore"):
        for a, b, t in zip(wa, wb, thr.tolist()):
            assert 0 <= t <= K_END, (a, b, t)
            if t > 0:
                assert first(t - 1, a, b), (a, b, t)
            if t < K_END:
                assert not first(t, a, b), (a, b, t)
            for k in rng.integers(0, K_END, 4, dtype=np.uint64).tolist():
                assert (k < t) == first(k, a, b), (a, b, t, k)
    return thr


def test_threshold_random_weights(engine):
    rng = np.random.default_rng(11)
    n = 20000
    # the weights the lattice tables hold: tau^alpha * eta^beta / (1 + load)
    wa = rng.uniform(0.0, 5.0, n) / (1.0 + rng.integers(0, 50, n))
    wb = rng.uniform(0.0, 5.0, n) / (1.0 + rng.integers(0, 50, n))
    check(engine, wa, wb)
    # the whole exponent range, both orders of magnitude apart
    ea = rng.uniform(-1000, 1000, n)
    eb = ea + rng.uniform(-60, 60, n)
    wa = np.ldexp(rng.uniform(0.5, 1.0, n), ea.astype(np.int64))
    wb = np.ldexp(rng.uniform(0.5, 1.0, n), np.clip(eb, -1070, 1020).astype(np.int64))
    check(engine, wa, wb)


def test_threshold_edge_cases(engine):
    tiny, huge, inf, nan = 5e-324, 1.7976931348623157e308, np.inf, np.nan
    pairs = [
        (1.0, 1.0), (1.0, 0.0), (0.0, 1.0), (0.0, 0.0), (tiny, tiny), (tiny, 0.0), (0.0, tiny),
        (tiny, 1.0), (1.0, tiny), (huge, huge), (huge, 1.0), (1.0, huge), (inf, 1.0), (1.0, inf),
        (nan, 1.0), (1.0, nan), (inf, inf), (-1.0, 3.0), (3.0, -1.0), (-1.0, -1.0),
        (1.0, 2.0 ** -53), (1.0, 2.0 ** -54), (2.0 ** -53, 1.0), (1.0 / 3.0, 2.0 / 3.0), (0.1, 0.2),
    ]
    wa = np.array([p[0] for p in pairs])
    wb = np.array([p[1] for p in pairs])
    thr = check(engine, wa, wb)
    got = dict(zip(pairs[:4], thr[:4].tolist()))
    assert got[(1.0, 0.0)] == K_END  # a lone positive weight is always taken
    assert got[(0.0, 1.0)] == 0
    assert got[(0.0, 0.0)] == 1 << 52  # uniform pick
    assert thr[pairs.index((inf, 1.0))] == 1 << 52 and thr[pairs.index((1.0, nan))] == 1 << 52


@pytest.mark.parametrize("shape", [(9, 23), (23, 9), (14, 14)])
@pytest.mark.parametrize("flags,ants", [("no_smem", 32), ("no_smem", 64), ("no_smem_no_bits", 32)])
def test_lattice_walker_record_layouts(shape, flags, ants):
    """The lattice walker reading its records from global memory in the
    diagonal-major quadrant tables (what C3/C5 run), on non-square lattices in
    both orientations, with multi-vehicle CTAs (K=32), one-vehicle CTAs (K=64)
    and scratch tours instead of move bits: every iteration equals the oracle
    (vehicles, signals, pheromone, occupancy, counters, planned tours)."""
    from oracle import oracle as O

    rows, cols = shape
    net = networks.grid(rows, cols, signals="all")
    V = rows * cols
    cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive", vehicle_count=V,
                                                   seed=rows * 7 + ants, max_steps=40), ants=ants)
    cfg.options.flags = abi.OPT_NO_SMEM | (abi.OPT_NO_BITS if flags == "no_smem_no_bits" else 0)
    gpu = Engine(net, cfg, net.grid_distance())
    cpu = O.PortWorld(net, cfg, net.grid_distance())
    for it in range(4):
        gpu.step(1)
        cpu.step(1)
        va, vb = gpu.vehicles(), cpu.vehicles()
        for f in abi.VEHICLE_FIELDS:
            assert np.array_equal(va[f], vb[f]), (it, f)
        sa, sb = gpu.signals(), cpu.signals()
        for f in sa:
            assert np.array_equal(sa[f], sb[f]), (it, f)
        assert np.array_equal(gpu.pheromone(), cpu.pheromone()), it
        assert np.array_equal(gpu.occupancy(), cpu.occupancy()), it
        a, b = gpu.counters(), cpu.counters()
        assert (a.ant_steps, a.candidates, a.degree_sum) == (b.ant_steps, b.candidates, b.degree_sum), it
        for vid in range(0, V, 5):
            assert np.array_equal(gpu.route(vid, True), cpu.route(vid, True)), (it, vid)
