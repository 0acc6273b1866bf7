"""The oracle port against the reference's own known-answer tests.

Each test restates a case of /root/reference/proj/tests (test_rng.cpp,
test_pheromone.cpp, test_signals.cpp, test_net.cpp, helpers.hpp,
signal_oracle.hpp) against the plain-C restatement in oracle/.  CPU only.
"""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks

L = None


@pytest.fixture(scope="module", autouse=True)
def lib():
    global L
    L = O.port_lib()
    yield


def draw(seed, a, b=0, c=0):
    return L.og_draw(seed, a, b, c)


def to_unit(bits):
    return L.og_to_unit(bits)


# --------------------------------------------------------------------------
# rng (test_rng.cpp:8-45)
# --------------------------------------------------------------------------
def test_rng_purity():
    assert draw(42, 1, 2, 3) == draw(42, 1, 2, 3)
    assert draw(42, 1, 2, 3) != draw(42, 1, 2, 4)
    assert draw(42, 1, 2, 3) != draw(43, 1, 2, 3)
    assert draw(7, 2, 0) != draw(7, 3, 0)  # SpawnPair vs SpawnSpeed


def test_rng_unit_range_and_mean():
    s = 0.0
    for i in range(100000):
        u = to_unit(draw(123, 1, i))
        assert 0.0 <= u < 1.0
        s += u
    assert abs(s / 100000 - 0.5) < 0.01


def test_rng_below_covers():
    hit = set()
    for i in range(1000):
        v = L.og_below(draw(9, 2, i), 10)
        assert v < 10
        hit.add(v)
    assert hit == set(range(10))


def test_rng_uniform_interval():
    for i in range(1000):
        v = L.og_uniform(draw(5, 3, i), 50.0, 80.0)
        assert 50.0 <= v < 80.0
    assert L.og_uniform(draw(5, 3, 0), 5.0, 5.0) == 5.0


def test_rng_matches_reference_mix64_constants():
    # splitmix64 finalizer of 0 (rng.hpp:21-26): published value of splitmix64's first output
    assert L.og_mix64(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("ctr,key,expect", [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
])
def test_philox4x32_10_random123_kat(ctr, key, expect):
    """Philox4x32-10 known-answer vectors of Random123 (kat_vectors)."""
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    L.og_philox4x32_10(c, k, o)
    assert tuple(o) == expect


# --------------------------------------------------------------------------
# pheromone (test_pheromone.cpp:22-189)
# --------------------------------------------------------------------------
def pp(**kw):
    p = abi.default_config().pheromone
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def tfd(v):
    return L.og_tau_from_double(v)


def maco_update(tau, chosen, p):
    """Literal apply_maco_update (pheromone.cpp:34-46) as a one-decision fold."""
    pos = (C.c_int32 * 1)(0)
    return [L.og_fold_maco_edge(t, pos if e == chosen else None, 1 if e == chosen else 0, 1, C.byref(p))
            for e, t in enumerate(tau)]


def evaporate(tau, p):
    return [L.og_evaporate_one(t, C.byref(p)) for t in tau]


def deposit(tau, path, length_mm, p):
    if not path:
        return list(tau)
    amt = L.og_deposit_amount(length_mm, C.byref(p))
    out = list(tau)
    for e in path:
        out[e] = min(out[e] + amt, tfd(p.tau_max))
    return out


def line_world(edges, p, seed=1):
    nodes = edges + 1
    net = networks.Network(nodes, np.zeros(nodes, np.uint8), np.arange(edges, dtype=np.int32),
                           np.arange(1, edges + 1, dtype=np.int32), np.full(edges, 100000, np.int64),
                           np.ones(edges, np.int32))
    cfg = abi.default_config(vehicle_count=1, seed=seed)
    cfg.pheromone = p
    return O.PortWorld(net, cfg)


def test_degenerate_init_range():
    p = pp(tau_init_lo=5.0, tau_init_hi=5.0)
    w = line_world(5, p)
    assert all(t == tfd(5.0) for t in w.pheromone())


def test_init_deterministic_in_seed():
    net = O.ref_city(52, 64) if O.ref_available() else networks.grid(6, 6)
    a = O.PortWorld(net, abi.default_config(vehicle_count=1, seed=42)).pheromone()
    b = O.PortWorld(net, abi.default_config(vehicle_count=1, seed=42)).pheromone()
    c = O.PortWorld(net, abi.default_config(vehicle_count=1, seed=43)).pheromone()
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_init_law_of_large_numbers():
    net = networks.grid(51, 51, 100, 1, "none")
    cfg = abi.default_config(vehicle_count=1, seed=7)
    cfg.pheromone.tau_init_lo, cfg.pheromone.tau_init_hi = 0.0, 10.0
    tau = O.PortWorld(net, cfg, net.grid_distance()).pheromone() / 1e6
    assert len(tau) >= 10000
    assert abs(tau.mean() - 5.0) < 0.2


def test_maco_update_inc_dec_clamp():
    p = pp()
    assert maco_update([tfd(3.0)], 0, p) == [tfd(4.0)]
    assert maco_update([0, 0, 0], 1, p) == [0, tfd(1.0), 0]


@pytest.mark.parametrize("k", [1, 3, 7, 12, 30])
def test_repeated_maco_closed_form(k):
    p = pp(tau_max=10.0)
    f = [tfd(3.0), tfd(8.0)]
    for _ in range(k):
        f = maco_update(f, 0, p)
    assert f[0] / 1e6 == min(3.0 + k, 10.0)


def test_fold_equals_literal_application():
    """fold_maco_edge (parallel.cpp:77-92) == literal per-decision updates."""
    rng = np.random.default_rng(0)
    p = pp(tau_max=20.0, tau_min=0.5, tau_init_lo=0.5)
    for _ in range(300):
        m = int(rng.integers(1, 6))
        D = int(rng.integers(0, 40))
        chosen = rng.integers(0, m, D)
        tau = [int(x) for x in rng.integers(tfd(0.5), tfd(20.0), m)]
        lit = list(tau)
        for ch in chosen:
            lit = maco_update(lit, int(ch), p)
        for e in range(m):
            pos = np.nonzero(chosen == e)[0].astype(np.int32)
            got = L.og_fold_maco_edge(tau[e], abi.ptr(pos, C.c_int32), len(pos), D, C.byref(p))
            assert got == lit[e]


def test_evaporation_identity_arithmetic_decay():
    p = pp(rho=0.0)
    f = [tfd(8.0), tfd(2.0)]
    assert evaporate(f, p) == f
    p = pp(rho=0.5)
    assert evaporate(f, p) == [tfd(4.0), tfd(1.0)]
    p = pp(rho=0.1)
    steps = math.ceil(math.log(1e-6 / 100.0) / math.log(1.0 - 0.1))
    g = [tfd(100.0), tfd(37.5)]
    prev = g[0]
    for _ in range(steps):
        g = evaporate(g, p)
        assert g[0] <= prev
        prev = g[0]
    assert g == [0, 0]


def test_aco_deposit_basics():
    p = pp()
    f = [tfd(1.0), tfd(2.0)]
    assert deposit(f, [], 1000000, p) == f
    after = deposit(f, [0], 1000000, p)
    assert after == [tfd(100.0), tfd(2.0)]
    assert L.og_deposit_amount(0, C.byref(p)) == -1  # nonpositive length rejected


def test_deposit_then_evaporate_le_evaporate_then_deposit():
    p = pp(rho=0.3)
    for s in range(500):
        tau = [tfd(L.og_uniform(draw(s, 11, e), 0.0, 100.0)) for e in range(4)]
        length = 1000 + L.og_below(draw(s, 12), 5000000)
        a = evaporate(deposit(tau, [0, 1, 2, 3], length, p), p)
        b = deposit(evaporate(tau, p), [0, 1, 2, 3], length, p)
        assert all(x <= y for x, y in zip(a, b))


def test_bounds_under_random_operations():
    p = pp(tau_max=20.0, tau_min=0.5, tau_init_lo=0.5, tau_init_hi=20.0)
    lo, hi = tfd(0.5), tfd(20.0)
    for seq in range(60):
        tau = [min(max(tfd(L.og_uniform(draw(seq, 1, e), 0.5, 20.0)), lo), hi) for e in range(6)]
        for op in range(50):
            pick = L.og_below(draw(seq, 21, op), 3)
            if pick == 0:
                tau = maco_update(tau, L.og_below(draw(seq, 22, op), 6), p)
            elif pick == 1:
                tau = evaporate(tau, p)
            else:
                tau = deposit(tau, [1, 2, 3], 2000000, p)
            assert all(lo <= t <= hi for t in tau)


def test_maco_rank_monotonicity():
    p = pp()
    for s in range(300):
        tau = [tfd(L.og_uniform(draw(s, 31, e), 0.0, 100.0)) for e in range(5)]
        ch = L.og_below(draw(s, 32), 5)
        g = maco_update(tau, ch, p)
        for e in range(5):
            if e != ch:
                assert g[ch] - g[e] >= tau[ch] - tau[e]


# --------------------------------------------------------------------------
# signals (test_signals.cpp:29-196, signal_oracle.hpp)
# --------------------------------------------------------------------------
def sp(**kw):
    s = abi.default_config().signal
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def select(kind, q, hw=None, cursor=0, s=None):
    s = s or sp()
    qa = (C.c_int32 * 8)(*q)
    ha = (C.c_double * 8)(*(hw or [0.0] * 8))
    return L.og_select_phase(kind, qa, ha, cursor, C.byref(s))


def preemptive_oracle(q, hw, cursor, s):
    """signal_oracle.hpp:14-55 restated (collect candidates per rule, then scan)."""
    over = [i for i in range(8) if q[i] > s.th_max]
    if over:
        best = over[0]
        for i in over:
            if q[i] > q[best]:
                best = i
        return best
    over = [i for i in range(8) if hw[i] > s.t_max]
    if over:
        best = over[0]
        for i in over:
            if hw[i] > hw[best]:
                best = i
        return best
    ne = [i for i in range(8) if q[i] > 0]
    if ne:
        best = ne[0]
        for i in ne:
            if q[i] > q[best]:
                best = i
        return best
    order = list(s.fixed_cycle_order)
    return order[(order.index(cursor) + 1) % 8]


def random_state(seed, index, s):
    """signal_oracle.hpp:60-77."""
    q, hw = [], []
    for i in range(8):
        n = L.og_below(draw(seed, 700, index, i), 26)
        q.append(n)
        hw.append(L.og_uniform(draw(seed, 701, index, i), 0.0, 2.0 * s.t_max) if n > 0 else 0.0)
    return q, hw, L.og_below(draw(seed, 702, index), 8)


def test_phase_mapping_round_robin():
    net = networks.grid(3, 3, 100, 3, "interior")
    w = O.PortWorld(net, abi.default_config(vehicle_count=1))
    sig = w.signals()
    assert list(sig["node"]) == [4]
    assert sig["discharge_lanes"][0] == 3
    assert sig["green_elapsed_s"][0] >= 10.0  # epoch at step 0
    assert sig["green"][0] == 7 and sig["cycle_cursor"][0] == 7


def test_preemptive_rules():
    assert select(2, [0] * 8, cursor=2) == 3
    assert select(2, [3, 0, 5, 1, 0, 0, 0, 0]) == 2
    assert select(2, [3, 0, 12, 1, 0, 0, 11, 0]) == 2
    assert select(2, [2] * 8, [5, 400, 5, 5, 5, 5, 5, 5], s=sp(t_max=300.0)) == 1
    assert select(2, [11, 2, 0, 0, 0, 0, 0, 0], [0, 500, 0, 0, 0, 0, 0, 0]) == 0
    assert select(2, [0, 7, 0, 7, 0, 0, 0, 0]) == 1
    assert select(2, [0, 12, 0, 12, 0, 0, 0, 0]) == 1


def test_preemptive_dominance_and_oracle():
    s = sp()
    for i in range(20000):
        q, hw, cur = random_state(17, i, s)
        got = select(2, q, hw, cur, s)
        assert got == preemptive_oracle(q, hw, cur, s)
        if any(x > s.th_max for x in q):
            assert q[got] > s.th_max


@pytest.mark.slow
def test_preemptive_oracle_1e5():
    s = sp()
    for i in range(100000):
        q, hw, cur = random_state(17, i, s)
        assert select(2, q, hw, cur, s) == preemptive_oracle(q, hw, cur, s)


def test_fixed_controller_cycles():
    assert select(0, [0, 9, 0, 0, 0, 0, 0, 0], cursor=7) == 0
    cur = 7
    granted = []
    for _ in range(8):
        g = select(0, [0] * 8, cursor=cur)
        granted.append(g)
        cur = g
    assert sorted(granted) == list(range(8))


def test_adaptive_controller():
    assert select(1, [0, 0, 4, 0, 0, 0, 0, 0], cursor=0) == 2
    assert select(1, [0] * 8, cursor=4) == select(0, [0] * 8, cursor=4)
    assert select(1, [1, 9, 0, 0, 0, 0, 0, 0], cursor=0) == 0


def test_discharge_fifo_fractional():
    s = sp(saturation_flow=1.0)
    rem = C.c_double(0.0)
    assert L.og_discharge(0, C.byref(rem), 1.0, 3, C.byref(s)) == 0
    rem = C.c_double(0.0)
    assert L.og_discharge(5, C.byref(rem), 1.0, 3, C.byref(s)) == 3
    half = sp()
    rem = C.c_double(0.0)
    got = [L.og_discharge(4, C.byref(rem), 1.0, 1, C.byref(half)) for _ in range(4)]
    assert got == [0, 1, 0, 1]


def test_discharge_conservation():
    s = sp(saturation_flow=0.7)
    rem = C.c_double(0.0)
    queued = released = arrived = 0
    for step in range(500):
        a = L.og_below(draw(99, 44, step), 3)
        queued += a
        arrived += a
        r = L.og_discharge(queued, C.byref(rem), 1.0, 2, C.byref(s))
        queued -= r
        released += r
    assert released + queued == arrived


# --------------------------------------------------------------------------
# net (test_net.cpp:31-242, helpers.hpp)
# --------------------------------------------------------------------------
def random_digraph(seed):
    """helpers.hpp:23-45 restated."""
    n = 2 + L.og_below(draw(seed, 900), 11)
    frm, to, ln = [], [], []
    c = 0
    for u in range(n):
        for v in range(n):
            if u == v:
                continue
            c += 1
            if to_unit(draw(seed, 901, c)) >= 0.3:
                continue
            frm.append(u)
            to.append(v)
            ln.append((1 + L.og_below(draw(seed, 902, c), 20)) * 1000)
    m = len(frm)
    return networks.Network(n, np.zeros(n, np.uint8), np.array(frm, np.int32), np.array(to, np.int32),
                            np.array(ln, np.int64), np.ones(m, np.int32))


def floyd_warshall(net):
    n = net.node_count
    INF = np.iinfo(np.int64).max
    d = np.full((n, n), INF, dtype=np.int64)
    np.fill_diagonal(d, 0)
    for a, b, l in zip(net.edge_from, net.edge_to, net.edge_length_mm):
        d[a, b] = min(d[a, b], l)
    for k in range(n):
        for i in range(n):
            if d[i, k] == INF:
                continue
            for j in range(n):
                if d[k, j] == INF:
                    continue
                d[i, j] = min(d[i, j], d[i, k] + d[k, j])
    return d


def test_apsp_equals_floyd_warshall_with_lexicographic_next_hop():
    INF = np.iinfo(np.int64).max
    for seed in range(100):
        net = random_digraph(seed)
        n = net.node_count
        fw = floyd_warshall(net)
        dist = np.zeros(n * n, np.int64)
        nxt = np.zeros(n * n, np.int32)
        assert L.og_apsp(C.byref(net.desc()), abi.ptr(dist, C.c_int64), abi.ptr(nxt, C.c_int32)) == 0
        assert np.array_equal(dist.reshape(n, n), fw)
        # fw_lexi_path (helpers.hpp:66-90): smallest neighbour on a shortest path
        out = {}
        for a, b, l in zip(net.edge_from, net.edge_to, net.edge_length_mm):
            out.setdefault(int(a), []).append((int(b), int(l)))
        for u in range(n):
            for v in range(n):
                if u == v or fw[u, v] == INF:
                    continue
                cand = sorted(x for x, l in out.get(u, []) if fw[x, v] != INF and l + fw[x, v] == fw[u, v])
                assert nxt[u * n + v] == cand[0]
        # triangle inequality
        for k in range(n):
            for i in range(n):
                for j in range(n):
                    if fw[i, k] != INF and fw[k, j] != INF:
                        assert fw[i, j] <= fw[i, k] + fw[k, j]


def test_generate_grid_counts():
    g = networks.grid(2, 2, 100, 1, "interior")
    assert g.edge_count == 8 and g.signalized_count() == 0
    g = networks.grid(3, 3, 100, 1, "interior")
    assert g.edge_count == 24 and g.signalized_count() == 1
    g = networks.grid(32, 32, signals="all")
    assert g.edge_count == 3968 and g.signalized_count() == 1024


@pytest.mark.parametrize("mut,msg", [
    (lambda n: n.edge_to.__setitem__(0, 99), "edge 0 references missing node 99"),
    (lambda n: n.edge_to.__setitem__(1, n.edge_from[1]), "edge 1 is a self-loop at node"),
    (lambda n: n.edge_length_mm.__setitem__(2, 0), "edge 2 has nonpositive length"),
    (lambda n: n.edge_lanes.__setitem__(3, 0), "edge 3 has lanes < 1"),
    (lambda n: (n.edge_to.__setitem__(2, n.edge_to[0]), n.edge_from.__setitem__(2, n.edge_from[0])),
     "duplicate edge between nodes"),
])
def test_graph_validation_messages(mut, msg):
    net = networks.grid(3, 3)
    mut(net)
    err = C.create_string_buffer(256)
    assert L.og_validate_graph(C.byref(net.desc()), err, 256) == 1
    assert msg in err.value.decode()
