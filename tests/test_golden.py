"""Parity against committed golden vectors produced by the reference itself
(tests/golden/make_golden.py over oracle/_ref).  The CPU tests pin the oracle
port; the GPU tests pin the CUDA engine to the same vectors, so both stay
anchored to the reference even where /root/reference is absent."""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))
ALGS = ["dijkstra", "aco", "maco", "maco-p"]


def city():
    c = G["city52"]
    return networks.Network(52, np.array(c["signalized"], np.uint8), np.array(c["edge_from"], np.int32),
                            np.array(c["edge_to"], np.int32), np.array(c["edge_length_mm"], np.int64),
                            np.array(c["edge_lanes"], np.int32))


def same(res, gold):
    r, tt, retired = res
    return (r.mean_travel_s.hex() == gold["mean_travel_s"] and r.mean_wait_s.hex() == gold["mean_wait_s"]
            and r.mean_queue_len.hex() == gold["mean_queue_len"]
            and r.max_edge_occupancy == gold["max_edge_occupancy"]
            and r.completed_count == gold["completed_count"] and r.retired_count == gold["retired_count"]
            and r.steps_executed == gold["steps_executed"]
            and [float(x).hex() for x in tt] == gold["travel_times_s"]
            and [list(x) for x in retired] == gold["retired"])


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def engines(net, cfg, dist=None, gpu=False):
    if gpu:
        from paper_2010_14244_b200.engine import Engine
        return Engine(net, cfg, dist)
    return O.PortWorld(net, cfg, dist)


@pytest.fixture(params=[pytest.param(False, id="port"), pytest.param(True, id="gpu", marks=pytest.mark.gpu)])
def gpu(request):
    return request.param


def test_c1_runs(gpu):
    net = networks.grid(10, 10)
    for case in G["c1_runs"]:
        cfg = abi.default_config(algorithm=case["alg"], vehicle_count=100, seed=case["seed"])
        assert same(engines(net, cfg, net.grid_distance(), gpu).run(), case["result"]), case["alg"]


def test_city_runs(gpu):
    net = city()
    for case in G["city_runs"]:
        cfg = abi.default_config(algorithm=case["alg"], vehicle_count=300, seed=case["seed"])
        assert same(engines(net, cfg, None, gpu).run(), case["result"]), case["alg"]


def test_c2_macop_stepwise(gpu):
    net = networks.grid(32, 32, signals="all")
    cfg = abi.default_config(algorithm="maco-p", vehicle_count=1000, seed=3, max_steps=60)
    w = engines(net, cfg, net.grid_distance(), gpu)
    for gold in G["c2_macop_steps"]:
        w.step(1)
        v, s = w.vehicles(), w.signals()
        assert w.current_step() == gold["step"]
        got = {"tau": digest(w.pheromone()), "occ": digest(w.occupancy()), "state": digest(v["state"]),
               "on_edge": digest(v["on_edge"]), "progress": digest(v["progress_mm"]),
               "queue_vid": digest(s["queue_vid"]), "queue_len": digest(s["queue_len"]),
               "green": digest(s["green"])}
        for k, val in got.items():
            assert val == gold[k], (gold["step"], k)
    assert same(w.run(), G["c2_macop_result"])


def test_next_node_city(gpu):
    q = G["next_node_city"]
    net = city()
    cfg = abi.default_config(algorithm="maco", vehicle_count=200, seed=4, max_steps=30)
    w = engines(net, cfg, None, gpu)
    w.step(10)
    assert w.pheromone().tolist() == q["tau"]
    assert w.occupancy().tolist() == q["occupancy"]
    cur, dst = np.array(q["current"]), np.array(q["dest"])
    ent, stp = np.array(q["entity"], np.uint64), np.array(q["step"], np.uint64)
    for alg, name in ((abi.DIJKSTRA, "dijkstra"), (abi.ACO, "aco"), (abi.MACO, "maco")):
        for n_t in (0, 5000):
            nx, via, dev = w.next_node(alg, cur, dst, ent, stp, n_t)
            g = q[f"{name}_{n_t}"]
            assert nx.tolist() == g["next"] and via.tolist() == g["via"] and dev.tolist() == g["deviated"]


def test_scalar_kats():
    L = O.port_lib()
    p = abi.default_config().pheromone
    p.tau_max, p.tau_min = G["fold_kats"]["params"]["tau_max"], G["fold_kats"]["params"]["tau_min"]
    for t, pos, D, want in G["fold_kats"]["cases"]:
        a = np.array(pos, np.int32)
        assert L.og_fold_maco_edge(t, abi.ptr(a, C.c_int32), len(a), D, C.byref(p)) == want
    p = abi.default_config().pheromone
    for length, want in G["deposit_kats"]:
        assert L.og_deposit_amount(length, C.byref(p)) == want
    s = abi.default_config().signal
    for kind, q, hw, cur, want in G["select_phase_kats"]:
        hwv = [float.fromhex(x) for x in hw]
        assert L.og_select_phase(kind, (C.c_int32 * 8)(*q), (C.c_double * 8)(*hwv), cur, C.byref(s)) == want
