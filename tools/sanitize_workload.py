"""Small engine workloads for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Covers every kernel family a production run
launches: the multi-kernel reference-algorithm step (k_decide, k_signals,
k_move, k_e3, k_edges, the decision scan), the cooperative PDL tail, the
lattice colony walker with TMA staging and signal CTAs, the ant-queue
walker over per-target rows (k_tt_*, k_colony_pro/qt/epi), the device
SSSP, the batched next_node query and the snapshot gather.

  compute-sanitizer --tool memcheck python tools/sanitize_workload.py

Each workload is compared with the oracle so a sanitizer run also shows
the results are unchanged under instrumentation.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2010_14244_b200 import abi, networks  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402


def check(name, gpu, cpu, steps):
    for k in steps:
        gpu.step(k)
        cpu.step(k)
        assert np.array_equal(gpu.pheromone(), cpu.pheromone()), name
        va, vb = gpu.vehicles(), cpu.vehicles()
        for f in abi.VEHICLE_FIELDS:
            assert np.array_equal(va[f], vb[f]), (name, f)
    print(f"{name}: ok at step {cpu.current_step()}", flush=True)


def main():
    only = sys.argv[1:]
    net = networks.grid(10, 10)
    if not only or "ref" in only:
        for alg in ("maco-p", "maco", "aco", "dijkstra"):
            cfg = abi.default_config(algorithm=alg, vehicle_count=100, seed=1, max_steps=60)
            check(f"c1 {alg}", Engine(net, cfg, net.grid_distance()), O.PortWorld(net, cfg, net.grid_distance()),
                  (1, 4, 10))
        cfg = abi.default_config(algorithm="maco-p", vehicle_count=100, seed=2, max_steps=30)
        check("c1 maco-p dense-sssp", Engine(net, cfg, abi.DistanceDesc(kind=abi.DIST_DENSE)),
              O.PortWorld(net, cfg), (1, 5))
    if not only or "grid" in only:
        g = networks.grid(32, 32, signals="all")
        cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive",
                                                       vehicle_count=300, seed=1, max_steps=30), ants=64)
        gpu = Engine(g, cfg, g.grid_distance())
        check("c2-shape colony (lattice walker, coop tail)", gpu, O.PortWorld(g, cfg, g.grid_distance()),
              (1, 2, 3))
        V = cfg.vehicle_count
        st = [np.zeros(V, np.uint8) for _ in range(2)]
        views = [abi.VehicleView(state=abi.ptr(st[i], C.c_uint8)) for i in range(2)]
        for k in range(4):
            gpu.step_snapshot(views[k & 1], k & 1)
            if k:
                gpu.vehicles_wait((k - 1) & 1, views[(k - 1) & 1])
        gpu.vehicles_wait(1, views[1])
        print("snapshot gather: ok", flush=True)
    if not only or "rgg" in only:
        rg = networks.random_geometric(1500, k=3, seed=3)
        tgt = np.array([5, 77, 400, 901, 1200, 1499], dtype=np.int32)
        dist = abi.DistanceDesc(kind=abi.DIST_TARGETS, targets=abi.ptr(tgt, C.c_int32), target_count=len(tgt))
        cfg = abi.colony_production(abi.default_config(algorithm="colony", vehicle_count=200, seed=4,
                                                       max_steps=20), ants=16)
        cfg.colony.max_hops = 256
        check("rgg targets colony (tt refresh, queue walker)", Engine(rg, cfg, dist), O.PortWorld(rg, cfg, dist),
              (1, 2))
    if not only or "query" in only:
        cfg = abi.default_config(algorithm="maco", vehicle_count=100, seed=4, max_steps=40)
        gpu, cpu = Engine(net, cfg), O.PortWorld(net, cfg)
        gpu.step(5)
        cpu.step(5)
        rng = np.random.default_rng(0)
        cur = rng.integers(0, 100, 500)
        dst = (cur + 1 + rng.integers(0, 98, 500)) % 100
        ent = rng.integers(0, 1 << 62, 500, dtype=np.uint64)
        stp = rng.integers(0, 1 << 20, 500, dtype=np.uint64)
        for alg in (abi.DIJKSTRA, abi.ACO, abi.MACO):
            a = gpu.next_node(alg, cur, dst, ent, stp, 0)
            b = cpu.next_node(alg, cur, dst, ent, stp, 0)
            for x, y in zip(a, b):
                assert np.array_equal(x, y), alg
        print("next_node batch: ok", flush=True)
    print("SANITIZE_WORKLOAD_DONE")


if __name__ == "__main__":
    main()
