"""Generates tests/golden/reference_golden.json from the UNMODIFIED reference
compiled in place (oracle/_ref/libmacosim_ref.so).  Run in the build
container (needs /root/reference):  python tests/golden/make_golden.py

Doubles are stored as float.hex() strings so comparisons stay bit-exact.
"""
import ctypes as C
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2010_14244_b200 import abi, networks  # noqa: E402

ALGS = ["dijkstra", "aco", "maco", "maco-p"]


def result_json(res):
    r, tt, retired = res
    return {
        "mean_travel_s": r.mean_travel_s.hex(), "mean_wait_s": r.mean_wait_s.hex(),
        "mean_queue_len": r.mean_queue_len.hex(), "max_edge_occupancy": r.max_edge_occupancy,
        "completed_count": r.completed_count, "retired_count": r.retired_count,
        "steps_executed": r.steps_executed, "travel_times_s": [float(x).hex() for x in tt],
        "retired": retired,
    }


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    O.build()
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj (compiled by oracle/Makefile)"}
    # the reference's own 52-node city network (generate_city(52, 64, 3, kCitySeed))
    city = O.ref_city(52, 64)
    out["city52"] = {k: getattr(city, k).tolist() for k in
                     ("signalized", "edge_from", "edge_to", "edge_length_mm", "edge_lanes")}
    # config 1 runs
    net = networks.grid(10, 10)
    out["c1_runs"] = []
    for alg in ALGS:
        for seed in (1, 2, 3):
            cfg = abi.default_config(algorithm=alg, vehicle_count=100, seed=seed)
            out["c1_runs"].append({"alg": alg, "seed": seed, "result": result_json(O.ref_run(net, cfg))})
    # city runs
    out["city_runs"] = []
    for alg in ALGS:
        cfg = abi.default_config(algorithm=alg, vehicle_count=300, seed=5)
        out["city_runs"].append({"alg": alg, "seed": 5, "result": result_json(O.ref_run(city, cfg))})
    # config 2 (32x32 all signalized, 1k vehicles, maco-p): per-step state digests
    net2 = networks.grid(32, 32, signals="all")
    cfg = abi.default_config(algorithm="maco-p", vehicle_count=1000, seed=3, max_steps=60)
    w = O.RefWorld(net2, cfg)
    steps = []
    for k in range(12):
        w.step(1)
        v = w.vehicles()
        s = w.signals()
        steps.append({"step": w.current_step(), "tau": digest(w.pheromone()), "occ": digest(w.occupancy()),
                      "state": digest(v["state"]), "on_edge": digest(v["on_edge"]),
                      "progress": digest(v["progress_mm"]), "queue_vid": digest(s["queue_vid"]),
                      "queue_len": digest(s["queue_len"]), "green": digest(s["green"])})
    out["c2_macop_steps"] = steps
    out["c2_macop_result"] = result_json(w.run())
    # next_node_* queries on the city network after 10 MACO steps
    cfg = abi.default_config(algorithm="maco", vehicle_count=200, seed=4, max_steps=30)
    w = O.RefWorld(city, cfg)
    w.step(10)
    rng = np.random.default_rng(7)
    cur = rng.integers(0, 52, 600)
    dst = rng.integers(0, 52, 600)
    keep = cur != dst
    cur, dst = cur[keep], dst[keep]
    ent = rng.integers(0, 1 << 60, len(cur), dtype=np.uint64)
    stp = rng.integers(0, 1 << 20, len(cur), dtype=np.uint64)
    q = {"current": cur.tolist(), "dest": dst.tolist(), "entity": ent.tolist(), "step": stp.tolist(),
         "tau": w.pheromone().tolist(), "occupancy": w.occupancy().tolist()}
    for alg, name in ((abi.DIJKSTRA, "dijkstra"), (abi.ACO, "aco"), (abi.MACO, "maco")):
        for n_t in (0, 5000):
            nx, via, dev = w.next_node(alg, cur, dst, ent, stp, n_t)
            q[f"{name}_{n_t}"] = {"next": nx.tolist(), "via": via.tolist(), "deviated": dev.tolist()}
    out["next_node_city"] = q
    # fold / evaporate / deposit / select KATs
    R = O.ref_lib()
    p = abi.default_config().pheromone
    p.tau_max, p.tau_min, p.tau_init_lo = 20.0, 0.5, 0.5
    folds = []
    for _ in range(300):
        D = int(rng.integers(0, 40))
        pos = np.sort(rng.choice(max(D, 1), size=int(rng.integers(0, max(D, 1) + 1)), replace=False)).astype(np.int32)
        pos = pos[pos < D]
        t = int(rng.integers(0, 25_000_000))
        folds.append([t, pos.tolist(), D, R.ref_fold_maco_edge(t, abi.ptr(pos, C.c_int32), len(pos), D, C.byref(p))])
    out["fold_kats"] = {"params": {"tau_max": 20.0, "tau_min": 0.5}, "cases": folds}
    p = abi.default_config().pheromone
    out["deposit_kats"] = [[int(L_), R.ref_deposit_amount(int(L_), C.byref(p))]
                           for L_ in list(rng.integers(1, 10 ** 9, 200)) + [1, 999, 10 ** 6]]
    s = abi.default_config().signal
    sel = []
    for _ in range(500):
        qq = rng.integers(0, 26, 8).tolist()
        hw = rng.uniform(0, 240, 8).tolist()
        cur_ = int(rng.integers(0, 8))
        kind = int(rng.integers(0, 3))
        sel.append([kind, qq, [x.hex() for x in hw], cur_,
                    R.ref_select_phase(kind, (C.c_int32 * 8)(*qq), (C.c_double * 8)(*hw), cur_, C.byref(s))])
    out["select_phase_kats"] = sel
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
