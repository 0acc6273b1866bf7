"""Where the e2e time of the C2 bench leg goes: create, step+D2H loop, collect."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2010_14244_b200 import abi, networks  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

net = networks.grid(32, 32, signals="all")
for rep in range(3):
    cfg = bench.workload_config(1, 400)
    t0 = time.perf_counter()
    e = Engine(net, cfg, net.grid_distance())
    t1 = time.perf_counter()
    V = cfg.vehicle_count
    st = np.zeros(V, dtype=np.uint8)
    oe = np.zeros(V, dtype=np.int32)
    view = abi.VehicleView(state=abi.ptr(st, C.c_uint8), on_edge=abi.ptr(oe, C.c_int32))
    e.step(5)
    t2 = time.perf_counter()
    ts, tg = 0.0, 0.0
    for _ in range(200):
        a = time.perf_counter()
        e.step(1, count=False)
        b = time.perf_counter()
        e._check(e.L.gmaco_get_vehicles(e.h, C.byref(view)))
        c = time.perf_counter()
        ts += b - a
        tg += c - b
    t3 = time.perf_counter()
    res = e.collect()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms | warmup 5 steps {1e3*(t2-t1):.2f} ms | per step: step(1) {1e6*ts/200:.1f} us "
          f"get_vehicles {1e6*tg/200:.1f} us | collect {1e3*(t4-t3):.2f} ms")
    e.close()
