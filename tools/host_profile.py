import ctypes as C, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2010_14244_b200 import abi, workloads
from paper_2010_14244_b200.engine import Engine
net, cfg, dist, keep = workloads.c2(seed=1, max_steps=100)
for rep in range(2):
    e = Engine(net, cfg, dist)
    V = cfg.vehicle_count
    st = [np.zeros(V, np.uint8) for _ in range(2)]
    oe = [np.zeros(V, np.int32) for _ in range(2)]
    views = [abi.VehicleView(state=abi.ptr(st[i], C.c_uint8), on_edge=abi.ptr(oe[i], C.c_int32)) for i in range(2)]
    e.step(5)
    ts, tw = [], []
    for k in range(40):
        t0 = time.perf_counter()
        e.step_snapshot(views[k & 1], k & 1)
        t1 = time.perf_counter()
        if k:
            e.vehicles_wait((k - 1) & 1, views[(k - 1) & 1])
        t2 = time.perf_counter()
        ts.append((t1 - t0) * 1e6); tw.append((t2 - t1) * 1e6)
    e.vehicles_wait(1, views[1])
    print("rep", rep, "snapshot call us", np.round(ts[:12], 1).tolist(), "median", np.median(ts[:20]), np.median(ts[25:]))
    print("rep", rep, "wait us", np.round(tw[:12], 1).tolist(), "median", np.median(tw[1:20]), np.median(tw[25:]))
    e.close()
