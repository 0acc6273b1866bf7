"""gmaco_create phase times (GMACO_OPT_PROFILE_CREATE, printed to stderr) and
the e2e leg's phases for one configuration.

  python tools/create_profile.py [c2|c3|...] [steps]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2010_14244_b200 import abi, engine, workloads  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

if os.environ.get("LIB"):  # A/B: another build of the library
    engine.load(os.environ["LIB"])

config = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for rep in range(3):
    net, cfg, dist, keep = workloads.CONFIGS[config](seed=1, max_steps=steps + 10)
    cfg.options.flags = (abi.OPT_PROFILE_CREATE if rep == 2 else 0) | int(os.environ.get("FLAGS", "0"))
    t0 = time.perf_counter()
    e = Engine(net, cfg, dist)
    t1 = time.perf_counter()
    V = cfg.vehicle_count
    st = [np.zeros(V, np.uint8) for _ in range(2)]
    oe = [np.zeros(V, np.int32) for _ in range(2)]
    views = [abi.VehicleView(state=abi.ptr(st[i], C.c_uint8), on_edge=abi.ptr(oe[i], C.c_int32)) for i in range(2)]
    e.step(5)
    t2 = time.perf_counter()
    ts = [t2]
    for k in range(steps):
        e.step_snapshot(views[k & 1], k & 1)
        if k:
            e.vehicles_wait((k - 1) & 1, views[(k - 1) & 1])
        ts.append(time.perf_counter())
    e.vehicles_wait((steps - 1) & 1, views[(steps - 1) & 1])
    t3 = time.perf_counter()
    e.collect()
    t4 = time.perf_counter()
    e.close()
    per = np.diff(ts) * 1e6
    print(f"rep {rep}: create {1e3 * (t1 - t0):.3f} ms, warmup(5) {1e3 * (t2 - t1):.3f} ms, loop {1e6 * (t3 - t2) / steps:.1f} us/step "
          f"(first 3 steps {per[:3].round(1).tolist()} us, median {np.median(per):.1f}), collect {1e3 * (t4 - t3):.3f} ms",
          flush=True)
