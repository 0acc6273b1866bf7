"""Walk-kernel scaling probe: p50 device time of stage B (colony walk) and of
the whole step versus fleet size and colony size on the C2 lattice."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2010_14244_b200 import abi, networks  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

net = networks.grid(32, 32, signals="all")
out = []
for V, K in [(1000, 64), (100, 64), (10, 64), (1000, 32), (1000, 128), (250, 256), (4000, 64), (16000, 64)]:
    cfg = abi.default_config(algorithm="colony", controller="preemptive", vehicle_count=V, seed=1, max_steps=100)
    abi.colony_production(cfg, K)
    e = Engine(net, cfg, net.grid_distance())
    e.step(5)
    c0 = e.counters().ant_steps
    walk, step = e.bench_steps(20, 512 << 20)
    steps = e.counters().ant_steps - c0
    walk2, step2 = e.bench_steps(20, 0)
    out.append(dict(V=V, K=K, walk_us=float(np.median(walk)) * 1e3, step_us=float(np.median(step)) * 1e3,
                    walk_noflush_us=float(np.median(walk2)) * 1e3, step_noflush_us=float(np.median(step2)) * 1e3,
                    ant_steps_per_iter=steps / 20))
    print(json.dumps(out[-1]), flush=True)
