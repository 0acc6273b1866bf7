"""Step time of the C2 bench sequence vs. the L2 flush size (fresh engine per size)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2010_14244_b200 import networks  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

net = networks.grid(32, 32, signals="all")
for fb in (0, 1 << 20, 128 << 20, 512 << 20, 0):
    e = Engine(net, bench.workload_config(1, 100000), net.grid_distance())
    e.step(5)
    _, s = e.bench_steps(100, fb, "step")
    print(f"flush {fb >> 20:4d} MiB: step p50 {np.median(s) * 1e3:.2f} us")
    e.close()
