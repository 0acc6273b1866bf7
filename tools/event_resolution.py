"""Distinct CUDA-event step times of the bench graph (clock quantization check)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2010_14244_b200 import networks  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

net = networks.grid(32, 32, signals="all")
e = Engine(net, bench.workload_config(1, 100000), net.grid_distance())
e.step(5)
_, s = e.bench_steps(200, 512 << 20, "step")
u, c = np.unique(np.round(s * 1e3, 4), return_counts=True)
print("distinct step times (us) and counts:", list(zip(u.tolist(), c.tolist()))[:40])
print("mean %.3f  p50 %.3f  min %.3f" % (s.mean() * 1e3, np.median(s) * 1e3, s.min() * 1e3))
