"""Per-stage latency of one engine step from the device stage trace."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2010_14244_b200 import abi, networks  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

net = networks.grid(32, 32, signals="all")
import os
for V in (10, 1000):
    cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive", vehicle_count=V,
                                                   seed=1, max_steps=100), 64)
    e = Engine(net, cfg, net.grid_distance())
    e.step(5)
    for rep in range(3):
        t = e.debug_trace(1).astype(np.int64)
        rel = (t - t[0]) / 1e3
        print(f"{os.environ.get('TAG', '')} V={V} walk: staged {rel[1]:.2f} end {rel[2]:.2f} | tail start {rel[3]:.2f} E12 {rel[4]:.2f} "
              f"E3 {rel[5]:.2f} FG {rel[6]:.2f} (us)")
