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
        raw = e.debug_trace(1)
        t = raw.astype(np.int64)
        rel = (t - t[0]) / 1e3
        print(f"{os.environ.get('TAG', '')} V={V} walk: staged {rel[1]:.2f} end {rel[2]:.2f} | "
              f"tail start {rel[3]:.2f} signals {rel[5]:.2f} FG {rel[6]:.2f} (us) | max epilogue cycles: "
              f"rebuild+deposit {raw[7]} take_edge {raw[8]} move {raw[9]} | walk(loop..epilogue start) {raw[10]} | block0 reduce {raw[11]}")
