"""Tiny fleet (latency-only) run for ncu: 10 vehicles, 64 ants on C2."""
import sys

sys.path.insert(0, ".")
from paper_2010_14244_b200 import abi, networks  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

V = int(sys.argv[1]) if len(sys.argv) > 1 else 10
net = networks.grid(32, 32, signals="all")
cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive", vehicle_count=V,
                                               seed=1, max_steps=100), 64)
e = Engine(net, cfg, net.grid_distance())
e.step(8)
print("ok", e.counters().ant_steps)
