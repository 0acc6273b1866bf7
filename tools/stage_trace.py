"""Per-stage latency of one engine step from the device stage trace.

  python tools/stage_trace.py            warm and L2-flushed traces at V=10 and V=1000 (C2 grid)
"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2010_14244_b200 import abi, engine, networks  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

if os.environ.get("LIB"):  # A/B: another build of the library (bind the entry points it has)
    import ctypes
    _probe = ctypes.CDLL(os.environ["LIB"])
    for _name in list(engine.SIGNATURES):
        if not hasattr(_probe, _name):
            del engine.SIGNATURES[_name]
    engine.load(os.environ["LIB"])

net = networks.grid(32, 32, signals="all")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for V in (10, 1000):
    cfg = abi.colony_production(abi.default_config(algorithm="colony", controller="preemptive", vehicle_count=V,
                                                   seed=1, max_steps=100), 64)
    e = Engine(net, cfg, net.grid_distance())
    e.step(5)
    for mode in ("warm", "flushed"):
        for rep in range(3):
            if mode == "flushed":
                flush.fill_(rep + 1)
                torch.cuda.synchronize()
            raw = e.debug_trace(1)
            t = raw.astype(np.int64)
            rel = (t - t[0]) / 1e3
            print(f"{os.environ.get('TAG', '')} V={V} {mode:7s} walk: last CTA start {rel[7]:.2f} prologue "
                  f"{rel[10]:.2f} staged {rel[1]:.2f} loop end {rel[8]:.2f} (warp 1 {rel[12]:.2f}) barrier "
                  f"{rel[13]:.2f} rebuilt {rel[14]:.2f} epilogue end {rel[9]:.2f} end {rel[2]:.2f} signal CTAs "
                  f"{rel[15]:.2f} prefetch CTA {rel[11]:.2f} | tail start {rel[3]:.2f} slots {rel[4]:.2f} "
                  f"signals {rel[5]:.2f} FG {rel[6]:.2f} (us)")
