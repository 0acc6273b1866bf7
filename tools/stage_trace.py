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
            # fine stamps (-DGMACO_TRACE_FINE builds) are 0 in the product build
            rel = [(x - t[0]) / 1e3 if x else None for x in t]
            names = [(7, "last CTA start"), (10, "prologue"), (1, "staged"), (8, "loop end"), (12, "warp 1"),
                     (13, "barrier"), (14, "rebuilt"), (9, "epilogue end"), (2, "end"), (15, "signal CTAs"),
                     (11, "prefetch CTA"), (3, "| tail start"), (4, "slots"), (5, "signals"), (6, "FG")]
            cols = " ".join(f"{n} {rel[i]:.2f}" for i, n in names if rel[i] is not None)
            print(f"{os.environ.get('TAG', '')} V={V} {mode:7s} walk: {cols} (us)")
