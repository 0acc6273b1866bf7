"""A/B timing of one workload on two builds of the engine library.

  python tools/ab_bench.py LIB CONFIG [steps] [warmup]

Loads LIB (a libgmaco.so build) instead of the in-tree library, then times
`steps` iterations of paper_2010_14244_b200.workloads.CONFIG with an L2 flush
before each (gmaco_bench_steps, events around the walk and the step), and
prints one JSON line: mean / p50 walk and step ms, ant-steps per step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2010_14244_b200 import engine, workloads  # noqa: E402

lib, config = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
warmup = int(sys.argv[4]) if len(sys.argv) > 4 else 3
import ctypes  # noqa: E402

_probe = ctypes.CDLL(lib)  # an older build may lack newer entry points (test hooks): bind what it has
for _name in list(engine.SIGNATURES):
    if not hasattr(_probe, _name):
        del engine.SIGNATURES[_name]
engine.load(lib)
kw = {}
if len(sys.argv) > 5:
    kw["vehicles"] = int(sys.argv[5])
if config.startswith("ref:"):  # ref:ALGORITHM:CONFIG -- a reference algorithm on a grid config (bench.py)
    import bench
    _, alg, cname = config.split(":")
    net, cfg = bench.ref_algorithm_world(alg, cname, 1, max_steps=100000)
    dist, keep = net.grid_distance(), None
else:
    net, cfg, dist, keep = workloads.CONFIGS[config](seed=1, max_steps=warmup + steps + 1, **kw)
cfg.options.flags |= int(os.environ.get("FLAGS", "0"))  # A/B of an engine option (abi.OPT_*)
e = engine.Engine(net, cfg, dist)
e.step(warmup)
c0 = e.counters()
walk, step = e.bench_steps(steps, 512 << 20, "both")
c1 = e.counters()
e.close()
# the step alone, as bench.py times it (two events per step: the walk -> tail
# programmatic launch is not broken by an event in between)
e = engine.Engine(net, cfg, dist)
e.step(warmup)
_, step_only = e.bench_steps(steps, 512 << 20, "step")
print(json.dumps({"lib": lib, "config": config, "walk_ms_mean": float(walk.mean()), "walk_ms_p50": float(np.median(walk)),
                  "step_ms_mean": float(step.mean()), "step_ms_p50": float(np.median(step)),
                  "step_only_ms_mean": float(step_only.mean()), "step_only_ms_p50": float(np.median(step_only)),
                  "ant_steps_per_step": (c1.ant_steps - c0.ant_steps) / steps}))
