"""Per-rank cost of the C4 world sharded by destination target, measured on
ONE GPU, one rank at a time (a C4 engine holds ~30 GB, so the shards of a
world cannot all be resident at once): rank r's engine plans only its own
targets' vehicles (gmaco_shard_by_target), and its stage B (k_tt_refresh
over its own targets, k_colony_pro/qt/epi over its own vehicles) and its
replicated tail are timed step by step.  The other ranks' records are not
available, so their vehicles stay where they are; iteration 0 is exact and
later iterations differ from the real run only through the congestion those
frozen vehicles would have moved.  Prints one JSON line per world size:

  python tools/shard_projection.py [vehicles] [worlds...]

The NCCL exchange itself cannot be timed on one GPU; the line gives its
bytes per step (decision-record allgather + int64 deposit allreduce)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2010_14244_b200 import engine, workloads  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

if os.environ.get("LIB"):  # A/B: another build of the library
    engine.load(os.environ["LIB"])

V = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
worlds = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
STEPS = 3
net, cfg, dist, keep = workloads.c4(seed=1, max_steps=STEPS + 2, vehicles=V)


def timed(fn):
    t0 = time.perf_counter()
    fn()
    return (time.perf_counter() - t0) * 1e3


for world in worlds:
    walk = np.zeros((STEPS, world))
    tail = np.zeros((STEPS, world))
    sizes, ants = [], 0
    for r in range(world):
        e = Engine(net, cfg, dist)
        e.shard_by_target(r, world)
        sizes.append(len(e.owned))
        dec = np.full(cfg.vehicle_count, -1, dtype=np.int32)
        for k in range(STEPS):
            walk[k, r] = timed(lambda: e.step_split(1))
            d, dep = e.exchange_export()
            dec[:] = -1
            dec[e.owned] = d
            e.exchange_import(dec, dep)
            tail[k, r] = timed(lambda: e.step_split(2))
        ants += e.counters().ant_steps
        e.close()
    P = max(sizes)
    out = {"world": world, "vehicles": cfg.vehicle_count, "shard_sizes": sizes,
           "walk_ms_iter0_per_rank": walk[0].round(3).tolist(),
           "walk_ms_iter0_max": float(walk[0].max()),
           "walk_ms_mean_max": float(walk.max(axis=1).mean()),
           "tail_ms": float(tail.mean()),
           "exchange_bytes_per_step": {"allgather_records": 4 * P * world, "allreduce_deposits": 8 * net.edge_count},
           "ant_steps_total": int(ants)}
    print(json.dumps(out), flush=True)
