"""Per-stage device trace of one engine step for a BASELINE config.

  python tools/stage_trace_cfg.py c1|c2|c3|c5     (L2 flushed before each traced step)
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2010_14244_b200 import workloads  # noqa: E402
from paper_2010_14244_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
net, cfg, dist, keep = workloads.CONFIGS[name](max_steps=60)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
e = Engine(net, cfg, dist)
e.step(5)
for rep in range(4):
    flush.fill_(rep + 1)
    torch.cuda.synchronize()
    t = e.debug_trace(1).astype(np.int64)
    rel = (t - t[0]) / 1e3
    print(f"{name} walk: staged {rel[1]:.2f} end {rel[2]:.2f} | tail start {rel[3]:.2f} FG {rel[6]:.2f} (us)")
