"""Summarise gpurun_out/ab/TAG.jsonl: mean walk / step us per library."""
import collections
import json
import sys

rows = collections.defaultdict(list)
for ln in open(sys.argv[1]):
    d = json.loads(ln)
    rows[d["lib"].split("/")[-1]].append((d["walk_ms_mean"] * 1e3, d["step_ms_mean"] * 1e3, d["step_ms_p50"] * 1e3))
for lib, v in rows.items():
    n = len(v)
    print(f"{lib:32s} walk {sum(x[0] for x in v) / n:9.2f}  step {sum(x[1] for x in v) / n:9.2f}  p50 {sum(x[2] for x in v) / n:9.2f}  (n={n})")
