"""Summarise tools/gpu/abn.sh output: mean of each metric per library path.

  python tools/ab_table.py gpurun_out/ab/TAG.jsonl"""
import collections
import json
import sys

rows = collections.defaultdict(list)
for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line)
        rows[d["lib"]].append(d)
for lib, rs in rows.items():
    keys = ("walk_ms_mean", "step_ms_mean", "step_only_ms_mean", "step_only_ms_p50")
    print(f"{lib:55s} " + "  ".join(f"{k} {1e3 * sum(r[k] for r in rs) / len(rs):8.2f}us" for k in keys) + f"  n={len(rs)}")
