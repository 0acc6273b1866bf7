"""Vehicle sharding of one world across ranks.

Every rank holds the whole (replicated, deterministic) world and plans only
its contiguous vehicle shard.  Per step the ranks exchange exactly two
things: the shard's decision records (allgather) and its best-tour deposits
(exact int64 allreduce-sum).  On GPUs the engine does this itself over NCCL
inside the step graph (gmaco_attach_comm); this module is the host-mediated
form of the same protocol, used with any transport that offers allgather and
allreduce (torch.distributed gloo on CPU, or in-process for tests)."""
from __future__ import annotations

import numpy as np


def shard_bounds(vehicles: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard of `rank`: the padded layout the NCCL allgather uses
    (shards of ceil(V/world) vehicles; the last ones may be short)."""
    pad = -(-vehicles // world)
    return min(vehicles, rank * pad), min(vehicles, (rank + 1) * pad)


def sharded_step(w, allgather, allreduce_sum) -> None:
    """One engine step of shard `w` (an Engine or an oracle PortWorld with
    set_shard applied).  allgather(np.int32[pad]) -> concatenated rank-major
    array; allreduce_sum(np.int64[m]) -> elementwise sum over ranks."""
    lo, hi = w.shard
    pad = -(-w.V // w.world_size) if hasattr(w, "world_size") else hi - lo
    w.step_split(1)
    dec, dep = w.exchange_export()
    buf = np.full(pad, -1, dtype=np.int32)
    buf[: hi - lo] = dec
    all_dec = allgather(buf)[: w.V]
    w.exchange_import(all_dec, allreduce_sum(dep))
    w.step_split(2)


def local_transport(worlds):
    """In-process 'collectives' over a list of shards stepping in lockstep."""
    def run_step():
        for w in worlds:
            w.step_split(1)
        exported = [w.exchange_export() for w in worlds]
        pad = -(-worlds[0].V // len(worlds))
        dec = np.full(pad * len(worlds), -1, dtype=np.int32)
        for r, (d, _) in enumerate(exported):
            dec[r * pad: r * pad + len(d)] = d
        dep = np.sum([p for _, p in exported], axis=0).astype(np.int64)
        for w in worlds:
            w.exchange_import(dec[: w.V], dep)
            w.step_split(2)
    return run_step


def local_transport_owned(worlds):
    """In-process collectives for shards with explicit vehicle lists
    (Engine.shard_by_target: `owned` = the shard's vehicles in the order its
    records are exported).  Records are scattered back to vehicle order --
    what the engine's own NCCL path does on the device (k_rec_unpack)."""
    V = worlds[0].V

    def run_step():
        for w in worlds:
            w.step_split(1)
        exported = [w.exchange_export() for w in worlds]
        dec = np.full(V, -1, dtype=np.int32)
        for w, (d, _) in zip(worlds, exported):
            dec[w.owned] = d
        dep = np.sum([p for _, p in exported], axis=0).astype(np.int64)
        for w in worlds:
            w.exchange_import(dec, dep)
            w.step_split(2)
    return run_step
