"""ctypes binding of libgmaco.so (the C ABI in include/gmaco.h).

`Engine` exposes the same interface as the oracle worlds (oracle/oracle.py)
so parity tests compare like with like.  There is no fallback: if the
in-tree library is missing, or no CUDA device is present, construction
raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libgmaco.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "gmaco.h")

P = C.POINTER
i32, i64, u64, u8, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_uint8, C.c_double

# every entry point include/gmaco.h declares, with its ctypes signature
SIGNATURES = {
    "gmaco_abi_version": (i32,),
    "gmaco_create": (C.c_int, P(abi.GraphDesc), P(abi.DistanceDesc), P(abi.SimConfig), i32, P(C.c_void_p)),
    "gmaco_attach_comm": (C.c_int, C.c_void_p, i32, i32, C.c_void_p),
    "gmaco_nccl_unique_id": (C.c_int, C.c_void_p),
    "gmaco_step": (C.c_int, C.c_void_p, i64, P(i64)),
    "gmaco_finished": (C.c_int, C.c_void_p, P(i32)),
    "gmaco_run": (C.c_int, C.c_void_p, P(abi.RunResult), P(f64)),
    "gmaco_collect": (C.c_int, C.c_void_p, P(abi.RunResult), P(f64), P(i32), P(i32), i32),
    "gmaco_get_pheromone": (C.c_int, C.c_void_p, P(i64)),
    "gmaco_set_pheromone": (C.c_int, C.c_void_p, P(i64)),
    "gmaco_get_occupancy": (C.c_int, C.c_void_p, P(i32)),
    "gmaco_get_vehicles": (C.c_int, C.c_void_p, P(abi.VehicleView)),
    "gmaco_get_signals": (C.c_int, C.c_void_p, P(abi.SignalView), i64),
    "gmaco_signal_count": (C.c_int, C.c_void_p, P(i32)),
    "gmaco_get_counters": (C.c_int, C.c_void_p, P(abi.Counters)),
    "gmaco_current_step": (C.c_int, C.c_void_p, P(i64)),
    "gmaco_route_query": (C.c_int, C.c_void_p, i32, i32, P(i32), i32, P(i32)),
    "gmaco_next_node": (C.c_int, C.c_void_p, i32, i32, P(i32), P(i32), P(u64), P(u64), i64, P(i32), P(i32),
                        P(u8)),
    "gmaco_last_timing": (C.c_int, C.c_void_p, P(f64), P(f64), P(i64)),
    "gmaco_set_timing": (C.c_int, C.c_void_p, i32),
    "gmaco_bench_steps": (C.c_int, C.c_void_p, i32, i64, P(f64), P(f64)),
    "gmaco_debug_trace": (C.c_int, C.c_void_p, i32, P(u64)),
    "gmaco_debug_check_redzones": (C.c_int, C.c_void_p, P(i64)),
    "gmaco_debug_roulette_threshold": (C.c_int, C.c_void_p, i32, P(C.c_double), P(C.c_double), P(u64)),
    "gmaco_set_shard": (C.c_int, C.c_void_p, i32, i32),
    "gmaco_step_split": (C.c_int, C.c_void_p, i32),
    "gmaco_shard_by_target": (C.c_int, C.c_void_p, i32, i32),
    "gmaco_shard_vehicles": (C.c_int, C.c_void_p, P(i32), i32, P(i32)),
    "gmaco_exchange_export": (C.c_int, C.c_void_p, P(i32), P(i64)),
    "gmaco_exchange_import": (C.c_int, C.c_void_p, P(i32), P(i64)),
    "gmaco_network_parse": (C.c_int, C.c_char_p, C.c_size_t, P(C.c_void_p)),
    "gmaco_network_load_file": (C.c_int, C.c_char_p, P(C.c_void_p)),
    "gmaco_network_info": (C.c_int, C.c_void_p, P(i32), P(i32)),
    "gmaco_network_export": (C.c_int, C.c_void_p, P(u8), P(i32), P(i32), P(i64), P(i32), P(f64), P(f64), P(u8)),
    "gmaco_network_free": (None, C.c_void_p),
    "gmaco_network_serialize": (C.c_int, P(abi.GraphDesc), P(f64), P(f64), P(u8), C.c_char_p, C.c_size_t,
                                P(C.c_size_t)),
    "gmaco_network_write_file": (C.c_int, P(abi.GraphDesc), P(f64), P(f64), P(u8), C.c_char_p),
    "gmaco_network_last_error": (C.c_char_p,),
    "gmaco_vehicles_enqueue": (C.c_int, C.c_void_p, P(abi.VehicleView), i32),
    "gmaco_step_snapshot": (C.c_int, C.c_void_p, P(abi.VehicleView), i32),
    "gmaco_vehicles_wait": (C.c_int, C.c_void_p, i32, P(abi.VehicleView)),
    "gmaco_last_error": (C.c_char_p, C.c_void_p),
    "gmaco_destroy": (None, C.c_void_p),
}

_lib = None


class EngineError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[status {code}] {msg}")
        self.code = code


def load(path: str = LIB_PATH):
    """Loads the in-tree engine library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise EngineError(abi.ERUNTIME, f"engine library not built: {path} (run __graft_entry__.build())")
        L = C.CDLL(path)
        for name, sig in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = sig[0]
            f.argtypes = list(sig[1:])
        _lib = L
    return _lib


class Engine:
    """One device world (gmaco_create ... gmaco_destroy)."""

    def __init__(self, net, cfg: abi.SimConfig, dist: abi.DistanceDesc | None = None, device: int = 0):
        self.L = load()
        self.net = net
        self.cfg = cfg
        self.V = cfg.vehicle_count
        self.m = net.edge_count
        self.dist = dist if dist is not None else abi.DistanceDesc(kind=abi.DIST_DENSE)
        h = C.c_void_p()
        rc = self.L.gmaco_create(C.byref(net.desc()), C.byref(self.dist), C.byref(cfg), device, C.byref(h))
        if rc:
            raise EngineError(rc, self.L.gmaco_last_error(None).decode())
        self.h = h

    def _check(self, rc):
        if rc:
            raise EngineError(rc, self.L.gmaco_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.L.gmaco_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # -- stepping ---------------------------------------------------------------
    def step(self, n: int = 1, count: bool = True):
        """Run up to n steps; returns the number executed, or None with
        count=False (steps only enqueued; later reads are ordered after them)."""
        if not count:
            self._check(self.L.gmaco_step(self.h, n, None))
            return None
        k = i64()
        self._check(self.L.gmaco_step(self.h, n, C.byref(k)))
        return k.value

    def finished(self) -> bool:
        f = i32()
        self._check(self.L.gmaco_finished(self.h, C.byref(f)))
        return bool(f.value)

    def current_step(self) -> int:
        s = i64()
        self._check(self.L.gmaco_current_step(self.h, C.byref(s)))
        return s.value

    def run(self):
        r = abi.RunResult()
        tt = np.zeros(self.V, dtype=np.float64)
        self._check(self.L.gmaco_run(self.h, C.byref(r), abi.ptr(tt, f64)))
        return self.collect()

    # -- snapshots --------------------------------------------------------------
    def collect(self):
        r = abi.RunResult()
        tt = np.zeros(self.V, dtype=np.float64)
        rv = np.zeros(self.V, dtype=np.int32)
        rn = np.zeros(self.V, dtype=np.int32)
        self._check(self.L.gmaco_collect(self.h, C.byref(r), abi.ptr(tt, f64), abi.ptr(rv, i32),
                                         abi.ptr(rn, i32), self.V))
        k = r.retired_count
        return r, tt, list(zip(rv[:k].tolist(), rn[:k].tolist()))

    def vehicles_enqueue(self, view, slot: int) -> None:
        """Snapshot the view's fields after all enqueued steps into slot 0/1 (no wait)."""
        self._check(self.L.gmaco_vehicles_enqueue(self.h, C.byref(view), slot))

    def step_snapshot(self, view, slot: int) -> None:
        """One step, then the view's fields snapshotted into slot 0/1: one graph launch, no wait."""
        self._check(self.L.gmaco_step_snapshot(self.h, C.byref(view), slot))

    def vehicles_wait(self, slot: int, view) -> None:
        """Wait for slot's snapshot and copy it into view."""
        self._check(self.L.gmaco_vehicles_wait(self.h, slot, C.byref(view)))

    def vehicles(self) -> dict:
        arrs, view = abi.vehicle_arrays(self.V)
        self._check(self.L.gmaco_get_vehicles(self.h, C.byref(view)))
        return arrs

    def signal_count(self) -> int:
        s = i32()
        self._check(self.L.gmaco_signal_count(self.h, C.byref(s)))
        return s.value

    def signals(self) -> dict:
        S = self.signal_count()
        arrs, view = abi.signal_arrays(S, self.V + 1)
        self._check(self.L.gmaco_get_signals(self.h, C.byref(view), self.V + 1))
        total = int(arrs["queue_len"].sum())
        arrs["queue_vid"] = arrs["queue_vid"][:total]
        arrs["queue_enqueue_step"] = arrs["queue_enqueue_step"][:total]
        return arrs

    def pheromone(self) -> np.ndarray:
        t = np.zeros(self.m, dtype=np.int64)
        self._check(self.L.gmaco_get_pheromone(self.h, abi.ptr(t, i64)))
        return t

    def set_pheromone(self, tau):
        t = np.ascontiguousarray(tau, dtype=np.int64)
        self._check(self.L.gmaco_set_pheromone(self.h, abi.ptr(t, i64)))

    def occupancy(self) -> np.ndarray:
        o = np.zeros(self.m, dtype=np.int32)
        self._check(self.L.gmaco_get_occupancy(self.h, abi.ptr(o, i32)))
        return o

    def counters(self) -> abi.Counters:
        c = abi.Counters()
        self._check(self.L.gmaco_get_counters(self.h, C.byref(c)))
        return c

    def route(self, vid: int, planned: bool = False) -> np.ndarray:
        cap = max(self.net.node_count, 1 << 16)
        out = np.zeros(cap, dtype=np.int32)
        n = i32()
        self._check(self.L.gmaco_route_query(self.h, vid, int(planned), abi.ptr(out, i32), cap, C.byref(n)))
        return out[: n.value].copy()

    def next_node(self, algorithm, current, dest, entity=None, step=None, n_t=0):
        cur = np.ascontiguousarray(current, dtype=np.int32)
        dst = np.ascontiguousarray(dest, dtype=np.int32)
        n = len(cur)
        ent = np.ascontiguousarray(entity if entity is not None else np.zeros(n), dtype=np.uint64)
        stp = np.ascontiguousarray(step if step is not None else np.zeros(n), dtype=np.uint64)
        nxt = np.zeros(n, dtype=np.int32)
        via = np.zeros(n, dtype=np.int32)
        dev = np.zeros(n, dtype=np.uint8)
        self._check(self.L.gmaco_next_node(self.h, algorithm, n, abi.ptr(cur, i32), abi.ptr(dst, i32),
                                           abi.ptr(ent, u64), abi.ptr(stp, u64), n_t, abi.ptr(nxt, i32),
                                           abi.ptr(via, i32), abi.ptr(dev, u8)))
        return nxt, via, dev

    # -- timing -----------------------------------------------------------------
    def set_timing(self, on: bool):
        self._check(self.L.gmaco_set_timing(self.h, int(on)))

    def bench_steps(self, steps: int, flush_bytes: int, what: str = "both"):
        """Per-step device times in ms of `steps` back-to-back steps with an L2
        flush before each (outside the events).  what = "step" (whole step,
        two events), "walk" (stage-B walk, two events) or "both" (three
        events); returns (walk, step), None for the leg not timed."""
        walk = np.zeros(steps, dtype=np.float64) if what in ("walk", "both") else None
        step = np.zeros(steps, dtype=np.float64) if what in ("step", "both") else None
        self._check(self.L.gmaco_bench_steps(self.h, steps, flush_bytes,
                                             abi.ptr(walk, f64) if walk is not None else None,
                                             abi.ptr(step, f64) if step is not None else None))
        return walk, step

    def debug_trace(self, steps: int = 1) -> np.ndarray:
        """Stage timestamps (ns) of the last of `steps` steps (DevCtl::trace)."""
        out = np.zeros(16, dtype=np.uint64)
        self._check(self.L.gmaco_debug_trace(self.h, steps, abi.ptr(out, u64)))
        return out

    def roulette_threshold(self, wa: np.ndarray, wb: np.ndarray) -> np.ndarray:
        """The lattice walker's integer roulette thresholds (LatRec.thr) of
        candidate weight pairs (gmaco_debug_roulette_threshold)."""
        wa = np.ascontiguousarray(wa, dtype=np.float64)
        wb = np.ascontiguousarray(wb, dtype=np.float64)
        out = np.zeros(len(wa), dtype=np.uint64)
        self._check(self.L.gmaco_debug_roulette_threshold(self.h, len(wa), abi.ptr(wa, C.c_double),
                                                          abi.ptr(wb, C.c_double), abi.ptr(out, u64)))
        return out

    # -- sharding (multi-GPU) -----------------------------------------------------
    def check_redzones(self) -> tuple[int, str]:
        """(overwritten guard bands, message) of a world created with
        abi.OPT_REDZONES."""
        n = i64()
        self._check(self.L.gmaco_debug_check_redzones(self.h, C.byref(n)))
        return n.value, self.L.gmaco_last_error(self.h).decode()

    def attach_comm(self, rank: int, world: int, nccl_id: bytes):
        buf = C.create_string_buffer(nccl_id, 128)
        self._check(self.L.gmaco_attach_comm(self.h, rank, world, buf))

    def set_shard(self, lo: int, hi: int):
        self.shard = (lo, hi)
        self._check(self.L.gmaco_set_shard(self.h, lo, hi))

    def shard_by_target(self, rank: int, world: int):
        """By-target shard (per-target-row worlds): plans the vehicles bound
        for the targets dealt to `rank`; self.owned lists them."""
        self._check(self.L.gmaco_shard_by_target(self.h, rank, world))
        n = i32()
        self._check(self.L.gmaco_shard_vehicles(self.h, None, 0, C.byref(n)))
        vids = np.zeros(max(n.value, 1), dtype=np.int32)
        self._check(self.L.gmaco_shard_vehicles(self.h, abi.ptr(vids, i32), len(vids), C.byref(n)))
        self.owned = vids[: n.value].copy()
        self.shard = (0, n.value)

    def step_split(self, part: int):
        self._check(self.L.gmaco_step_split(self.h, part))

    def exchange_export(self):
        lo, hi = self.shard
        dec = np.zeros(max(hi - lo, 1), dtype=np.int32)
        dep = np.zeros(self.m, dtype=np.int64)
        self._check(self.L.gmaco_exchange_export(self.h, abi.ptr(dec, i32), abi.ptr(dep, i64)))
        return dec[: hi - lo], dep

    def exchange_import(self, decisions, deposits):
        d = np.ascontiguousarray(decisions, dtype=np.int32)
        p = np.ascontiguousarray(deposits, dtype=np.int64)
        self._check(self.L.gmaco_exchange_import(self.h, abi.ptr(d, i32), abi.ptr(p, i64)))

    def last_timing(self):
        a, b, n = f64(), f64(), i64()
        self._check(self.L.gmaco_last_timing(self.h, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value


def declared_symbols(header: str = HEADER) -> list[str]:
    """Function names declared in include/gmaco.h."""
    import re
    text = open(header).read()
    return sorted(set(re.findall(r"\b(gmaco_[a-z_0-9]+)\s*\(", text)))
