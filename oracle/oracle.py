"""ctypes loaders for the CPU oracles — TEST INFRASTRUCTURE ONLY.

* PortWorld — our plain-C restatement (oracle/_build/libgmaco_oracle.so).
* RefWorld  — the unmodified reference compiled in place
              (oracle/_ref/libmacosim_ref.so, via oracle/ref_shim.cpp).

Both expose the same interface as paper_2010_14244_b200.engine.Engine so the
parity tests compare like with like.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2010_14244_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libgmaco_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmacosim_ref.so")
BRIDGE_SO = os.path.join(HERE, "_ref", "libmacosim_bridge.so")
REFERENCE_SRC = "/root/reference/proj"

P = C.POINTER
i32, i64, u64, u8, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_uint8, C.c_double


def build(force: bool = False) -> None:
    """Builds the port, and the reference library when its sources exist."""
    targets = ["port"]
    if os.path.isdir(REFERENCE_SRC):
        targets += ["ref", "bridge"]
    if force or not os.path.exists(PORT_SO) or "ref" in targets:
        subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_port = None
_ref = None


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        L = C.CDLL(PORT_SO)
        _sig(L, "og_mix64", u64, u64)
        _sig(L, "og_draw", u64, u64, u64, u64, u64)
        _sig(L, "og_to_unit", f64, u64)
        _sig(L, "og_uniform", f64, u64, f64, f64)
        _sig(L, "og_below", u64, u64, u64)
        _sig(L, "og_philox4x32_10", None, P(C.c_uint32), P(C.c_uint32), P(C.c_uint32))
        _sig(L, "og_ant_uniform", f64, C.c_int, u64, i64, i32, i32, i32)
        _sig(L, "og_tau_from_double", i64, f64)
        _sig(L, "og_evaporate_one", i64, i64, P(abi.PheromoneParams))
        _sig(L, "og_deposit_amount", i64, i64, P(abi.PheromoneParams))
        _sig(L, "og_fold_maco_edge", i64, i64, P(i32), i32, i64, P(abi.PheromoneParams))
        _sig(L, "og_select_phase", C.c_int, C.c_int, P(i32), P(f64), C.c_int, P(abi.SignalParams))
        _sig(L, "og_discharge", C.c_int, i32, P(f64), f64, C.c_int, P(abi.SignalParams))
        _sig(L, "og_validate_graph", C.c_int, P(abi.GraphDesc), C.c_char_p, i32)
        _sig(L, "og_generate_grid", C.c_int, C.c_int, C.c_int, f64, C.c_int, C.c_int, C.c_int,
             P(u8), P(i32), P(i32), P(i64), P(i32))
        _sig(L, "og_apsp", C.c_int, P(abi.GraphDesc), P(i64), P(i32))
        _sig(L, "og_dijkstra_to", C.c_int, P(abi.GraphDesc), i32, P(i64))
        _sig(L, "og_world_create", C.c_void_p, P(abi.GraphDesc), P(abi.DistanceDesc),
             P(abi.SimConfig), C.c_char_p, i32)
        _sig(L, "og_world_destroy", None, C.c_void_p)
        _sig(L, "og_world_step", i64, C.c_void_p, i64)
        _sig(L, "og_world_finished", C.c_int, C.c_void_p)
        _sig(L, "og_world_current_step", i64, C.c_void_p)
        _sig(L, "og_world_vehicles", C.c_int, C.c_void_p, P(abi.VehicleView))
        _sig(L, "og_world_signal_count", i32, C.c_void_p)
        _sig(L, "og_world_signals", C.c_int, C.c_void_p, P(abi.SignalView), i64)
        _sig(L, "og_world_pheromone", C.c_int, C.c_void_p, P(i64))
        _sig(L, "og_world_set_pheromone", C.c_int, C.c_void_p, P(i64))
        _sig(L, "og_world_occupancy", C.c_int, C.c_void_p, P(i32))
        _sig(L, "og_world_collect", C.c_int, C.c_void_p, P(abi.RunResult), P(f64), P(i32), P(i32), i32)
        _sig(L, "og_world_route", C.c_int, C.c_void_p, i32, i32, P(i32), i32, P(i32))
        _sig(L, "og_world_counters", C.c_int, C.c_void_p, P(abi.Counters))
        _sig(L, "og_world_next_node", C.c_int, C.c_void_p, C.c_int, i32, P(i32), P(i32), P(u64),
             P(u64), i64, P(i32), P(i32), P(u8))
        _sig(L, "og_world_set_vehicle_range", C.c_int, C.c_void_p, i32, i32)
        _sig(L, "og_world_step_part", C.c_int, C.c_void_p, i32)
        _sig(L, "og_world_exchange_export", C.c_int, C.c_void_p, P(i32), P(i64))
        _sig(L, "og_world_exchange_import", C.c_int, C.c_void_p, P(i32), P(i64))
        _port = L
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        L = C.CDLL(REF_SO)
        _sig(L, "ref_last_error", C.c_char_p)
        _sig(L, "ref_mix64", u64, u64)
        _sig(L, "ref_draw", u64, u64, u64, u64, u64)
        _sig(L, "ref_to_unit", f64, u64)
        _sig(L, "ref_uniform", f64, u64, f64, f64)
        _sig(L, "ref_below", u64, u64, u64)
        _sig(L, "ref_generate_grid", C.c_int, C.c_int, C.c_int, f64, C.c_int, C.c_int, P(u8), P(i32),
             P(i32), P(i64), P(i32))
        _sig(L, "ref_generate_city", C.c_int, C.c_int, C.c_int, C.c_int, u64, P(u8), P(i32), P(i32),
             P(i64), P(i32))
        _sig(L, "ref_validate_graph", C.c_int, P(abi.GraphDesc))
        _sig(L, "ref_serialize_city", C.c_int, C.c_int, C.c_int, C.c_int, u64, C.c_char_p, C.c_size_t,
             P(C.c_size_t))
        _sig(L, "ref_serialize_desc", C.c_int, P(abi.GraphDesc), C.c_char_p, C.c_size_t, P(C.c_size_t))
        _sig(L, "ref_load_network", C.c_int, C.c_char_p, C.c_size_t, P(i32), P(i32), P(u8), P(i32), P(i32),
             P(i64), P(i32), P(f64), P(f64), P(u8))
        _sig(L, "ref_apsp", C.c_int, P(abi.GraphDesc), P(i64), P(i32))
        _sig(L, "ref_evaporate_one", i64, i64, P(abi.PheromoneParams))
        _sig(L, "ref_deposit_amount", i64, i64, P(abi.PheromoneParams))
        _sig(L, "ref_fold_maco_edge", i64, i64, P(i32), i32, i64, P(abi.PheromoneParams))
        _sig(L, "ref_apply_maco_update", C.c_int, P(i64), i32, i32, P(abi.PheromoneParams))
        _sig(L, "ref_fold_bench", f64, P(i64), i32, P(i32), i32, i32, i32, P(abi.PheromoneParams))
        _sig(L, "ref_init_random", C.c_int, P(abi.GraphDesc), P(abi.PheromoneParams), u64, P(i64))
        _sig(L, "ref_select_phase", C.c_int, C.c_int, P(i32), P(f64), C.c_int, P(abi.SignalParams))
        _sig(L, "ref_discharge", C.c_int, i32, P(f64), f64, C.c_int, P(abi.SignalParams))
        _sig(L, "ref_run", C.c_int, P(abi.GraphDesc), P(abi.SimConfig), i32, P(abi.RunResult), P(f64),
             P(i32), P(i32), i32)
        _sig(L, "ref_spawn", C.c_int, P(abi.GraphDesc), P(abi.SimConfig), P(i32), P(i32), P(f64),
             P(i64), P(i64))
        _sig(L, "ref_world_create", C.c_void_p, P(abi.GraphDesc), P(abi.SimConfig))
        _sig(L, "ref_world_destroy", None, C.c_void_p)
        _sig(L, "ref_world_step", i64, C.c_void_p, i64)
        _sig(L, "ref_world_finished", C.c_int, C.c_void_p)
        _sig(L, "ref_world_current_step", i64, C.c_void_p)
        _sig(L, "ref_world_vehicles", C.c_int, C.c_void_p, P(abi.VehicleView))
        _sig(L, "ref_world_path", C.c_int, C.c_void_p, i32, P(i32), i32, P(i32))
        _sig(L, "ref_world_pheromone", C.c_int, C.c_void_p, P(i64))
        _sig(L, "ref_world_occupancy", C.c_int, C.c_void_p, P(i32))
        _sig(L, "ref_world_signal_count", i32, C.c_void_p)
        _sig(L, "ref_world_signals", C.c_int, C.c_void_p, P(abi.SignalView), i64)
        _sig(L, "ref_world_collect", C.c_int, C.c_void_p, P(abi.RunResult), P(f64), P(i32), P(i32), i32)
        _sig(L, "ref_world_next_node", C.c_int, C.c_void_p, C.c_int, i32, P(i32), P(i32), P(u64),
             P(u64), i64, P(i32), P(i32), P(u8))
        _sig(L, "ref_world_colony_iteration", i64, C.c_void_p, i32, i32, P(i64))
        _ref = L
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class _WorldBase:
    """Shared snapshot plumbing; subclasses bind the C entry points."""

    V: int
    m: int

    def vehicles(self) -> dict:
        arrs, view = abi.vehicle_arrays(self.V)
        self._vehicles(C.byref(view))
        return arrs

    def signals(self) -> dict:
        S = self.signal_count()
        arrs, view = abi.signal_arrays(S, self.V + 1)
        self._signals(C.byref(view), self.V + 1)
        total = int(arrs["queue_len"].sum())
        arrs["queue_vid"] = arrs["queue_vid"][:total]
        arrs["queue_enqueue_step"] = arrs["queue_enqueue_step"][:total]
        return arrs

    def pheromone(self) -> np.ndarray:
        t = np.zeros(self.m, dtype=np.int64)
        self._pheromone(abi.ptr(t, i64))
        return t

    def occupancy(self) -> np.ndarray:
        o = np.zeros(self.m, dtype=np.int32)
        self._occupancy(abi.ptr(o, i32))
        return o

    def collect(self):
        r = abi.RunResult()
        tt = np.zeros(self.V, dtype=np.float64)
        rv = np.zeros(self.V, dtype=np.int32)
        rn = np.zeros(self.V, dtype=np.int32)
        self._collect(C.byref(r), abi.ptr(tt, f64), abi.ptr(rv, i32), abi.ptr(rn, i32), self.V)
        k = r.retired_count
        return r, tt, list(zip(rv[:k].tolist(), rn[:k].tolist()))

    def next_node(self, algorithm, current, dest, entity=None, step=None, n_t=0):
        cur = np.ascontiguousarray(current, dtype=np.int32)
        dst = np.ascontiguousarray(dest, dtype=np.int32)
        n = len(cur)
        ent = np.ascontiguousarray(entity if entity is not None else np.zeros(n), dtype=np.uint64)
        stp = np.ascontiguousarray(step if step is not None else np.zeros(n), dtype=np.uint64)
        nxt = np.zeros(n, dtype=np.int32)
        via = np.zeros(n, dtype=np.int32)
        dev = np.zeros(n, dtype=np.uint8)
        self._next_node(algorithm, n, abi.ptr(cur, i32), abi.ptr(dst, i32), abi.ptr(ent, u64),
                        abi.ptr(stp, u64), n_t, abi.ptr(nxt, i32), abi.ptr(via, i32), abi.ptr(dev, u8))
        return nxt, via, dev

    def run(self):
        while not self.finished():
            self.step(1 << 20)
        return self.collect()


class PortWorld(_WorldBase):
    def __init__(self, net, cfg, dist: abi.DistanceDesc | None = None):
        self.L = port_lib()
        self.net = net
        self.cfg = cfg
        self.V = cfg.vehicle_count
        self.m = net.edge_count
        if dist is None:
            dist = abi.DistanceDesc(kind=abi.DIST_DENSE)
        self.dist = dist
        err = C.create_string_buffer(512)
        self.h = self.L.og_world_create(C.byref(net.desc()), C.byref(dist), C.byref(cfg), err, 512)
        if not self.h:
            raise OracleError(1, err.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.og_world_destroy(self.h)
            self.h = None

    def step(self, n=1):
        return self.L.og_world_step(self.h, n)

    def finished(self):
        return bool(self.L.og_world_finished(self.h))

    def current_step(self):
        return self.L.og_world_current_step(self.h)

    def signal_count(self):
        return self.L.og_world_signal_count(self.h)

    def _vehicles(self, v):
        self.L.og_world_vehicles(self.h, v)

    def _signals(self, v, cap):
        self.L.og_world_signals(self.h, v, cap)

    def _pheromone(self, p):
        self.L.og_world_pheromone(self.h, p)

    def set_pheromone(self, tau):
        t = np.ascontiguousarray(tau, dtype=np.int64)
        self.L.og_world_set_pheromone(self.h, abi.ptr(t, i64))

    def _occupancy(self, p):
        self.L.og_world_occupancy(self.h, p)

    def _collect(self, *a):
        self.L.og_world_collect(self.h, *a)

    def _next_node(self, *a):
        self.L.og_world_next_node(self.h, *a)

    def route(self, vid, planned=False):
        cap = self.net.node_count + 1
        out = np.zeros(max(cap, 1 << 16), dtype=np.int32)
        n = i32()
        self.L.og_world_route(self.h, vid, int(planned), abi.ptr(out, i32), len(out), C.byref(n))
        return out[: n.value].copy()

    def counters(self):
        c = abi.Counters()
        self.L.og_world_counters(self.h, C.byref(c))
        return c

    def set_shard(self, lo, hi):
        self.shard = (lo, hi)
        assert self.L.og_world_set_vehicle_range(self.h, lo, hi) == 0

    def step_split(self, part):
        return self.L.og_world_step_part(self.h, part)

    def exchange_export(self):
        lo, hi = self.shard
        dec = np.zeros(max(hi - lo, 1), dtype=np.int32)
        dep = np.zeros(self.m, dtype=np.int64)
        self.L.og_world_exchange_export(self.h, abi.ptr(dec, i32), abi.ptr(dep, i64))
        return dec[: hi - lo], dep

    def exchange_import(self, decisions, deposits):
        d = np.ascontiguousarray(decisions, dtype=np.int32)
        p = np.ascontiguousarray(deposits, dtype=np.int64)
        self.L.og_world_exchange_import(self.h, abi.ptr(d, i32), abi.ptr(p, i64))


class RefWorld(_WorldBase):
    """The unmodified reference (init_world + sequential_step), dense APSP."""

    def __init__(self, net, cfg):
        self.L = ref_lib()
        self.net = net
        self.cfg = cfg
        self.V = cfg.vehicle_count
        self.m = net.edge_count
        self.h = self.L.ref_world_create(C.byref(net.desc()), C.byref(cfg))
        if not self.h:
            raise OracleError(1, self.L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_world_destroy(self.h)
            self.h = None

    def step(self, n=1):
        return self.L.ref_world_step(self.h, n)

    def finished(self):
        return bool(self.L.ref_world_finished(self.h))

    def current_step(self):
        return self.L.ref_world_current_step(self.h)

    def signal_count(self):
        return self.L.ref_world_signal_count(self.h)

    def _vehicles(self, v):
        self.L.ref_world_vehicles(self.h, v)

    def _signals(self, v, cap):
        self.L.ref_world_signals(self.h, v, cap)

    def _pheromone(self, p):
        self.L.ref_world_pheromone(self.h, p)

    def _occupancy(self, p):
        self.L.ref_world_occupancy(self.h, p)

    def _collect(self, *a):
        self.L.ref_world_collect(self.h, *a)

    def _next_node(self, *a):
        self.L.ref_world_next_node(self.h, *a)

    def route(self, vid, planned=False):
        out = np.zeros(1 << 16, dtype=np.int32)
        n = i32()
        self.L.ref_world_path(self.h, vid, abi.ptr(out, i32), len(out), C.byref(n))
        return out[: n.value].copy()

    def colony_iteration(self, ants, threads):
        routes = i64()
        steps = self.L.ref_world_colony_iteration(self.h, ants, threads, C.byref(routes))
        return steps, routes.value


def ref_fold_bench(tau, dec_edge, iters, threads, params):
    """Seconds for `iters` passes of the reference's F+G edge kernel
    (evaporate_one(fold_maco_edge(...)) per edge, parallel.cpp:195-231) over
    `tau` (updated in place) on `threads` std::threads."""
    L = ref_lib()
    t = np.ascontiguousarray(tau, dtype=np.int64)
    d = np.ascontiguousarray(dec_edge, dtype=np.int32)
    sec = L.ref_fold_bench(abi.ptr(t, i64), len(t), abi.ptr(d, i32), len(d), iters, threads, C.byref(params))
    return sec, t


def ref_run(net, cfg, workers=0):
    """run(cfg) (workers<=0) or parallel_run(cfg, workers) of the reference."""
    L = ref_lib()
    r = abi.RunResult()
    V = cfg.vehicle_count
    tt = np.zeros(V, dtype=np.float64)
    rv = np.zeros(V, dtype=np.int32)
    rn = np.zeros(V, dtype=np.int32)
    rc = L.ref_run(C.byref(net.desc()), C.byref(cfg), workers, C.byref(r), abi.ptr(tt, f64),
                   abi.ptr(rv, i32), abi.ptr(rn, i32), V)
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    k = r.retired_count
    return r, tt, list(zip(rv[:k].tolist(), rn[:k].tolist()))


def ref_grid(rows, cols, length_m=200.0, lanes=3, interior=True):
    from paper_2010_14244_b200.networks import Network
    L = ref_lib()
    n = rows * cols
    m = 2 * (rows * (cols - 1) + cols * (rows - 1))
    sig = np.zeros(n, dtype=np.uint8)
    frm = np.zeros(m, dtype=np.int32)
    to = np.zeros(m, dtype=np.int32)
    ln = np.zeros(m, dtype=np.int64)
    la = np.zeros(m, dtype=np.int32)
    rc = L.ref_generate_grid(rows, cols, length_m, lanes, int(interior), abi.ptr(sig, u8),
                             abi.ptr(frm, i32), abi.ptr(to, i32), abi.ptr(ln, i64), abi.ptr(la, i32))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return Network(n, sig, frm, to, ln, la, grid_shape=(rows, cols))


def ref_city(nodes, links, lanes=3, seed=20250810):
    from paper_2010_14244_b200.networks import Network
    L = ref_lib()
    m = 2 * links
    sig = np.zeros(nodes, dtype=np.uint8)
    frm = np.zeros(m, dtype=np.int32)
    to = np.zeros(m, dtype=np.int32)
    ln = np.zeros(m, dtype=np.int64)
    la = np.zeros(m, dtype=np.int32)
    rc = L.ref_generate_city(nodes, links, lanes, seed, abi.ptr(sig, u8), abi.ptr(frm, i32),
                             abi.ptr(to, i32), abi.ptr(ln, i64), abi.ptr(la, i32))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return Network(nodes, sig, frm, to, ln, la)


def _ref_text(call):
    L = ref_lib()
    need = C.c_size_t()
    rc = call(None, 0, C.byref(need))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    buf = C.create_string_buffer(need.value)
    rc = call(buf, need.value, C.byref(need))
    if rc:
        raise OracleError(rc, L.ref_last_error().decode())
    return buf.raw[:need.value].decode()


def ref_serialize_city(nodes, links, lanes=3, seed=20250810) -> str:
    """serialize_network (net.cpp:179-200) of the reference's generate_city."""
    L = ref_lib()
    return _ref_text(lambda b, c, n: L.ref_serialize_city(nodes, links, lanes, seed, b, c, n))


def ref_serialize(net) -> str:
    """serialize_network of a descriptor network (reference code)."""
    L = ref_lib()
    return _ref_text(lambda b, c, n: L.ref_serialize_desc(C.byref(net.desc()), b, c, n))


def ref_load_network(text: str):
    """load_network (net.cpp:112-168) by the reference: (status, message or
    dict of SoA arrays in id order)."""
    L = ref_lib()
    raw = text.encode()
    n, m = C.c_int32(), C.c_int32()
    rc = L.ref_load_network(raw, len(raw), C.byref(n), C.byref(m), None, None, None, None, None, None, None, None)
    if rc:
        return rc, L.ref_last_error().decode()
    n, m = n.value, m.value
    a = dict(signalized=np.zeros(n, np.uint8), edge_from=np.zeros(m, np.int32), edge_to=np.zeros(m, np.int32),
             edge_length_mm=np.zeros(m, np.int64), edge_lanes=np.zeros(m, np.int32), x=np.zeros(n, np.float64),
             y=np.zeros(n, np.float64), has_position=np.zeros(n, np.uint8))
    L.ref_load_network(raw, len(raw), C.byref(C.c_int32()), C.byref(C.c_int32()), abi.ptr(a["signalized"], u8),
                       abi.ptr(a["edge_from"], i32), abi.ptr(a["edge_to"], i32), abi.ptr(a["edge_length_mm"], i64),
                       abi.ptr(a["edge_lanes"], i32), abi.ptr(a["x"], f64), abi.ptr(a["y"], f64),
                       abi.ptr(a["has_position"], u8))
    return 0, a


def results_identical(a, b) -> bool:
    """RunResult::identical_to (engine.cpp:34-40) over (RunResult, travel, retired)."""
    ra, ta, da = a
    rb, tb, db = b
    return (np.array_equal(ta, tb) and ra.mean_travel_s == rb.mean_travel_s
            and ra.mean_wait_s == rb.mean_wait_s and ra.mean_queue_len == rb.mean_queue_len
            and ra.max_edge_occupancy == rb.max_edge_occupancy
            and ra.completed_count == rb.completed_count and ra.retired_count == rb.retired_count
            and ra.steps_executed == rb.steps_executed and da == db)
