"""Road-network construction (host side, setup only — not the hot path).

`grid` reproduces the reference generator `generate_grid`
(R/src/net.cpp:208-244) edge-for-edge (same ids, order, lengths, lanes,
signal flags) and adds the "signals at every intersection" variant of
BASELINE config 2.  `random_geometric` is the scalable replacement for
`generate_city` (net.cpp:246-355, O(n^2)) used by config 4: k-nearest-neighbour
links over seeded points, components bridged, integer-mm lengths and the
reference's degree >= 3 signal rule (net.cpp:338-341).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi


@dataclass
class Network:
    node_count: int
    signalized: np.ndarray        # uint8 [n]
    edge_from: np.ndarray         # int32 [m]
    edge_to: np.ndarray           # int32 [m]
    edge_length_mm: np.ndarray    # int64 [m]
    edge_lanes: np.ndarray        # int32 [m]
    grid_shape: tuple | None = None
    _desc: abi.GraphDesc | None = field(default=None, repr=False)

    @property
    def edge_count(self) -> int:
        return int(self.edge_from.shape[0])

    def desc(self) -> abi.GraphDesc:
        if self._desc is None:
            for name in ("signalized", "edge_from", "edge_to", "edge_length_mm", "edge_lanes"):
                setattr(self, name, np.ascontiguousarray(getattr(self, name)))
            self._desc = abi.GraphDesc(
                node_count=self.node_count,
                edge_count=self.edge_count,
                signalized=abi.ptr(self.signalized, C.c_uint8),
                edge_from=abi.ptr(self.edge_from, C.c_int32),
                edge_to=abi.ptr(self.edge_to, C.c_int32),
                edge_length_mm=abi.ptr(self.edge_length_mm, C.c_int64),
                edge_lanes=abi.ptr(self.edge_lanes, C.c_int32),
            )
        return self._desc

    def grid_distance(self) -> abi.DistanceDesc:
        """Closed-form Manhattan distance service (exact for `grid`)."""
        if self.grid_shape is None:
            raise ValueError("not a grid network")
        return abi.DistanceDesc(kind=abi.DIST_GRID, grid_rows=self.grid_shape[0],
                                grid_cols=self.grid_shape[1])

    def signalized_count(self) -> int:
        return int(self.signalized.sum())


def grid(rows: int, cols: int, edge_length_m: float = 200.0, lanes: int = 3,
         signals: str = "interior") -> Network:
    """generate_grid(rows, cols, len, lanes, signalized_interior, seed)
    (net.cpp:208-244).  signals: "interior" (reference), "all" (BASELINE
    config 2: signals at every intersection) or "none"."""
    if rows < 2 or cols < 2:
        raise ValueError("grid needs rows >= 2 and cols >= 2")
    r, c = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    interior = (r > 0) & (r < rows - 1) & (c > 0) & (c < cols - 1)
    if signals == "interior":
        sig = interior
    elif signals == "all":
        sig = np.ones_like(interior)
    elif signals == "none":
        sig = np.zeros_like(interior)
    else:
        raise ValueError(signals)
    here = (r * cols + c).ravel()
    has_right = (c < cols - 1).ravel()
    has_down = (r < rows - 1).ravel()
    # per node: [right pair (2 edges)] then [down pair (2 edges)], row-major
    n_pairs = has_right.astype(np.int64) + has_down.astype(np.int64)
    m = int(2 * n_pairs.sum())
    start = np.zeros(rows * cols + 1, dtype=np.int64)
    np.cumsum(2 * n_pairs, out=start[1:])
    frm = np.empty(m, dtype=np.int32)
    to = np.empty(m, dtype=np.int32)
    o = start[:-1]
    hr = np.nonzero(has_right)[0]
    frm[o[hr]] = here[hr]; to[o[hr]] = here[hr] + 1
    frm[o[hr] + 1] = here[hr] + 1; to[o[hr] + 1] = here[hr]
    hd = np.nonzero(has_down)[0]
    od = o[hd] + 2 * has_right[hd]
    frm[od] = here[hd]; to[od] = here[hd] + cols
    frm[od + 1] = here[hd] + cols; to[od + 1] = here[hd]
    length = int(round(edge_length_m * 1000.0))  # meters_to_mm, net.cpp:34 (llround)
    return Network(
        node_count=rows * cols,
        signalized=sig.ravel().astype(np.uint8),
        edge_from=frm, edge_to=to,
        edge_length_mm=np.full(m, length, dtype=np.int64),
        edge_lanes=np.full(m, lanes, dtype=np.int32),
        grid_shape=(rows, cols),
    )


def _splitmix_unit(seed: int, stream: int, idx: np.ndarray, sub: int) -> np.ndarray:
    """Vectorized rng::to_unit(rng::draw(seed, stream, idx, sub)) (rng.hpp)."""
    M = np.uint64(0xFFFFFFFFFFFFFFFF)

    def mix(x):
        x = (x + np.uint64(0x9E3779B97F4A7C15)) & M
        x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M
        x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M
        return x ^ (x >> np.uint64(31))

    with np.errstate(over="ignore"):
        h = mix(np.full(idx.shape, np.uint64(seed), dtype=np.uint64))
        h = mix(h ^ np.uint64(stream))
        h = mix(h ^ idx.astype(np.uint64))
        h = mix(h ^ np.uint64(sub))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0**-53


def random_geometric(nodes: int, k: int = 3, lanes: int = 3, seed: int = 20250810,
                     density_per_km2: float = 100.0, links: int | None = None) -> Network:
    """Random geometric road graph: `nodes` seeded points in a square box
    (density_per_km2 points per km^2), every point linked to its k nearest
    neighbours (undirected, deduplicated), disconnected components bridged to
    their nearest outside point, each link materialized as two directed edges
    with integer-mm Euclidean lengths (>= 1 m, as net.cpp:348).  Undirected
    degree >= 3 ⇒ signalized (net.cpp:338-341).  k=3 alone gives ≈1.87·n
    undirected links; `links` tops the set up to that many undirected links
    with the shortest (k+1)-th-neighbour links (links=2·n: exactly 4M directed
    edges at 1M nodes before bridging, BASELINE config 4)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import cKDTree

    side_m = np.sqrt(nodes / density_per_km2) * 1000.0
    idx = np.arange(nodes, dtype=np.uint64)
    pts = np.stack([_splitmix_unit(seed, 6, idx, 0), _splitmix_unit(seed, 6, idx, 1)], axis=1) * side_m
    tree = cKDTree(pts)
    dd, nn = tree.query(pts, k=k + 2)
    a = np.repeat(np.arange(nodes), k)
    b = nn[:, 1:k + 1].ravel()
    lo = np.minimum(a, b).astype(np.int64)
    hi = np.maximum(a, b).astype(np.int64)
    key = np.unique(lo * nodes + hi)
    if links is not None and len(key) < links:
        # shortest (k+1)-th-neighbour links not already present, in (length, key) order
        xa = np.arange(nodes, dtype=np.int64)
        xb = nn[:, k + 1].astype(np.int64)
        xkey = np.minimum(xa, xb) * nodes + np.maximum(xa, xb)
        order = np.lexsort((xkey, dd[:, k + 1]))
        xkey = xkey[order]
        _, first = np.unique(xkey, return_index=True)
        xkey = xkey[np.sort(first)]
        xkey = xkey[~np.isin(xkey, key)]
        key = np.unique(np.concatenate([key, xkey[:links - len(key)]]))
    lo, hi = key // nodes, key % nodes
    # bridge components: connect each non-giant component to the nearest point outside it
    while True:
        g = coo_matrix((np.ones(len(lo)), (lo, hi)), shape=(nodes, nodes))
        ncomp, label = connected_components(g, directed=False)
        if ncomp == 1:
            break
        giant = np.bincount(label).argmax()
        outside = np.nonzero(label == giant)[0]
        otree = cKDTree(pts[outside])
        add_lo, add_hi = [], []
        for comp in np.unique(label):
            if comp == giant:
                continue
            members = np.nonzero(label == comp)[0]
            d, j = otree.query(pts[members], k=1)
            best = int(np.argmin(d))
            u, v = int(members[best]), int(outside[j[best]])
            add_lo.append(min(u, v)); add_hi.append(max(u, v))
        key = np.unique(np.concatenate([lo * nodes + hi, np.array(add_lo) * nodes + np.array(add_hi)]))
        lo, hi = key // nodes, key % nodes
    deg = np.bincount(lo, minlength=nodes) + np.bincount(hi, minlength=nodes)
    d = np.sqrt(((pts[lo] - pts[hi]) ** 2).sum(axis=1))
    length = np.maximum(1000, np.rint(d * 1000.0)).astype(np.int64)
    npairs = len(lo)
    frm = np.empty(2 * npairs, dtype=np.int32)
    to = np.empty(2 * npairs, dtype=np.int32)
    frm[0::2], to[0::2] = lo, hi
    frm[1::2], to[1::2] = hi, lo
    return Network(
        node_count=nodes,
        signalized=(deg >= 3).astype(np.uint8),
        edge_from=frm, edge_to=to,
        edge_length_mm=np.repeat(length, 2),
        edge_lanes=np.full(2 * npairs, lanes, dtype=np.int32),
    )


# ---- reference-schema JSON (load_network / serialize_network, net.cpp:112-209) ----

def _net_check(L, rc):
    if rc != 0:
        from .engine import EngineError
        raise EngineError(rc, L.gmaco_network_last_error().decode())


def _from_handle(L, h) -> "Network":
    n, m = C.c_int32(), C.c_int32()
    L.gmaco_network_info(h, C.byref(n), C.byref(m))
    n, m = n.value, m.value
    sig = np.zeros(n, np.uint8)
    frm, to, lanes = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m, np.int32)
    ln = np.zeros(m, np.int64)
    x, y, hp = np.zeros(n, np.float64), np.zeros(n, np.float64), np.zeros(n, np.uint8)
    _net_check(L, L.gmaco_network_export(h, abi.ptr(sig, C.c_uint8), abi.ptr(frm, C.c_int32), abi.ptr(to, C.c_int32),
                                         abi.ptr(ln, C.c_int64), abi.ptr(lanes, C.c_int32), abi.ptr(x, C.c_double),
                                         abi.ptr(y, C.c_double), abi.ptr(hp, C.c_uint8)))
    net = Network(node_count=n, signalized=sig, edge_from=frm, edge_to=to, edge_length_mm=ln, edge_lanes=lanes)
    net.positions = (x, y, hp) if hp.any() else None
    return net


def parse_json(text: str) -> "Network":
    """load_network (net.cpp:112-168): a reference-schema network from JSON
    text, parsed natively by the engine library (gmaco_network_parse)."""
    from .engine import load
    L = load()
    h = C.c_void_p()
    raw = text.encode()
    _net_check(L, L.gmaco_network_parse(raw, len(raw), C.byref(h)))
    try:
        return _from_handle(L, h)
    finally:
        L.gmaco_network_free(h)


def load_json(path: str) -> "Network":
    """load_network_file (net.cpp:170-176) via gmaco_network_load_file."""
    from .engine import load
    L = load()
    h = C.c_void_p()
    _net_check(L, L.gmaco_network_load_file(path.encode(), C.byref(h)))
    try:
        return _from_handle(L, h)
    finally:
        L.gmaco_network_free(h)


def _pos_args(net):
    pos = getattr(net, "positions", None)
    if pos is None:
        return None, None, None
    x, y, hp = (np.ascontiguousarray(a) for a in pos)
    return abi.ptr(x, C.c_double), abi.ptr(y, C.c_double), abi.ptr(hp, C.c_uint8)


def serialize_json(net: "Network") -> str:
    """serialize_network (net.cpp:179-200): the reference's dump(2) text."""
    from .engine import load
    L = load()
    px, py, ph = _pos_args(net)
    need = C.c_size_t()
    _net_check(L, L.gmaco_network_serialize(C.byref(net.desc()), px, py, ph, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _net_check(L, L.gmaco_network_serialize(C.byref(net.desc()), px, py, ph, buf, need.value, C.byref(need)))
    return buf.raw[:need.value].decode()


def save_json(net: "Network", path: str) -> None:
    """write_network_file (net.cpp:202-206)."""
    from .engine import load
    L = load()
    px, py, ph = _pos_args(net)
    _net_check(L, L.gmaco_network_write_file(C.byref(net.desc()), px, py, ph, path.encode()))
