"""Reference-schema network files: the engine library's
native loader / writer (gmaco_network_*) against the reference's own
load_network / serialize_network (net.cpp:112-209, compiled into
oracle/_ref): identical parsed arrays, byte-identical text, identical
status and message on malformed documents.  CPU only."""
import json
import os
import time

import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import networks
from paper_2010_14244_b200.engine import EngineError

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference library not built")

FIELDS = ("signalized", "edge_from", "edge_to", "edge_length_mm", "edge_lanes")


def _same(ours, ref):
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(ours, f)), ref[f]), f
    if ref["has_position"].any():
        x, y, hp = ours.positions
        assert np.array_equal(hp, ref["has_position"])
        assert np.array_equal(x, ref["x"]) and np.array_equal(y, ref["y"])


@pytest.mark.parametrize("nodes,links,seed", [(52, 64, 20250810), (30, 45, 7), (120, 200, 3)])
def test_city_text_and_arrays_match_reference(nodes, links, seed):
    text = O.ref_serialize_city(nodes, links, seed=seed)
    ours = networks.parse_json(text)
    rc, ref = O.ref_load_network(text)
    assert rc == 0
    _same(ours, ref)
    assert networks.serialize_json(ours) == text  # nlohmann dump(2), byte for byte


@pytest.mark.parametrize("net", [networks.grid(6, 9, 137.5, 2, "all"), networks.grid(10, 10)])
def test_grid_text_matches_reference(net):
    text = networks.serialize_json(net)
    assert text == O.ref_serialize(net)
    rc, ref = O.ref_load_network(text)
    assert rc == 0
    _same(networks.parse_json(text), ref)


def test_millimetre_lengths_round_trip():
    """Integer-mm lengths of a random-geometric graph survive length_m text and
    meters_to_mm (llround(m * 1000), net.cpp:34) on both sides."""
    net = networks.random_geometric(3000, k=3, seed=11)
    text = networks.serialize_json(net)
    assert text == O.ref_serialize(net)
    back = networks.parse_json(text)
    assert np.array_equal(back.edge_length_mm, net.edge_length_mm)
    rc, ref = O.ref_load_network(text)
    assert rc == 0
    _same(back, ref)


def test_node_and_edge_order_is_by_id():
    doc = {"edges": [{"id": 1, "from": 1, "to": 0, "length_m": 2.5, "lanes": 1},
                     {"id": 0, "from": 0, "to": 1, "length_m": 0.0015, "lanes": 2}],
           "nodes": [{"id": 1, "signalized": True}, {"id": 0, "signalized": False, "x": 1.5, "y": -2.0}]}
    text = json.dumps(doc)
    ours = networks.parse_json(text)
    rc, ref = O.ref_load_network(text)
    assert rc == 0
    _same(ours, ref)
    assert list(ours.edge_length_mm) == [2, 2500]  # llround(1.5) = 2


BAD = [
    "[]",
    '{"nodes": []}',
    '{"nodes": [], "edges": [], "zzz": 1, "aaa": 2}',
    '{"nodes": [], "edges": []}',
    '{"nodes": [1], "edges": []}',
    '{"nodes": [{"signalized": true}], "edges": []}',
    '{"nodes": [{"id": 0.0, "signalized": true}], "edges": []}',
    '{"nodes": [{"id": 0, "signalized": 1}], "edges": []}',
    '{"nodes": [{"id": 0, "signalized": true, "x": 1}], "edges": []}',
    '{"nodes": [{"id": 0, "signalized": true, "w": 1, "q": 2}], "edges": []}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [5]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 0, "to": 1, "length_m": 1}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 0, "to": 1, "length_m": "1", "lanes": 1}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 0, "to": 1, "length_m": 1, "lanes": 1.0}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 3, "from": 0, "to": 1, "length_m": 1, "lanes": 1}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 0, "signalized": false}], "edges": []}',
    '{"nodes": [{"id": 2, "signalized": true}, {"id": 0, "signalized": false}], "edges": []}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 0, "to": 7, "length_m": 1, "lanes": 1}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 1, "to": 1, "length_m": 1, "lanes": 1}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 0, "to": 1, "length_m": 0.0001, "lanes": 1}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 0, "to": 1, "length_m": 1, "lanes": 0}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 0, "to": 1, "length_m": 1, "lanes": 1}, {"id": 0, "from": 1, "to": 0, "length_m": 1, "lanes": 1}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": 0, "to": 1, "length_m": 1, "lanes": 1}, {"id": 1, "from": 0, "to": 1, "length_m": 2, "lanes": 1}]}',
    '{"nodes": [{"id": 0, "signalized": true}, {"id": 1, "signalized": false}], "edges": [{"id": 0, "from": "0", "to": 1, "length_m": 1, "lanes": 1}]}',
]


@pytest.mark.parametrize("text", BAD)
def test_malformed_documents_match_reference(text):
    rc, ref_msg = O.ref_load_network(text)
    assert rc != 0
    with pytest.raises(EngineError) as ei:
        networks.parse_json(text)
    assert ei.value.code == rc
    if rc == 1:
        assert str(ei.value).endswith(ref_msg), (str(ei.value), ref_msg)


def test_parse_error_is_a_validation_error():
    for text in ['{"nodes": [', '{"nodes": [], "edges": [] } x', "{'nodes': []}"]:
        rc, _ = O.ref_load_network(text)
        with pytest.raises(EngineError) as ei:
            networks.parse_json(text)
        assert rc == 1 and ei.value.code == 1 and "network parse error" in str(ei.value)


def test_file_round_trip_and_scale(tmp_path):
    """write_network_file / load_network_file at 2*10^5 nodes (~7.5*10^5
    edges): native text I/O in seconds, arrays unchanged."""
    net = networks.random_geometric(200_000, k=3, seed=5)
    path = os.path.join(tmp_path, "rgg.json")
    t0 = time.perf_counter()
    networks.save_json(net, path)
    t1 = time.perf_counter()
    back = networks.load_json(path)
    t2 = time.perf_counter()
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(back, f)), np.asarray(getattr(net, f))), f
    assert t1 - t0 < 20 and t2 - t1 < 20, (t1 - t0, t2 - t1)
