"""The reference-side drop-in: integration/macosim_gpu.cpp's gpu_run(),
compiled against the reference headers and linked with the reference and
libgmaco.so (oracle/_ref/libmacosim_bridge.so), must return a RunResult that
the reference's own RunResult::identical_to (engine.cpp:34-40) accepts as
identical to run(cfg, dist).  The reference harness patched with the "gpu"
executor (oracle/harness_gpu.patch: harness.cpp:118-127 validation,
harness.cpp:345-346 dispatch) runs a scenario matrix whose gpu rows carry the
same metric columns as the sequential rows."""
import csv
import ctypes as C
import json
import os

import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks

pytestmark = pytest.mark.skipif(not os.path.exists(O.BRIDGE_SO), reason="integration bridge not built")


def bridge():
    L = C.CDLL(O.BRIDGE_SO)
    L.bridge_identical.restype = C.c_int
    L.bridge_identical.argtypes = [C.POINTER(abi.GraphDesc), C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int]
    L.bridge_run_matrix.restype = C.c_int
    L.bridge_run_matrix.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
    L.bridge_load_scenario.restype = C.c_int
    L.bridge_load_scenario.argtypes = [C.c_char_p]
    L.bridge_last_error.restype = C.c_char_p
    return L


def test_bridge_links_and_exports():
    L = bridge()
    assert hasattr(L, "bridge_identical")
    assert hasattr(L, "_ZN7macosim7gpu_runERKNS_9SimConfigERKNS_13DistanceTableEi")
    assert hasattr(L, "_ZN7macosim7gpu_runERKNS_9SimConfigEi")
    assert hasattr(L, "_ZN7macosim10run_matrixERKNS_8ScenarioERKNS_11RoadNetworkEiPSo")


def scenario(executors, **kw):
    doc = {"network": {"grid": {"rows": 6, "cols": 7}},
           "algorithms": ["dijkstra", "aco", "maco", "maco-p"],
           "executors": executors, "vehicle_counts": [40, 120], "seeds": [1, 2],
           "engine": {"max_steps": 400}}
    doc.update(kw)
    return json.dumps(doc).encode()


def test_patched_harness_accepts_gpu_executor():
    """load_scenario (patched) accepts "gpu" and still rejects unknown names
    with the reference's message style."""
    L = bridge()
    assert L.bridge_load_scenario(scenario(["sequential", "gpu"])) == 0
    assert L.bridge_load_scenario(scenario(["sequential", "cuda"])) == 1
    assert L.bridge_last_error() == b'scenario: executor must be "sequential", "parallel" or "gpu"'


@pytest.mark.gpu
@pytest.mark.parametrize("alg", [0, 1, 2, 3])
def test_gpu_run_identical_to_reference_run(alg):
    L = bridge()
    for net, V in ((networks.grid(10, 10), 100), (networks.grid(32, 32, signals="all"), 1000)):
        for seed in (1, 2):
            rc = L.bridge_identical(C.byref(net.desc()), alg, V, seed, 0, 1)
            assert rc == 1, (alg, seed, L.bridge_last_error())


@pytest.mark.gpu
@pytest.mark.parametrize("alg", [0, 1, 2, 3])
def test_gpu_run_without_table_uses_device_sssp(alg):
    """gpu_run(cfg, device): no host all_pairs_distances; the engine's device
    SSSP builds the exact table, and the result is still identical_to run()."""
    L = bridge()
    net = O.ref_city(52, 64) if O.ref_available() else networks.grid(12, 12)
    for seed in (1, 3):
        rc = L.bridge_identical(C.byref(net.desc()), alg, 200, seed, 0, 0)
        assert rc == 1, (alg, seed, L.bridge_last_error())


@pytest.mark.gpu
def test_run_matrix_gpu_executor_csv(tmp_path):
    """Scenario with executors [sequential, parallel, gpu] -> run_matrix ->
    write_results_csv -> read back: every gpu row's metric columns equal the
    sequential row of the same (algorithm, vehicle_count, seed)."""
    L = bridge()
    out, rep = tmp_path / "results.csv", tmp_path / "report.txt"
    n = L.bridge_run_matrix(scenario(["sequential", "parallel", "gpu"]), str(out).encode(), str(rep).encode(), 4)
    assert n == 4 * 3 * 2 * 2, L.bridge_last_error()
    with open(out) as f:
        rows = list(csv.DictReader(f))
    assert list(rows[0].keys()) == ["algorithm", "executor", "vehicle_count", "seed", "mean_travel_s",
                                    "mean_wait_s", "wall_clock_ms"]
    by = {}
    for r in rows:
        by[(r["algorithm"], r["executor"], r["vehicle_count"], r["seed"])] = r
    gpu_rows = [k for k in by if k[1] == "gpu"]
    assert len(gpu_rows) == 16
    for alg, _, cnt, seed in gpu_rows:
        for ex in ("sequential", "parallel"):
            ref = by[(alg, ex, cnt, seed)]
            got = by[(alg, "gpu", cnt, seed)]
            assert got["mean_travel_s"] == ref["mean_travel_s"], (alg, ex, cnt, seed)
            assert got["mean_wait_s"] == ref["mean_wait_s"], (alg, ex, cnt, seed)
    assert "maco-p" in rep.read_text()
