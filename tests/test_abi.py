"""The C ABI boundary (include/gmaco.h) without a GPU: the in-tree library
loads, exports every declared entry point, rejects invalid input with the
reference's validation messages (status 1, before any device work) and
fails loudly (status 2) when no CUDA device exists — there is no CPU path."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, engine, networks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    L = engine.load()
    declared = engine.declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", engine.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(declared) <= exported
    assert set(engine.SIGNATURES) == set(declared)


def test_abi_version():
    assert engine.load().gmaco_abi_version() == 2


def test_struct_layouts_match_header():
    # sizes of the POD blocks as compiled into the library's callers
    assert C.sizeof(abi.PheromoneParams) == 72
    assert C.sizeof(abi.SignalParams) == 64
    assert C.sizeof(abi.RoutingParams) == 32
    assert C.sizeof(abi.ColonyParams) == 32
    assert C.sizeof(abi.EngineOptions) == 16
    assert C.sizeof(abi.SimConfig) == 320
    assert C.sizeof(abi.RunResult) == 56


def _create(net, cfg, dist=None):
    L = engine.load()
    h = C.c_void_p()
    d = dist or abi.DistanceDesc(kind=abi.DIST_DENSE)
    rc = L.gmaco_create(C.byref(net.desc()), C.byref(d), C.byref(cfg), 0, C.byref(h))
    if h:
        L.gmaco_destroy(h)
    return rc, L.gmaco_last_error(None).decode()


CONFIG_ERRORS = [
    dict(vehicle_count=0), dict(dt_s=0.0), dict(max_steps=-1), dict(decision_latency_s=-1.0),
    dict(speed_min_mps=0.0), dict(speed_min_mps=90.0), dict(spawn=abi.UNIFORM_WINDOW, spawn_window_steps=0),
]


@pytest.mark.parametrize("kw", CONFIG_ERRORS)
def test_config_validation_matches_oracle(kw):
    net = networks.grid(3, 3)
    cfg = abi.default_config(**kw)
    rc, msg = _create(net, cfg)
    assert rc == abi.EVALIDATION
    with pytest.raises(O.OracleError) as e:
        O.PortWorld(net, cfg)
    assert msg == str(e.value)


@pytest.mark.parametrize("field,val", [("rho", 1.0), ("delta_inc", 0.0), ("delta_dec", -1.0),
                                       ("tau_min", -1.0), ("tau_init_hi", 200.0)])
def test_pheromone_validation_matches_oracle(field, val):
    net = networks.grid(3, 3)
    cfg = abi.default_config()
    setattr(cfg.pheromone, field, val)
    rc, msg = _create(net, cfg)
    assert rc == abi.EVALIDATION
    with pytest.raises(O.OracleError) as e:
        O.PortWorld(net, cfg)
    assert msg == str(e.value)


def test_signal_routing_colony_validation():
    net = networks.grid(3, 3)
    for mut in (lambda c: setattr(c.signal, "th_max", 0), lambda c: setattr(c.signal, "t_max", 0.0),
                lambda c: c.signal.fixed_cycle_order.__setitem__(3, 0),
                lambda c: setattr(c.routing, "deviation_threshold", -1),
                lambda c: setattr(c.routing, "aco_beta", -1.0)):
        cfg = abi.default_config()
        mut(cfg)
        rc, msg = _create(net, cfg)
        assert rc == abi.EVALIDATION
        with pytest.raises(O.OracleError) as e:
            O.PortWorld(net, cfg)
        assert msg == str(e.value)
    cfg = abi.default_config(algorithm="colony")
    cfg.colony.ants = 0
    assert _create(net, cfg)[0] == abi.EVALIDATION


@pytest.mark.parametrize("mut,msg", [
    (lambda n: n.edge_to.__setitem__(0, 99), "edge 0 references missing node 99"),
    (lambda n: n.edge_to.__setitem__(1, n.edge_from[1]), "edge 1 is a self-loop at node"),
    (lambda n: n.edge_length_mm.__setitem__(2, 0), "edge 2 has nonpositive length"),
    (lambda n: n.edge_lanes.__setitem__(3, 0), "edge 3 has lanes < 1"),
])
def test_graph_validation(mut, msg):
    net = networks.grid(3, 3)
    mut(net)
    rc, err = _create(net, abi.default_config())
    assert rc == abi.EVALIDATION and msg in err


def test_engine_options_validation():
    """gmaco_sim_config.options (implementation switches) are validated
    before any device work: unknown bits and a negative SSSP step are status 1."""
    net = networks.grid(3, 3)
    cfg = abi.default_config()
    cfg.options.flags = 1 << 20
    rc, msg = _create(net, cfg)
    assert rc == abi.EVALIDATION and msg == "options: unknown flag bits"
    cfg = abi.default_config()
    cfg.options.sssp_delta = -1.0
    rc, msg = _create(net, cfg)
    assert rc == abi.EVALIDATION and msg == "options: sssp_delta must be >= 0"
    cfg = abi.default_config()
    cfg.options.flags = abi.OPT_REDZONES | abi.OPT_NO_PDL | abi.OPT_PROFILE_CREATE
    assert _create(net, cfg)[0] != abi.EVALIDATION  # valid switches pass validation


def test_grid_distance_requires_lattice():
    net = networks.grid(4, 4)
    net.edge_length_mm[5] += 1  # no longer uniform
    rc, err = _create(net, abi.default_config(), net.grid_distance())
    assert rc == abi.EVALIDATION and "grid distance" in err


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    rc, err = _create(networks.grid(4, 4), abi.default_config(vehicle_count=5))
    assert rc == abi.ERUNTIME and "no CUDA device" in err


def test_null_arguments_are_rejected():
    L = engine.load()
    assert L.gmaco_step(None, 1, None) == abi.EVALIDATION
    assert L.gmaco_create(None, None, None, 0, None) == abi.EVALIDATION


def test_struct_layouts_match_the_c_compiler(tmp_path):
    """ctypes mirrors (abi.py) against the header as gcc lays it out."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    structs = {"gmaco_pheromone_params": abi.PheromoneParams, "gmaco_signal_params": abi.SignalParams,
               "gmaco_routing_params": abi.RoutingParams, "gmaco_colony_params": abi.ColonyParams,
               "gmaco_engine_options": abi.EngineOptions, "gmaco_sim_config": abi.SimConfig,
               "gmaco_graph_desc": abi.GraphDesc, "gmaco_distance_desc": abi.DistanceDesc,
               "gmaco_run_result": abi.RunResult, "gmaco_vehicle_view": abi.VehicleView,
               "gmaco_signal_view": abi.SignalView, "gmaco_counters": abi.Counters}
    src = tmp_path / "sz.c"
    body = "".join(f'  printf("%zu\\n", sizeof({k}));\n' for k in structs)
    src.write_text(f'#include <stdio.h>\n#include "gmaco.h"\nint main(void) {{\n{body}  return 0;\n}}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    sizes = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    for (name, st), n in zip(structs.items(), sizes):
        assert C.sizeof(st) == n, name
