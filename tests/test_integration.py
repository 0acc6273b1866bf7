"""The reference-side drop-in: integration/macosim_gpu.cpp's gpu_run(),
compiled against the reference headers and linked with the reference and
libgmaco.so (oracle/_ref/libmacosim_bridge.so), must return a RunResult that
the reference's own RunResult::identical_to (engine.cpp:34-40) accepts as
identical to run(cfg, dist)."""
import ctypes as C
import os

import pytest

from oracle import oracle as O
from paper_2010_14244_b200 import abi, networks

pytestmark = pytest.mark.skipif(not os.path.exists(O.BRIDGE_SO), reason="integration bridge not built")


def bridge():
    L = C.CDLL(O.BRIDGE_SO)
    L.bridge_identical.restype = C.c_int
    L.bridge_identical.argtypes = [C.POINTER(abi.GraphDesc), C.c_int, C.c_int, C.c_uint64, C.c_int]
    L.bridge_last_error.restype = C.c_char_p
    return L


def test_bridge_links_and_exports():
    L = bridge()
    assert hasattr(L, "bridge_identical")
    assert hasattr(L, "_ZN7macosim7gpu_runERKNS_9SimConfigERKNS_13DistanceTableEi")


@pytest.mark.gpu
@pytest.mark.parametrize("alg", [0, 1, 2, 3])
def test_gpu_run_identical_to_reference_run(alg):
    L = bridge()
    for net, V in ((networks.grid(10, 10), 100), (networks.grid(32, 32, signals="all"), 1000)):
        for seed in (1, 2):
            rc = L.bridge_identical(C.byref(net.desc()), alg, V, seed, 0)
            assert rc == 1, (alg, seed, L.bridge_last_error())
