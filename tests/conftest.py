import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


_cache = {}


@pytest.fixture(scope="session")
def tiny_scene():
    from synth import tiny
    if "tiny" not in _cache:
        _cache["tiny"] = tiny()
    return _cache["tiny"]


@pytest.fixture(scope="session")
def tiny_stress_scene():
    from synth import tiny
    if "tiny-stress" not in _cache:
        _cache["tiny-stress"] = tiny(stress=True)
    return _cache["tiny-stress"]


@pytest.fixture(scope="session")
def tiny_oracle(tiny_scene):
    import oracle
    if "tiny-oracle" not in _cache:
        nbr = oracle.neighbours(tiny_scene.coords)
        u64, ub64, p64 = oracle.regularise_scene(tiny_scene, precision="f64", nbr=nbr)
        u32, ub32, p32 = oracle.regularise_scene(tiny_scene, precision="f32", nbr=nbr)
        _cache["tiny-oracle"] = dict(nbr=nbr, u64=u64, p64=p64, u32=u32, p32=p32, ub32=ub32)
    return _cache["tiny-oracle"]
