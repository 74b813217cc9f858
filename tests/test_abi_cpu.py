"""CPU checks of the C-ABI library: it loads without a GPU, exports every symbol include/vol.h
declares, its host-only helpers agree with the oracle, the product path never touches oracle/, and
compute calls fail loudly without CUDA (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import oracle
from synth import random_instance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def native():
    from paper_1604_03734_b200 import build
    build.build()
    from paper_1604_03734_b200 import _native
    return _native


def declared_functions():
    src = open(os.path.join(ROOT, "include", "vol.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vol_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(native):
    lib = native.lib()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/vol.h but not exported"
    out = subprocess.check_output(["nm", "-D", "--defined-only", native.LIB_PATH]).decode()
    exported = set(re.findall(r" T (vol_\w+)", out))
    assert set(names) <= exported
    assert set(native.EXPORTS) <= exported


def test_library_targets_sm100a(native):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", native.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_block_hash_matches_oracle(native):
    from paper_1604_03734_b200 import block_hash
    g = np.random.default_rng(0)
    for _ in range(500):
        x, y, z = (int(v) for v in g.integers(-2**31, 2**31 - 1, 3))
        T = 1 << int(g.integers(0, 26))
        assert block_hash(x, y, z, T) == oracle.block_hash(x, y, z, T)


OFF12 = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1),
         (-1, 1, 0), (-1, 0, 1), (1, -1, 0), (0, -1, 1), (1, 0, -1), (0, 1, -1)]


def _brute_ghosts(c, part, rank):
    """Remote blocks among the 12 stencil neighbours (6 faces + 6 edges) of the rank's blocks."""
    idx = {tuple(v): i for i, v in enumerate(c.tolist())}
    out = set()
    for g in np.nonzero(part == rank)[0]:
        for o in OFF12:
            k = idx.get(tuple(np.add(c[g], o)), -1)
            if k >= 0 and part[k] != rank:
                out.add(k)
    return out


@pytest.mark.parametrize("world", [2, 3, 4])
def test_shard_plan_consistent(native, world):
    from paper_1604_03734_b200 import plan_shard
    s = random_instance(400, seed=world, extent=5)
    c = s.coords.numpy()
    part = (np.argsort(np.argsort(c[:, 0] * 100 + c[:, 1], kind="stable"), kind="stable") * world // len(c)).astype(np.int32)
    plans = [plan_shard(c, part, world, r) for r in range(world)]
    assert sum(p["n_local"] for p in plans) == len(c)
    for r, p in enumerate(plans):
        assert set(p["ghost"].tolist()) == _brute_ghosts(c, part, r)
        assert all(part[g] != r for g in p["ghost"])
        for q in range(world):
            assert p["peer_recv"][q] == plans[q]["peer_send"][r]
        # what r receives from q, in order, is exactly what q sends to r
        off = 0
        for q in range(world):
            k = int(p["peer_recv"][q])
            mine = p["ghost"][off:off + k]
            off += k
            qs = plans[q]
            so = int(sum(qs["peer_send"][:r]))
            assert np.array_equal(mine, qs["send"][so:so + int(qs["peer_send"][r])])


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1604_03734_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), fn
                assert "hvg_oracle" not in txt and "liboracle" not in txt, fn


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(native):
    from paper_1604_03734_b200 import Volume
    s = random_instance(4, seed=0, extent=1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        Volume(s.coords, s.f, s.W)
