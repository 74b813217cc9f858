"""Pins of the oracle's block store (hash, CSR bucket table, neighbour table) — SURVEY §8(c) 'Hash' and
'CSR / neighbour tables' rows.  CPU only."""
import os

import numpy as np
import pytest

import oracle
from synth import rng, random_instance, tiny
import torch

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_hash():
    rows = []
    for line in open(os.path.join(GOLD, "hash_values.txt")):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(tuple(int(t) for t in line.split()))
    return rows


@pytest.mark.parametrize("x,y,z,T,h", _golden_hash())
def test_hash_hand_values(x, y, z, T, h):
    # tests/golden/hash_values.txt: hand evaluation of S:56's hash (uint32 wrap, reading c-14)
    assert oracle.block_hash(x, y, z, T) == h


def test_hash_python_definition_random():
    # the hash is the written formula evaluated with Python integers mod 2^32 (independent of the C code)
    g = np.random.default_rng(0)
    for _ in range(2000):
        x, y, z = (int(v) for v in g.integers(-2**20, 2**20, 3))
        T = 1 << int(g.integers(0, 24))
        ref = (((x & 0xFFFFFFFF) * 73856093) ^ ((y & 0xFFFFFFFF) * 19349669) ^ ((z & 0xFFFFFFFF) * 83492791)) & 0xFFFFFFFF
        assert oracle.block_hash(x, y, z, T) == ref % T


def test_table_size_rule():
    for n, T in [(0, 1), (1, 2), (2, 4), (3, 8), (4, 8), (5, 16), (224, 512), (1000, 2048)]:
        assert oracle.table_size(n) == T


def test_insert_lookup_10k_random():
    # 10,000 random block coordinates in [−2^20, 2^20)^3, insert then lookup
    g = np.random.default_rng(1)
    c = g.integers(-2**20, 2**20, size=(10000, 3)).astype(np.int32)
    c = np.unique(c, axis=0)
    g.shuffle(c)
    tables = oracle.build_table(c)
    assert tables[3] is None
    for i in range(0, c.shape[0], 7):
        assert oracle.lookup(c, tables, *c[i]) == i
    # absent coordinates report −1
    for _ in range(200):
        q = g.integers(2**20, 2**21, 3)
        assert oracle.lookup(c, tables, *q) == -1


def test_csr_layout_invariants():
    s = random_instance(300, seed=3, extent=5)
    c = s.coords.numpy()
    T, bs, be, dup = oracle.build_table(c)
    assert dup is None and T == 1024
    assert bs[0] == 0 and bs[-1] == c.shape[0] and np.all(np.diff(bs.astype(np.int64)) >= 0)
    assert sorted(be.tolist()) == list(range(c.shape[0]))
    for b in range(T):
        ent = be[bs[b]:bs[b + 1]]
        assert np.all(np.diff(ent) > 0), "entries of a bucket are in caller order"
        for i in ent:
            assert oracle.block_hash(*c[i], T) == b


def test_duplicates_reported():
    c = np.array([[0, 0, 0], [1, 2, 3], [5, 5, 5], [1, 2, 3], [0, 0, 0]], np.int32)
    _, _, _, dup = oracle.build_table(c)
    assert dup == (0, 4) or dup == (1, 3)
    assert dup == (1, 3), "first repeated block in caller order"


def _brute_neighbours(c):
    D = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    n = c.shape[0]
    out = np.full((n, 6), -1, np.int32)
    for i in range(n):
        for d, dv in enumerate(D):
            q = c[i] + np.array(dv)
            hit = np.nonzero(np.all(c == q, axis=1))[0]
            if hit.size:
                out[i, d] = hit[0]
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_neighbours_match_brute_force(seed):
    s = random_instance(400 + 300 * seed, seed=seed, extent=6)
    c = s.coords.numpy()
    assert np.array_equal(oracle.neighbours(c), _brute_neighbours(c))


def test_neighbours_translation_invariant():
    s = random_instance(500, seed=5, extent=5)
    c = s.coords.numpy()
    nb = oracle.neighbours(c)
    for off in ([1000, -7, 3], [-2**19, 2**19, -12345]):
        assert np.array_equal(oracle.neighbours(c + np.array(off, np.int32)), nb)


def test_tiny_config_block_count():
    # 224 blocks / 114,688 voxels for the sphere centred at the origin
    s = tiny()
    assert s.n_blocks == 224 and s.n_alloc == 114688


def test_splitmix_matches_python_reference():
    xs = [0, 1, 2, 12345, 2**40 + 17, 2**62 + 3]
    got = rng.splitmix64(torch.tensor(xs, dtype=torch.int64))
    for x, gv in zip(xs, got.tolist()):
        assert gv & ((1 << 64) - 1) == rng.splitmix64_py(x)
