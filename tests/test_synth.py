"""The seeded generators are reproducible, index-addressable and have the stated shapes."""
import numpy as np

import synth


def test_uniform_reproducible_and_offsettable():
    a = synth.uniform_symbols(10000, 26, seed=3)
    b = synth.uniform_symbols(10000, 26, seed=3)
    assert np.array_equal(a, b)
    c = synth.uniform_symbols(5000, 26, seed=3, offset=5000)
    assert np.array_equal(a[5000:], c)
    assert a.max() < 26 and len(np.unique(a)) == 26
    # roughly uniform
    h = np.bincount(a, minlength=26)
    assert h.min() > 300


def test_tables_in_range():
    t = synth.random_dfa(256, 26, 1)
    assert t.shape == (256, 26) and t.max() < 256
    s = synth.sparse_dfa(64, 256, 4, 4)
    assert all(len(np.unique(s[q])) <= 4 for q in range(64))
    p = synth.partial_dfa(20, 4, 0.2, 9)
    assert (p == 0xFFFF).any() and (p[p != 0xFFFF] < 20).all()


def test_markov_block_restart_and_skew():
    x = synth.markov_bytes(3 << 20, 5)
    y = synth.markov_bytes(1 << 20, 5)
    assert np.array_equal(x[: 1 << 20], y)
    # skewed order-1 conditionals: the top next-symbol has ~21% probability in every row
    j = np.zeros((256, 256))
    np.add.at(j, (x[:-1], x[1:]), 1)
    top = j.max(axis=1) / j.sum(axis=1)
    assert 0.17 < top.mean() < 0.25


def test_configs_shapes():
    for k, (Q, A) in {1: (4, 2), 2: (13, 4), 3: (256, 26), 4: (4096, 256), 5: (1024, 256)}.items():
        c = synth.config(k, n=4096)
        assert (c.Q, c.A) == (Q, A) and c.accept.size == Q
        x = c.make_input()
        assert x.size == 4096 and int(x.max()) < A
