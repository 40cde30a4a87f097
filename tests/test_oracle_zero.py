"""Pins of oracle/zero.py, Alg. 1 (§2.3)."""
import itertools
import json
import os

import numpy as np

from oracle.zero import greedy_distribute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_traced_example():
    g = json.load(open(os.path.join(GOLD, "alg1_example.json")))
    owner, load, parts = greedy_distribute(g["sizes"], g["m"])
    assert owner == g["owner"] and load == g["load"]
    assert sorted(parts[0]) == [0, 3, 4] and sorted(parts[1]) == [1, 2]


def test_degenerate_cases():
    assert greedy_distribute([3, 1, 2], 1)[1] == [6]
    assert greedy_distribute([], 3) == ([], [0, 0, 0], [[], [], []])
    owner, load, _ = greedy_distribute([7], 2)
    assert owner == [0] and load == [7, 0]


def test_complete_exclusive_and_lpt_bound():
    rng = np.random.default_rng(21)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        m = int(rng.integers(1, 9))
        sizes = rng.integers(1, 10 ** 6, size=n).tolist()
        owner, load, parts = greedy_distribute(sizes, m)
        assert sorted(i for p in parts for i in p) == list(range(n))
        assert all(load[j] == sum(sizes[i] for i in parts[j]) for j in range(m))
        if n >= m:
            assert max(load) - min(load) <= max(sizes)     # greedy/LPT property


def test_within_4_3_of_optimal_bruteforce():
    """Graham's LPT bound max_load <= 4/3 OPT, OPT by exhaustive search."""
    rng = np.random.default_rng(22)
    for _ in range(60):
        n = int(rng.integers(1, 9))
        m = int(rng.integers(2, 4))
        sizes = rng.integers(1, 100, size=n).tolist()
        _, load, _ = greedy_distribute(sizes, m)
        opt = min(max(sum(s for s, a in zip(sizes, asg) if a == j) for j in range(m))
                  for asg in itertools.product(range(m), repeat=n))
        assert max(load) * 3 <= 4 * opt
