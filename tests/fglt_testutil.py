"""Test-side graph fixtures mirroring the reference's generators
(proj/tests/testutil.hpp:64-193): path, cycle, star, complete, er, tree,
regular, permutation. Built through the package's CSR sanitiser."""
import numpy as np

from paper_2007_11111_b200 import graphs

DEMO_EDGES = [(5, 3), (3, 4), (4, 0), (0, 1), (1, 4), (1, 2), (2, 3), (2, 4), (1, 3)]

# Fig. 2 golden tables (proj/tests/testutil.hpp:40-62)
DEMO_RAW = np.array([
    [1, 2, 6, 1, 1, 14, 4, 6, 0, 6, 4, 0, 2, 2, 0, 0],
    [1, 4, 9, 6, 4, 12, 19, 7, 4, 3, 12, 8, 5, 3, 5, 1],
    [1, 3, 9, 3, 3, 14, 12, 9, 1, 5, 12, 3, 4, 4, 3, 1],
    [1, 4, 8, 6, 3, 12, 18, 7, 4, 5, 10, 6, 4, 4, 3, 1],
    [1, 4, 9, 6, 4, 12, 19, 7, 4, 3, 12, 8, 5, 3, 5, 1],
    [1, 1, 3, 0, 0, 8, 0, 3, 0, 3, 0, 0, 0, 0, 0, 0],
], dtype=np.uint64)
DEMO_NET = np.array([
    [1, 2, 4, 0, 1, 2, 0, 0, 0, 2, 0, 0, 0, 2, 0, 0],
    [1, 4, 1, 2, 4, 0, 1, 0, 0, 0, 2, 1, 0, 0, 2, 1],
    [1, 3, 3, 0, 3, 0, 0, 0, 0, 0, 4, 0, 0, 1, 0, 1],
    [1, 4, 2, 3, 3, 0, 2, 0, 0, 0, 2, 3, 0, 1, 0, 1],
    [1, 4, 1, 2, 4, 0, 1, 0, 0, 0, 2, 1, 0, 0, 2, 1],
    [1, 1, 3, 0, 0, 2, 0, 0, 0, 3, 0, 0, 0, 0, 0, 0],
], dtype=np.uint64)


def from_pairs(pairs, n=0):
    if len(pairs) == 0:
        return graphs.csr_from_pairs(np.zeros(0, np.int64), np.zeros(0, np.int64), n)[:2]
    a = np.asarray(pairs, dtype=np.int64)
    return graphs.csr_from_pairs(a[:, 0], a[:, 1], n)[:2]


def demo():
    return from_pairs(DEMO_EDGES)


def path(n):
    return from_pairs([(v, v + 1) for v in range(n - 1)], n)


def cycle(n):
    return from_pairs([(v, (v + 1) % n) for v in range(n)], n)


def star(leaves):
    return from_pairs([(0, v) for v in range(1, leaves + 1)], leaves + 1)


def complete(n):
    return from_pairs([(u, v) for u in range(n) for v in range(u + 1, n)], n)


def tree(n, seed):
    rng = np.random.default_rng(seed)
    return from_pairs([(int(rng.integers(0, v)), v) for v in range(1, n)], n)


def er(n, p, seed):
    return graphs.er(n, p, seed)


def regular(n, d, seed):
    """Random d-regular-ish simple graph by a seeded configuration pairing
    (repeats and loops dropped — a fixture, not an exact regular sampler)."""
    rng = np.random.default_rng(seed)
    stubs = np.repeat(np.arange(n), d)
    rng.shuffle(stubs)
    pairs = stubs[: len(stubs) // 2 * 2].reshape(-1, 2)
    return from_pairs([tuple(p) for p in pairs], n)


def permute(rp, ci, pi):
    n = len(rp) - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    keep = ci > rows
    return graphs.csr_from_pairs(pi[rows[keep]], pi[ci[keep]], n)[:2]
