"""Pins of the consumer-step oracle (sage_mean_layer, NEXT-4 i; -m "not gpu").

  dense form   -> z = X_dst W_self^T + (D^-1 A) X_src W_neigh^T with the block's dense
                  adjacency A (multiplicity counted) and D = diag(in-degree): a numpy
                  matmul, not the oracle's per-vertex loop
  closed forms -> constant features: z[v] = (W_self + W_neigh) 1 * c for deg > 0 and
                  W_self 1 * c for deg 0; no self term + deg 0 -> 0
  invariance   -> permuting a dst's neighbour list does not change z
"""
import numpy as np

import oracle


def _block(rng, n_dst, n_src, max_deg):
    deg = rng.integers(0, max_deg + 1, n_dst)
    indptr = np.concatenate([[0], np.cumsum(deg)])
    indices = rng.integers(0, n_src, indptr[-1])
    return indptr, indices


def test_sage_matches_dense_matrix_form():
    rng = np.random.default_rng(1)
    n_dst, n_src, F, H = 37, 80, 12, 9
    indptr, indices = _block(rng, n_dst, n_src, 7)
    xs = rng.standard_normal((n_src, F))
    xd = xs[:n_dst]                                     # dst-in-src prefix
    w = rng.standard_normal((H, 2 * F))
    z = oracle.sage_mean_layer(indptr, indices, xs, xd, w)
    A = np.zeros((n_dst, n_src))
    for v in range(n_dst):
        for u in indices[indptr[v]:indptr[v + 1]]:
            A[v, u] += 1.0
    deg = A.sum(axis=1, keepdims=True)
    M = np.divide(A, deg, out=np.zeros_like(A), where=deg > 0) @ xs
    want = xd @ w[:, :F].T + M @ w[:, F:].T
    np.testing.assert_allclose(z, want, rtol=1e-12, atol=1e-12)
    z2 = oracle.sage_mean_layer(indptr, indices, xs, None, w[:, F:])   # no self term
    np.testing.assert_allclose(z2, M @ w[:, F:].T, rtol=1e-12, atol=1e-12)


def test_sage_closed_forms():
    n_dst, n_src, F, H, c = 5, 9, 4, 3, 2.5
    indptr = np.array([0, 0, 3, 4, 4, 6])              # dsts 0 and 3 have no in-edge
    indices = np.array([1, 2, 2, 8, 0, 0])
    xs = np.full((n_src, F), c)
    w = np.arange(H * 2 * F, dtype=np.float64).reshape(H, 2 * F) / 7
    z = oracle.sage_mean_layer(indptr, indices, xs, xs[:n_dst], w)
    ws, wn = w[:, :F].sum(axis=1) * c, w[:, F:].sum(axis=1) * c
    for v in range(n_dst):
        want = ws + (wn if indptr[v + 1] > indptr[v] else 0)
        np.testing.assert_allclose(z[v], want, rtol=1e-13)
    z0 = oracle.sage_mean_layer(indptr, indices, xs, None, w[:, F:])
    assert np.all(z0[0] == 0) and np.all(z0[3] == 0)


def test_sage_neighbour_order_invariance():
    rng = np.random.default_rng(3)
    indptr, indices = _block(rng, 20, 30, 6)
    xs = rng.standard_normal((30, 8))
    w = rng.standard_normal((5, 16))
    z = oracle.sage_mean_layer(indptr, indices, xs, xs[:20], w)
    perm = indices.copy()
    for v in range(20):
        seg = perm[indptr[v]:indptr[v + 1]]
        perm[indptr[v]:indptr[v + 1]] = seg[rng.permutation(len(seg))]
    np.testing.assert_allclose(oracle.sage_mean_layer(indptr, perm, xs, xs[:20], w), z, rtol=1e-12, atol=1e-12)
