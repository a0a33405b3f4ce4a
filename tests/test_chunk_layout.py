"""CPU pin of the chunk-major index arithmetic (layout.cu k_chunk_transpose and the walk's
position formula in lpa_kernels.cuh k_thread / k_chunk_walk).

The layout maps position a + j of the range to bucket-order entry e(j) = k*L + r (column r,
row k); the walk computes the position of entry r of chunk k as a + r*q + min(r, rem) + k
for M = q*L + rem. The two must be inverse bijections of [0, M) for every (M, L), and a
chunk's consecutive entries must sit one column apart (coalesced across lanes).
"""
import numpy as np
import pytest


def walk_position(r, k, M, L):
    q, rem = divmod(M, L)
    return r * q + np.minimum(r, rem) + k


def transpose_entry(j, M, L):
    """k_chunk_transpose: position j of the range -> bucket-order entry."""
    q, rem = divmod(M, L)
    wide = rem * (q + 1)
    j = np.asarray(j, dtype=np.int64)
    r = np.where(j < wide, j // (q + 1), rem + (j - wide) // max(q, 1))
    k = np.where(j < wide, j % (q + 1), (j - wide) % max(q, 1))
    return k * L + r


@pytest.mark.parametrize("M,L", [(32, 32), (33, 32), (1000, 32), (65536, 32), (100003, 37),
                                 (16773120, 111), (262144, 32), (333000, 32), (77, 76)])
def test_walk_and_layout_are_inverse(M, L):
    e = np.arange(M, dtype=np.int64)
    k, r = e // L, e % L
    pos = walk_position(r, k, M, L)
    assert np.array_equal(np.sort(pos), e)  # a bijection onto [0, M)
    assert np.array_equal(transpose_entry(pos, M, L), e)  # the layout's inverse


@pytest.mark.parametrize("M,L", [(100003, 37), (262144, 32)])
def test_lanes_read_adjacent_positions(M, L):
    q, rem = divmod(M, L)
    for r in (0, L // 2, L - 1):
        k = np.arange(min(32, q))
        pos = walk_position(r, k, M, L)
        assert np.array_equal(np.diff(pos), np.ones(len(k) - 1, dtype=np.int64))
