"""Pins of the oracle's reading of the paper's parallel schedule (Sec. 4-5,
PAPER.md P:135-299), CPU only."""
import math

import numpy as np
import pytest

import fixtures
import oracle
from golden_util import read_golden


def test_table1_products():
    """Eq. (multi) against the numbers the paper prints in Table 1 (four
    processors, l = 2): Pfp, N Log2 N, and the ratio RSP to two decimals."""
    for row in read_golden("table1_parallel_products.txt"):
        N, N2, NL, pfp, rsp = row.split()
        N = int(N)
        m = int(round(math.log2(N)))
        assert int(N2) == N * N and int(NL) == N * m
        got = oracle.paper_parallel_products(m, 2)
        assert got == int(pfp)
        assert f"{N * m / got:.2f}" == rsp


def test_example_of_the_paper():
    """P:139-224's example: N = 8 data on 4 processors; processor 0's branch
    is C(0), C(4), processor 2's C(2), C(6) (the tree's leaf order), and the
    MASTER's result is the DFT with the paper's 1/N."""
    x = fixtures.complex_input(8, fixtures.UNIFORM, seed=31, dtype=np.complex128)
    assert np.array_equal(x[0::4], x[[0, 4]]) and np.array_equal(x[2::4], x[[2, 6]])
    ref = oracle.dft_bruteforce(x)
    assert oracle.rel_l2(oracle.paper_tree_fft(x, 4), ref) <= 1e-15


@pytest.mark.parametrize("P", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("m", [4, 10, 16])
def test_tree_equals_dft(P, m):
    """The schedule computes the paper's DFT (Eq. E2) for every processor
    count, against numpy's pocketfft (an independent library routine)."""
    n = 1 << m
    if n < P:
        pytest.skip("fewer data than processors")
    x = fixtures.complex_input(n, fixtures.NORMAL, seed=40 + m, dtype=np.complex128)
    ref = np.fft.fft(x) / n
    assert oracle.rel_l2(oracle.paper_tree_fft(x, P), ref) <= 1e-13
