"""Host-side layout detection of the Python binding (no GPU): which dense
cost layouts reach the C-ABI without a copy, and with which leading
dimension / order (potgpu.h: element (i, j) at C[i*ldc + j] if row_major,
else C[i + j*ldc])."""
import numpy as np

from paper_2601_17196_b200.pot import _dense_layout


def element(buf_base, C, ldc, row_major, i, j):
    off = (C.ctypes.data - buf_base.ctypes.data) // 8
    flat = buf_base.reshape(-1, order="A" if buf_base.flags.f_contiguous else "C")
    k = off + (i * ldc + j if row_major else i + j * ldc)
    return flat[k]


def test_layouts_without_copy():
    n = 7
    A = np.arange(n * n, dtype=np.float64).reshape(n, n)
    C, ldc, rm = _dense_layout(A, n)
    assert C is A and (ldc, rm) == (n, 1)
    F = np.asfortranarray(A)
    C, ldc, rm = _dense_layout(F, n)
    assert C is F and (ldc, rm) == (n, 0)
    wide = np.zeros((n, n + 5))
    wide[:, :n] = A
    V = wide[:, :n]
    C, ldc, rm = _dense_layout(V, n)
    assert C is V and (ldc, rm) == (n + 5, 1)
    for i, j in ((0, 0), (3, 5), (n - 1, n - 1)):
        assert element(wide, C, ldc, rm, i, j) == A[i, j]
    tall = np.asfortranarray(np.zeros((n + 3, n)))
    tall[:n, :] = A
    T = tall[:n, :]
    C, ldc, rm = _dense_layout(T, n)
    assert C is T and (ldc, rm) == (n + 3, 0)
    for i, j in ((0, 0), (3, 5), (n - 1, n - 1)):
        assert element(tall, C, ldc, rm, i, j) == A[i, j]


def test_other_layouts_are_copied():
    n = 6
    A = np.arange(2 * n * 2 * n, dtype=np.float64).reshape(2 * n, 2 * n)
    S = A[::2, ::2]  # neither stride is one element
    C, ldc, rm = _dense_layout(S, n)
    assert C is not S and C.flags.c_contiguous and (ldc, rm) == (n, 1)
    assert np.array_equal(C, S)
    I = np.arange(n * n, dtype=np.int64).reshape(n, n)
    C, ldc, rm = _dense_layout(I, n)
    assert C.dtype == np.float64 and np.array_equal(C, I)
