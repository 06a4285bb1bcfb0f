"""extend / extract_block (extend.hpp:22-60) in the Python mirror (host data
movement, no device work): shapes, dummy marginals, penalty check,
block split."""
import numpy as np
import pytest

from oracle import binding
from paper_2601_17196_b200 import pot


def test_extend_and_extract_block():
    r, c, C, s = binding.random_instance(3, 6)
    inst = pot.Instance(r=r, c=c, s=s, C=C)
    ext = pot.extend(inst, 5.0)
    assert ext.C_ext.shape == (7, 7) and ext.original_size() == 6
    assert np.array_equal(ext.C_ext[:6, :6], C) and ext.C_ext[6, 6] == 5.0
    assert ext.C_ext[:6, 6].sum() == 0 and ext.C_ext[6, :6].sum() == 0
    assert ext.r_ext[6] == max(c.sum() - s, 0.0) and ext.c_ext[6] == max(r.sum() - s, 0.0)
    with pytest.raises(pot.PotError) as e:
        pot.extend(inst, C.max())
    assert e.value.code == pot.ErrorCode.PenaltyTooSmall
    X = np.arange(49.0).reshape(7, 7)
    b = pot.extract_block(X)
    assert np.array_equal(b.block, X[:6, :6]) and np.array_equal(b.dummy_col, X[:6, 6])
    assert np.array_equal(b.dummy_row, X[6, :6]) and b.corner == 48.0
    with pytest.raises(pot.PotError):
        pot.extract_block(np.zeros((1, 1)))
