"""Row f1, generic Schur API: host logic (partition numbering, argument checks)."""
import numpy as np
import pytest

from paper_1108_4181_b200 import errors
from paper_1108_4181_b200.schur import INTERFACE_LABEL, partition_numbering


def test_partition_numbering():
    labels = np.array([1, -1, 0, 1, 0, -1, 2])
    perm, inv, slices = partition_numbering(labels)
    assert perm.tolist() == [2, 4, 0, 3, 6, 1, 5]
    assert np.array_equal(perm[inv], np.arange(7))
    assert slices[0] == slice(0, 2) and slices[1] == slice(2, 4) and slices[2] == slice(4, 5)
    assert slices[INTERFACE_LABEL] == slice(5, 7)


def test_partition_numbering_errors():
    with pytest.raises(errors.DimensionMismatch):
        partition_numbering([])
    with pytest.raises(errors.UnlabeledNode):
        partition_numbering([0, -2])
    with pytest.raises(errors.UnlabeledNode):
        partition_numbering([0.5, 1.0])
