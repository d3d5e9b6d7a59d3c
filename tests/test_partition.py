"""Host-side partition logic (reference partition.py:52-141 semantics).

Mirrors the cases of the reference's own test_partition.py: sizing, overlap
rounding, remainder handling, coverage, complements, validation errors and
JSON loading; plus the device-facing range / relabelling helpers.
"""

import json

import numpy as np
import pytest

from paper_2502_06377_b200 import (
    DuplicateWithinSet,
    IndexOutOfRange,
    InvalidOverlap,
    Partition,
    TooManyBlocks,
    UncoveredIndices,
    complement,
    contiguous_partition,
    load_partition_json,
    overlap_depth,
    red_black_partition,
    validate,
)
from paper_2502_06377_b200.partition import block_permutation, contiguous_ranges


def test_two_even_blocks():
    part = contiguous_partition(8, 2, 0.0)
    assert [list(s) for s in part.sets] == [[0, 1, 2, 3], [4, 5, 6, 7]]


def test_quarter_overlap():
    part = contiguous_partition(8, 2, 0.25)
    assert list(part.sets[0]) == list(range(5))
    assert list(part.sets[1]) == list(range(3, 8))


def test_remainder_to_last():
    part = contiguous_partition(10, 3, 0.0)
    assert [len(s) for s in part.sets] == [3, 3, 4]


@pytest.mark.parametrize("k", [2, 3, 5])
def test_overlap_sizes(k):
    m, f = 20, 0.2
    part = contiguous_partition(k * m, k, f)
    h = overlap_depth(m, f)
    sizes = [len(s) for s in part.sets]
    assert h == 4 and sizes[0] == sizes[-1] == m + h
    assert all(s == m + 2 * h for s in sizes[1:-1])


@pytest.mark.parametrize("p,k,f", [(64, 4, 0.0), (100, 3, 0.1), (37, 5, 0.3), (4096, 6, 0.2), (16384, 8, 0.125)])
def test_coverage(p, k, f):
    part = contiguous_partition(p, k, f)
    validate(part)
    assert np.array_equal(np.unique(np.concatenate(part.sets)), np.arange(p))


def test_baseline_partitions():
    """c3 sets 1152/1280 overlap 256; c4 2304/2560; c5 4608/5120."""
    for p, k, edge, inner in [(8192, 8, 1152, 1280), (16384, 8, 2304, 2560), (65536, 16, 4608, 5120)]:
        sizes = [len(s) for s in contiguous_partition(p, k, 0.125).sets]
        assert sizes[0] == sizes[-1] == edge and set(sizes[1:-1]) == {inner}


def test_errors():
    with pytest.raises(ValueError):
        contiguous_partition(10, 1)
    with pytest.raises(TooManyBlocks):
        contiguous_partition(7, 4)
    with pytest.raises(InvalidOverlap):
        contiguous_partition(100, 2, 0.5)
    with pytest.raises(InvalidOverlap):
        contiguous_partition(100, 2, -0.1)


def test_overlap_depth_half_up():
    assert overlap_depth(10, 0.05) == 1
    assert overlap_depth(10, 0.04) == 0
    assert overlap_depth(4, 0.25) == 1


def test_complement_and_red_black():
    part = contiguous_partition(10, 2, 0.2)
    assert list(complement(part, 0)) == [6, 7, 8, 9]
    rb = red_black_partition(9)
    assert list(rb.sets[0]) == [0, 2, 4, 6, 8] and list(rb.sets[1]) == [1, 3, 5, 7]
    with pytest.raises(ValueError):
        red_black_partition(3)


def test_validate_errors():
    with pytest.raises(ValueError):
        validate(Partition(p=4, sets=[np.arange(4)]))
    with pytest.raises(IndexOutOfRange):
        validate(Partition(p=4, sets=[np.array([0, 1]), np.array([2, 4])], ordering="custom"))
    with pytest.raises(DuplicateWithinSet):
        validate(Partition(p=4, sets=[np.array([0, 0, 1]), np.array([2, 3])], ordering="custom"))
    with pytest.raises(UncoveredIndices) as ei:
        validate(Partition(p=5, sets=[np.array([0, 1]), np.array([3])], ordering="custom"))
    assert ei.value.indices == [2, 4]
    with pytest.raises(ValueError):
        validate(Partition(p=4, sets=[np.array([0, 2]), np.array([1, 3])]))   # contiguous ordering violated


def test_load_json(tmp_path):
    payload = {"p": 6, "sets": [[0, 1, 2, 3], [2, 3, 4, 5]]}
    part = load_partition_json(payload)
    assert part.k == 2 and part.ordering == "custom"
    assert load_partition_json(json.dumps(payload)).p == 6
    f = tmp_path / "part.json"
    f.write_text(json.dumps(payload))
    assert load_partition_json(str(f)).k == 2
    with pytest.raises(UncoveredIndices):
        load_partition_json({"p": 6, "sets": [[0, 1], [2, 3]]})


def test_ranges_and_relabelling():
    assert contiguous_ranges(contiguous_partition(20, 4, 0.1)) == [(0, 6), (4, 11), (9, 16), (14, 20)]
    rb = red_black_partition(8)
    assert contiguous_ranges(rb) is None
    perm, ranges = block_permutation(rb)
    assert list(perm) == [0, 2, 4, 6, 1, 3, 5, 7] and ranges == [(0, 4), (4, 8)]
    overl = load_partition_json({"p": 6, "sets": [[0, 2, 4], [1, 2, 3, 5]]})
    assert block_permutation(overl) is None
