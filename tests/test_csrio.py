"""CSR construction, row blocks and the text dump format (host side, no GPU).

Mirrors the reference's test_csr.py dump / triplet tests (test_csr.py:185-215):
the product's C++-built operators dump to the reference's golden text, and the
row-block helpers agree with the builder's own segment / half exports."""

from __future__ import annotations

import io
import os

import numpy as np
import pytest

import paper_2504_15814_b200 as th
from paper_2504_15814_b200.operators import HostOperator

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def lib():
    try:
        th._native.load()
    except Exception as e:  # pragma: no cover - build missing
        pytest.skip(f"native library not built: {e}")


def test_dump_golden_minimal_interpolation(lib):
    """matrix_linear interpolation at p = k = 1 dumps to GOLDEN_P1K1 byte for byte."""
    with open(os.path.join(GOLDEN, "golden_p1k1.txt")) as fh:
        want = fh.read()
    op = HostOperator("interpolate", "matrix_linear", 1, 1).csr()
    assert th.dumps_operator(op) == want


def test_dump_round_trip(lib):
    op = HostOperator("restrict", "matrix_linear", 2, 1).csr()
    text = th.dumps_operator(op)
    assert text.splitlines()[0].split() == [str(op.n_rows), str(op.n_cols), str(op.nnz), "matrix_linear", "2", "1"]
    loaded, p, k = th.load_operator(io.StringIO(text))
    assert (p, k) == (2, 1)
    assert loaded.arrays_equal(op)


@pytest.mark.parametrize("scheme", ("matrix_linear", "order2", "order3"))
def test_round_trip_is_bit_exact(lib, scheme):
    op = HostOperator("interpolate", scheme, 5, 3).csr(segment=4)
    loaded, _, _ = th.load_operator(io.StringIO(th.dumps_operator(op)))
    assert loaded.arrays_equal(op)  # %.17g round-trips every double


def test_dump_requires_fingerprint():
    with pytest.raises(th.ContractViolationError):
        th.dumps_operator(th.from_triplets(1, 1, [(0, 0, 1.0)]))


def test_load_rejects_bad_dumps():
    with pytest.raises(th.ContractViolationError):
        th.load_operator(io.StringIO("1 1 1 matrix_linear 1\n0 0 1.0\n"))
    with pytest.raises(th.ContractViolationError):
        th.load_operator(io.StringIO("1 1 2 matrix_linear 1 1\n0 0 1.0\n"))


def test_from_triplets_canonical():
    rng = np.random.default_rng(0)
    entries = [(int(r), int(c), float(v)) for r, c, v in zip(rng.integers(0, 4, 40), rng.integers(0, 6, 40),
                                                              rng.standard_normal(40))]
    entries += [(1, 2, 1e-15), (3, 5, 0.5), (3, 5, -0.5)]  # dropped: tiny, and cancelling duplicates
    a = th.from_triplets(4, 6, entries)
    b = th.from_triplets(4, 6, entries[::-1])
    assert a.arrays_equal(b)  # order invariant (duplicates summed in sorted-value order)
    dense = np.zeros((4, 6))
    for r, c, v in entries:
        dense[r, c] += v
    dense[np.abs(dense) < 1e-14] = 0.0
    assert np.allclose(a.to_dense(), dense, atol=1e-15)
    for r in range(4):
        cols = a.col_indices[a.row_offsets[r]:a.row_offsets[r + 1]]
        assert np.all(np.diff(cols) > 0)
    with pytest.raises(th.ContractViolationError):
        th.from_triplets(2, 2, [(2, 0, 1.0)])


@pytest.mark.parametrize("scheme", ("tensor_linear", "matrix_linear", "order2", "order3"))
def test_extract_matches_builder_blocks(lib, scheme):
    op = HostOperator("interpolate", scheme, 4, 3)
    full = op.csr()
    for seg in range(9):
        assert th.extract_segment(full, seg).arrays_equal(op.csr(segment=seg))
        assert th.extract_segment(full, seg).target_region == op.csr(segment=seg).target_region
    rop = HostOperator("restrict", scheme, 4, 3)
    rfull = rop.csr()
    for half in ("inner", "outer"):
        assert th.extract_half(rfull, half).arrays_equal(rop.csr(half=half))
    with pytest.raises(th.ContractViolationError):
        th.extract_half(full, "inner")
    with pytest.raises(th.ConfigurationError):
        th.extract_segment(full, 9)
