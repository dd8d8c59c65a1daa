"""On-disk formats: the reference text format (matrix_core.py:242-310) and .npy."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_text_and_npy_roundtrip(tmp_path):
    import paper_2008_11480_b200 as P

    rng = np.random.default_rng(3)
    a = rng.standard_normal((7, 7))
    v = rng.standard_normal(7)
    for ext in (".txt", ".npy"):
        P.save_matrix(tmp_path / f"a{ext}", a, comment="fixture\nsecond line")
        P.save_vector(tmp_path / f"v{ext}", v)
        ta = P.load_matrix(tmp_path / f"a{ext}")
        tv = P.load_vector(tmp_path / f"v{ext}")
        assert ta.is_cuda and torch.equal(ta.cpu(), torch.as_tensor(a))  # 17 digits round-trip
        assert torch.equal(tv.cpu(), torch.as_tensor(v))


def test_text_format_errors(tmp_path):
    import paper_2008_11480_b200 as P

    (tmp_path / "bad.txt").write_text("3\n1 2 3\n4 5 6\n")
    with pytest.raises(ValueError):
        P.load_matrix(tmp_path / "bad.txt")
    (tmp_path / "empty.txt").write_text("# only a comment\n")
    with pytest.raises(ValueError):
        P.load_matrix(tmp_path / "empty.txt")
    (tmp_path / "nan.txt").write_text("1\nnan\n")
    with pytest.raises(ValueError):
        P.load_matrix(tmp_path / "nan.txt")
