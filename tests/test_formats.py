"""Text formats (formats.py) against files written by the reference itself
(tests/golden/text_fixtures.json, made by tests/golden/make_text_fixtures.py)."""

import json
import os

import numpy as np
import pytest

from paper_1301_4438_b200.formats import factors_from_text, matrix_from_text

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def fixtures():
    with open(os.path.join(HERE, "golden", "text_fixtures.json")) as fh:
        return json.load(fh)


def test_matrix_and_factor_files_roundtrip_byte_identical(fixtures):
    for c in fixtures:
        a = matrix_from_text(c["matrix_text"])
        assert a.shape == (c["m"], c["n"]) and a.p == c["p"]
        assert a.to_text() == c["matrix_text"]
        if not c["factors_readable"]:  # the reference raises on this file too
            with pytest.raises(ValueError):
                factors_from_text(c["factors_text"])
            continue
        f = factors_from_text(c["factors_text"])
        assert f.rank == c["rank"]
        assert f.to_text() == c["factors_text"]


@pytest.mark.parametrize("text", ["", "2 2\n1 2\n3 4\n", "2 2 7\n1 2\n", "2 2 7\n1 2\n3\n", "2 2 7\n1 2\n3 4\n5 6\n",
                                  "2 2 7\n1 2\n3 7\n", "-1 2 7\n", "2 2 8\n1 2\n3 4\n"])
def test_matrix_parse_errors(text):
    with pytest.raises(ValueError):
        matrix_from_text(text)


@pytest.mark.parametrize("text", ["2 2 7\n0 1\n", "2 2 7 1\n0 1\n0\n2 2 7\n1 0\n0 0\n", "2 2 7 3\n0 1\n0 1\n2 2 7\n1 0\n0 0\n",
                                  "2 2 7 1\n0 1\n0 1\n2 2 5\n1 0\n0 0\n"])
def test_factor_parse_errors(text):
    with pytest.raises(ValueError):
        factors_from_text(text)
