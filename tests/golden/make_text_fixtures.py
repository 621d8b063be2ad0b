"""Text-format fixtures written by the REAL reference (matrix.py:128-158, 351-375), so the
CPU tests can check that formats.py reads and writes byte-identical files.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_text_fixtures.py
"""
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import pluq  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))
cases = []
for seed, (m, n, p) in enumerate([(4, 5, 7), (6, 3, 101), (1, 8, 65521), (5, 5, 8388593), (0, 3, 5), (3, 0, 5)]):
    rng = np.random.default_rng(seed)
    field = pluq.PrimeField(p)
    a = pluq.DenseMatrix(field, rng.integers(0, p, (m, n)) * (rng.random((m, n)) < 0.7))
    mtext = a.to_text()
    f = pluq.pluq(pluq.DenseMatrix(field, a.data.copy()))
    ftext = f.to_text()
    try:  # the reference cannot read back every file it writes (n = 0 factor files)
        pluq.PluqFactors.from_text(ftext)
        readable = True
    except ValueError:
        readable = False
    cases.append({"m": m, "n": n, "p": p, "matrix_text": mtext, "factors_text": ftext,
                  "rank": f.rank, "factors_readable": readable})
with open(os.path.join(HERE, "text_fixtures.json"), "w") as fh:
    json.dump(cases, fh, indent=1)
print(len(cases), "cases")
