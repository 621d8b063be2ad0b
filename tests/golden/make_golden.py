"""Generate golden PLUQ fixtures by running the REAL reference package.

Run in the build container (the only place `/root/reference` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `pluq` from /root/reference/pkg/src (read-only; bytecode writing is
disabled so nothing lands in the reference tree), decomposes a fixed, seeded
case list with `pluq.pluq(a, threshold=t)` and `pluq.pluq_iterative(a)`, and
writes `tests/golden/golden.npz` + `tests/golden/manifest.json`:
inputs, P.sigma, Q.sigma, rank, OpCounts and the packed output (or its SHA-256
for the few larger cases).  The fixtures pin both the oracle
(tests/test_oracle_golden.py, CPU) and the CUDA path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import pluq as ref  # noqa: E402  (the reference package)

from oracle.pluq_oracle import gen_cfg4, gen_xy_rank  # noqa: E402  (input generators only)

BIG = 64 * 64  # packed outputs larger than this are stored as sha256


def sha(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr.astype(np.int64)).tobytes()).hexdigest()


def run_case(arr: np.ndarray, p: int, route: str, threshold: int):
    field = ref.PrimeField(p)
    a = ref.DenseMatrix(field, arr.copy())
    counts = ref.OpCounts()
    if route == "iterative":
        f = ref.pluq_iterative(a, counts)
    else:
        f = ref.pluq(a, threshold=threshold, counts=counts)
    return f, counts


def cases():
    out = []
    # --- known-answer tests from the reference suite -------------------------------
    kat = [
        ([[0, 0, 0], [0, 0, 0]], 5, 30),            # test_recursive.py:25-30
        (np.eye(6, dtype=np.int64).tolist(), 7, 1),   # test_recursive.py:33-39
        ([[0, 0], [1, 0]], 2, 1),                     # test_recursive.py:42-47
        ([[0, 0, 5]], 7, 30),                         # test_recursive.py:65-74
        ([[0], [2], [4]], 5, 30),                     # test_recursive.py:77-87
        ([[0, 1], [1, 0]], 2, 30),                    # test_iterative.py:28-33
        ([[0, 0, 0], [0, 0, 1], [0, 1, 0]], 2, 1),    # test_iterative.py:36-46
        ([[0, 0, 3], [0, 2, 1], [0, 0, 5]], 1009, 30),  # README.md:132-141
    ]
    for rows, p, t in kat:
        out.append(("kat", np.array(rows, dtype=np.int64), p, t))
    # --- seeded random small cases over several fields / thresholds -------------------
    rng = np.random.default_rng(20261019)
    primes = [2, 3, 5, 101, 1009, 65521, 8388593]
    for idx in range(260):
        p = int(rng.choice(primes))
        m = int(rng.integers(0, 48))
        n = int(rng.integers(0, 48))
        t = int(rng.choice([1, 2, 3, 4, 8, 30]))
        kind = idx % 4
        if kind == 0 or m == 0 or n == 0:
            a = rng.integers(0, p, (m, n), dtype=np.int64)
        else:
            r = [0, 1, min(m, n) // 2, min(m, n)][int(rng.integers(0, 4))]
            a = ref.gen_rank_deficient_rect(m, n, r, p, int(rng.integers(0, 2**62))).data.astype(np.int64)
        out.append(("rand", a, p, t))
    # --- sparse / structured (many zero blocks, skinny base cases) ---------------------
    for idx in range(40):
        p = int(rng.choice([3, 101, 65521]))
        m = int(rng.integers(1, 90))
        n = int(rng.integers(1, 90))
        dens = float(rng.choice([0.02, 0.1, 0.3]))
        a = rng.integers(1, p, (m, n), dtype=np.int64) * (rng.random((m, n)) < dens)
        out.append(("sparse", a.astype(np.int64), p, int(rng.choice([1, 4, 30]))))
    # --- medium cases at threshold 30 (shapes of the BASELINE configs, scaled) -------
    out.append(("cfg1_s", gen_xy_rank(128, 128, 96, 65521, 1), 65521, 30))
    out.append(("cfg5_s", gen_xy_rank(256, 256, 128, 65521, 5), 65521, 30))
    a4, _, _ = gen_cfg4(seed=4, m=128, n=256, r=64, p=8388593)
    out.append(("cfg4_s", a4, 8388593, 30))
    a4b, _, _ = gen_cfg4(seed=7, m=256, n=512, r=128, p=8388593)
    out.append(("cfg4_m", a4b, 8388593, 30))
    g = np.random.default_rng(2)
    for b in range(8):
        out.append(("cfg2_s", g.integers(0, 65521, (64, 64), dtype=np.int64), 65521, 30))
    out.append(("cfg3_s", np.random.default_rng(3).integers(0, 65521, (256, 256), dtype=np.int64), 65521, 30))
    out.append(("rect_wide", np.random.default_rng(9).integers(0, 1009, (40, 300), dtype=np.int64), 1009, 30))
    out.append(("rect_tall", np.random.default_rng(10).integers(0, 1009, (300, 40), dtype=np.int64), 1009, 30))
    out.append(("cfg1", gen_xy_rank(512, 512, 384, 65521, 0), 65521, 30))
    return out


def main():
    store = {}
    manifest = []
    for idx, (tag, a, p, t) in enumerate(cases()):
        for route in ("recursive", "iterative"):
            if route == "iterative" and a.size > 128 * 128:
                continue
            f, c = run_case(a, p, route, t)
            key = f"c{idx}_{route[0]}"
            packed = np.asarray(f.packed.data, dtype=np.int64)
            entry = {
                "key": key,
                "tag": tag,
                "route": route,
                "p": p,
                "threshold": t,
                "m": int(a.shape[0]),
                "n": int(a.shape[1]),
                "rank": int(f.rank),
                "counts": [c.field_mul, c.field_add, c.field_inv, c.modular_reductions],
                "packed_sha256": sha(packed),
                "input_sha256": sha(a),
                "has_packed": bool(a.size <= BIG),
            }
            manifest.append(entry)
            store[key + "_in"] = a.astype(np.int64)
            store[key + "_P"] = f.p_perm.sigma.astype(np.int64)
            store[key + "_Q"] = f.q_perm.sigma.astype(np.int64)
            if entry["has_packed"]:
                store[key + "_out"] = packed
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **store)
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "pluq " + ref.__version__,
                   "cases": manifest}, fh, indent=0)
    print(f"wrote {len(manifest)} golden decompositions")


if __name__ == "__main__":
    main()
