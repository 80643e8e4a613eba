"""Regenerates tests/golden/oracle_golden.json from the CPU oracle.

The hash entries restate PolyHash::from_seed / eval (hashing.cpp:8-16,
hashing.hpp:29-34); the first one is the corrected frozen KAT of
proj/tests/test_hashing.cpp:58-68. The small symmetric case is a regression
fixture for the oracle and a fixed-size parity fixture for the GPU path.
Run: python tests/golden/make_golden.py
"""
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracle_py as O  # noqa: E402


def main():
    out = {"hash": []}
    for k, b, seed in [(6, 1024, 42), (2, 16, 7), (6, 4, 5), (6, 2, 31), (2, 4096, 123456789)]:
        c = O.polyhash_from_seed(k, b, seed)
        out["hash"].append({"k": k, "b": b, "seed": seed, "coeffs": [int(x) for x in c],
                            "eval": [int(x) for x in O.polyhash_eval(c, b, np.arange(16))]})
    n, b, B, seed = 5, 16, 3, 2024
    rng = np.random.default_rng(2024)
    A = np.round(rng.normal(size=(n, n, n)), 3)
    T = sum(A.transpose(p) for p in [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)])
    u = np.round(rng.normal(size=n), 3)
    s = O.SymSet(n, b, B, seed)
    s.accumulate_dense(T)
    d = s.data()
    out["sym_small"] = {"n": n, "b": b, "B": B, "seed": seed, "T": T.reshape(-1).tolist(), "u": u.tolist(),
                        "data_re": d.real.reshape(-1).tolist(), "data_im": d.imag.reshape(-1).tolist(),
                        "ivv": s.ivv(u).tolist(), "vvv": s.vvv(u)}
    (HERE / "oracle_golden.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
