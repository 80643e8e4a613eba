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


def rtpm_c0():
    """BASELINE config 0 in full (n=100, rank 10 + 0.01 noise, b=2^12, B=20, RTPM k=10,
    L=50, T=30) through the oracle: the full-size RTPM parity fixture (rtpm_c0.json).
    The tensor comes from the repository's host generator (bit-exact, no GPU)."""
    import os

    sys.path.insert(0, str(HERE.parents[1]))
    import paper_1506_04448_b200 as skb

    n, rank, b, B, k, L, T = 100, 10, 1 << 12, 20, 10, 50, 30
    Tt, lam, V = skb.gen_planted_tensor(n, rank, 0.01, 11)
    O.lib().orc_set_num_threads(os.cpu_count() or 1)
    o = O.SymSet(n, b, B, 5)
    o.accumulate_dense(Tt, True)
    lo, Vo, bto = o.rtpm(k, L, T, seed=3)
    (HERE / "rtpm_c0.json").write_text(json.dumps({
        "config": {"n": n, "rank": rank, "sigma": 0.01, "gen_seed": 11, "b": b, "B": B, "set_seed": 5, "k": k, "L": L,
                   "T": T, "rtpm_seed": 3},
        "lambda": lo.tolist(), "V": Vo.tolist(), "best_tau": [int(x) for x in bto]}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--rtpm-c0":
        rtpm_c0()
    else:
        main()
