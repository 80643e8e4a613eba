"""Small shapes through every hot kernel (class-list builds in lockstep, sums pre-pass,
half-length contraction, paired moment and LDA document kernels at local length 2048 with odd
and even item counts, a short RTPM), each checked against the oracle. The same script is the
target for compute-sanitizer runs where the tool is available (microbench/sanitize_small.py)."""
import pathlib
import runpy

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_small_shapes_every_kernel_matches_oracle(gpu_ctx, monkeypatch):
    monkeypatch.chdir(ROOT)
    runpy.run_path(str(ROOT / "microbench" / "sanitize_small.py"), run_name="__main__")
