"""CPU emulation of the CTA-local FFT index algebra (skc_fft.cuh): every pass is
run for all work items and checked against a direct DFT, for the residue split,
both twiddle-table indexings and the compile-time pass plans."""
import pathlib
import subprocess

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_fft_core_emulation(tmp_path):
    exe = tmp_path / "fft_core_check"
    subprocess.run(["/usr/bin/g++", "-O2", "-std=c++20", "-o", str(exe),
                    str(ROOT / "tests" / "cpu_emulation" / "fft_core_check.cpp")], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout
