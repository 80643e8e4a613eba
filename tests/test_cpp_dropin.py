"""The drop-in C++ API (include/sketchcp/*.hpp over the C-ABI) compiles as a user
would compile against the reference headers, and (on a B200) passes the
reference-style tests in tests/cpp/test_dropin.cpp."""
import pathlib
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_1506_04448_b200" / "_lib"


def build_dropin(out: pathlib.Path) -> pathlib.Path:
    exe = out / "test_dropin"
    subprocess.run(["/usr/bin/g++", "-O1", "-std=c++20", "-I", str(ROOT / "include"), "-I", str(ROOT / "compat"),
                    str(ROOT / "tests" / "cpp" / "test_dropin.cpp"), "-o", str(exe), "-L", str(LIB), "-lsketchcp",
                    "-lsketchcp_b200", f"-Wl,-rpath,{LIB}"], check=True)
    return exe


def test_dropin_compiles_and_links(tmp_path):
    assert build_dropin(tmp_path).exists()


@pytest.mark.gpu
def test_dropin_reference_style_suite(tmp_path):
    exe = build_dropin(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " 0 failed" in out.stdout
