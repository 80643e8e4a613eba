"""bench.py contract checks that need no GPU: the reference arm's JSON line (the oracle
restatement timed on the host cores) and the roofline helpers."""
import json
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "1"],
                         check=True, capture_output=True, text=True, cwd=str(ROOT), timeout=600)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "entries/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["n"] == 1000 and line["config"]["b"] == 1 << 16 and line["config"]["B"] == 10
    assert line["config"]["workload"].startswith("config2")


def test_reference_arm_does_not_load_the_product_library():
    """The CPU arm builds its input with the oracle's generator: the product .so must not
    appear in its address space (bench.py asserts it; this checks the import graph too)."""
    code = ("import sys, bench; bench.cpu_sample_tensor(2); "
            "assert not any('libsketchcp_b200' in l for l in open('/proc/self/maps')); "
            "assert 'paper_1506_04448_b200' not in sys.modules; print('ok')")
    out = subprocess.run([sys.executable, "-c", code], check=True, capture_output=True, text=True, cwd=str(ROOT),
                         timeout=600)
    assert out.stdout.strip().endswith("ok")


def test_equal_work_slices_match_distributed_helper():
    import bench
    from paper_1506_04448_b200.distributed import equal_work_slices

    for n, w in [(1000, 1), (1000, 2), (1000, 8), (400, 4), (7, 8)]:
        assert bench.equal_work_slices(n, w) == equal_work_slices(n, w)


def test_scatter_roofline_uses_measured_ceiling():
    import bench

    r = bench.scatter_roofline(10746800 * 20, 0.43)
    assert r["bound"] == "smem_atomics" and r["unit"] == "u32 atomics/s"
    assert 0.0 < r["frac"] < 1.0
    assert abs(r["achieved"] - 2 * 10746800 * 20 / 0.43e-3) < 1.0
    assert bench.scatter_roofline(1, None) is None
    g = bench.scatter_roofline(167167000 * 10, 1.5, limbs=1, gather_stride=4)
    assert g["limbs"] == 1 and "t_gather_ms" in g and 0.0 < g["frac"] < 1.5
