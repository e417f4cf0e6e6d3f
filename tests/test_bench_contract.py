"""CPU tests of bench.py's contract that need no GPU: the reference arm runs
the compiled reference on host-generated inputs without importing the product
package, torch or CUDA, and prints the GPU arm's exact config / dtype."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(code):
    return subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                          timeout=600)


@pytest.mark.parametrize("cfg", ["C1", "C5"])
def test_reference_arm_is_cpu_only_and_matches_the_gpu_config(cfg):
    from oracle.py import available_ref
    if not available_ref():
        pytest.skip("oracle/_ref not built")
    code = f"""
import sys
sys.argv = ["bench.py", "--impl", "reference", "--config", "{cfg}", "--steps", "1", "--warmup", "1"]
import bench
bench.main()
loaded = [m for m in ("paper_1303_4312_b200", "torch") if m in sys.modules]
print("LOADED", loaded)
"""
    r = _run(code)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "LOADED []", lines[-1]
    line = json.loads(lines[-2])
    sys.path.insert(0, ROOT)
    import bench
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["dtype"] == bench.dtype_str(cfg)
    assert line["config"] == bench.config_dict(cfg, line["config"]["elements"], 1, False)
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0
    if cfg == "C5":
        assert line["config"]["elements"] == 67354964  # seed 5


def test_host_inputs_match_the_reference_generator():
    """bench.make_host_inputs (the reference arm's inputs) equals the
    reference's own seeded generator (generate.cpp:69-97, few-distinct with
    param 16 = C2's keys) element for element at full size."""
    from oracle.py import Ref, available_ref
    if not available_ref():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, ROOT)
    import numpy as np

    import bench
    h = bench.make_host_inputs("C2")
    ra, rb = Ref().generate(2, 5, 16, 2**24, 2**24)
    assert np.array_equal(h["a"].astype(np.uint64), ra)
    assert np.array_equal(h["b"].astype(np.uint64), rb)
    assert np.array_equal(h["av"], np.arange(2**24, dtype=np.uint32))
    assert np.array_equal(h["bv"], np.arange(2**24, dtype=np.uint32) | np.uint32(1 << 31))
