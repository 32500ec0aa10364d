"""The grouped GEMM's static tile stride (MOE_STATIC_TILES=1) gives the same
results as the default dynamic schedule (separate process: the switch is read
once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_static_tile_schedule_matches_gemm_tests():
    env = dict(os.environ, MOE_STATIC_TILES="1")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", os.path.join(ROOT, "tests", "test_gpu_gemm.py"),
                        os.path.join(ROOT, "tests", "test_gpu_layer.py") + "::test_layer_fwd_bwd_vs_oracle"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
