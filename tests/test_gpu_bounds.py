"""Memory-safety evidence without compute-sanitizer (closed on the GPU pool):
the bounds-checked build (`make -C paper_2504_09307_b200/csrc debug`,
-DLUMOS_DEBUG_BOUNDS) checks every slot, mailbox, ring and output index the
kernels compute.  These tests run the sanitizer workload
(tools/sanitize_driver.py: every kernel family at test size) on that build and
show the checks fire on a deliberately corrupted program."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2504_09307_b200", "lib", "variants", "liblumos_debug.so")


def _run(extra_env, code):
    env = dict(os.environ, LUMOS_B200_LIB=DEBUG_LIB, **extra_env)
    return subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                          timeout=900, cwd=ROOT)


@pytest.mark.skipif(not os.path.exists(DEBUG_LIB), reason="debug build missing (make debug)")
def test_every_kernel_in_bounds():
    r = _run({}, "import runpy; runpy.run_path('tools/sanitize_driver.py', run_name='__main__')")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "sanitize driver ok" in r.stdout
    assert "bounds check failed" not in r.stdout + r.stderr


@pytest.mark.skipif(not os.path.exists(DEBUG_LIB), reason="debug build missing (make debug)")
def test_bounds_checks_fire_on_a_corrupt_program():
    code = """
import sys
sys.path.insert(0, 'tests')
import refshim as R
from paper_2504_09307_b200 import ScenarioSpec, simulate_batch
h, _ = R.generate(R.synth_spec(pp=2, dp=1, m=2, layers=2))
try:
    simulate_batch(h.export(), ScenarioSpec(count=4, jitter=0.1))
except Exception as e:
    print('caught:', e)
"""
    r = _run({"LUMOS_DEBUG_CORRUPT": "1"}, code)
    assert "bounds check failed" in r.stdout + r.stderr, r.stdout + r.stderr
