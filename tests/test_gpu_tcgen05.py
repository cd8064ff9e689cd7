"""The tcgen05 / TMEM variant of the batch >= 8 GEMV (decode_kernel.cuh
gemv_kc under FFB_KCP_TCGEN05, built as paper_2505_22758_b200/
libffb200_tc05.so): the whole batch-16 parity suite (tests/test_gpu_batch16.py:
toy and 8B-width rows against the f64 oracle, all run modes bit-identical,
device decode loop) re-run in a subprocess with that library loaded
(FFB200_LIB), plus a check that the library reports layout 3."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2505_22758_b200", "libffb200_tc05.so")


def test_tcgen05_variant_passes_the_batch16_suite():
    assert os.path.exists(LIB), "build the variant first (make -C paper_2505_22758_b200)"
    env = dict(os.environ, FFB200_LIB=LIB, FFB_EXPECT_KC_LAYOUT="3")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(ROOT, "tests", "test_gpu_batch16.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
