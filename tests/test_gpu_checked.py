"""The bounds-checked build (-DRK_CHECKED) in place of compute-sanitizer,
which is closed on the GPU pool: every kernel family runs the sanitize slice
(tools/sanitize_slice.py) against librocket_b200_checked.so, whose kernels
trap on any shared-memory window read outside the staged rows (or the NaN
slot), any global row read outside the scratch, any unaligned pair load and
any feature store outside the launch's rows.  A trap would surface as a
CUDA error and a non-zero exit; the slice also compares every result with
the oracle."""

import os
import subprocess
import sys

import pytest

from paper_2601_17091_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_has_trap_instructions():
    import shutil

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    if not os.path.exists(_lib.CHECKED_LIB_PATH):
        pytest.fail("checked library not built (run __graft_entry__.build())")
    objs = os.path.join(os.path.dirname(_lib.CHECKED_LIB_PATH), "obj_librocket_b200_checked", "kernels_len9_r3.o")
    sass = subprocess.run(["cuobjdump", "-sass", objs], capture_output=True, text=True).stdout
    assert "BPT.TRAP" in sass


@pytest.mark.gpu
def test_sanitize_slice_under_checked_build(cuda_ready):
    env = dict(os.environ, RK_LIB_PATH=_lib.CHECKED_LIB_PATH)
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sanitize_slice.py")], cwd=REPO, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "sanitize slice ok" in r.stdout
