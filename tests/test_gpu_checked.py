"""The parity suites once more against the bounds-checked build
(libtopo_b200_checked.so: -DTOPO_CHECKED, device asserts on every computed
gather / scatter / mirror-folded index, TOPO_CHECK in csrc/common.cuh). A
failed check traps the kernel, so the run fails. Stands in for
compute-sanitizer memcheck, which the GPU pool does not allow."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_suites_under_bounds_checks():
    from paper_2005_05436_b200 import build as B
    if not os.path.exists(B.LIB_CHECKED):
        B.build(checked=True)  # (built by __graft_entry__.build(); here if missing)
    env = dict(os.environ, TOPO_LIB_PATH=B.LIB_CHECKED)
    probe = subprocess.run([sys.executable, "-c", "import paper_2005_05436_b200._lib as L; "
                            "print(L.LIB_PATH)"], env=env, capture_output=True, text=True,
                           cwd=ROOT, timeout=300)
    assert probe.stdout.strip() == B.LIB_CHECKED, probe.stdout + probe.stderr
    files = ["tests/test_gpu_pass.py", "tests/test_gpu_stages.py", "tests/test_gpu_multirank.py",
             "tests/test_gpu_variants.py", "tests/test_gpu_loop.py", "tests/test_gpu_csc.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "-k", "not config5_full and not index_pairs_c5_full"] + files,
                       env=env, capture_output=True, text=True, cwd=ROOT, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
