"""Device-side bounds checks in place of compute-sanitizer (closed on this GPU pool): the library
rebuilt with -DFMM_CHECK traps on any data-dependent index outside the capacity of the buffer it
addresses (P2P source runs and target chunks, merged run lists, P2M / L2P leaf particle ranges,
tcgen05 M2L source rows, result rows and per-pair slots, traversal source / target cells, the
ordered M2L reduction's slots; common.cuh FMM_DCHECK). The all-kernel workload of
tools/sanitize_run.py (every mode, the three M2L paths, both summation modes, distinct target /
source sets, an in-process 2-rank group) must run clean, and a deliberately violated bound
(FMM_CHECK_SELFTEST) must trap -- the checks are live."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1108_5815_b200", "libfmm_check.so")


@pytest.fixture(scope="module")
def checked_lib():
    sys.path.insert(0, ROOT)
    from paper_1108_5815_b200 import build as b

    if b.stale() or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(b.LIB):
        b.build(out=LIB, extra=["-DFMM_CHECK"])
    return LIB


def run_workload(lib, extra_env=None):
    env = dict(os.environ, FMM_LIB=lib, **(extra_env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")],
                          capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)


def test_checked_build_runs_clean(checked_lib):
    r = run_workload(checked_lib)
    out = r.stdout + r.stderr
    assert "FMM_CHECK failed" not in out, out[-3000:]
    assert r.returncode == 0 and "SANITIZE_DONE" in out, out[-3000:]


def test_checks_are_live(checked_lib):
    r = run_workload(checked_lib, {"FMM_CHECK_SELFTEST": "1"})
    out = r.stdout + r.stderr
    assert r.returncode != 0 and "FMM_CHECK failed" in out, out[-3000:]
