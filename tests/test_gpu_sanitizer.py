"""compute-sanitizer over every decode mode, both u8 variants, fp32 and the error paths
(SURVEY.md §4 item 5): no memory errors, no shared-memory races, no uninitialised reads.

Some GPU pools close compute-sanitizer (its wrapper exits 86 with a message saying so). There the
sanitizer legs skip, and `test_sanitize_case_plain` still runs the same cases without it: every
status, the truncated-last-file cases and the canary bytes around each output are checked by the
script itself."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = os.path.join(ROOT, "scripts", "sanitize_case.py")


def _check_case_output(out: str) -> None:
    # the truncated file and the k = 0 file must be reported
    assert "5, 4]" in out or "5, 4" in out, out[-2000:]
    assert "truncated-last cases ok" in out, out[-2000:]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "initcheck", "synccheck"])
def test_compute_sanitizer(tool):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    # no caching allocator: every tensor is its own cudaMalloc, so a read past a buffer is reported
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "9", sys.executable, CASE],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "closed" in out:
        pytest.skip("compute-sanitizer is closed on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-4000:]
    assert "0 errors" in out or "0 hazards" in out, out[-2000:]
    _check_case_output(out)


def test_sanitize_case_plain():
    """The sanitizer's cases without the sanitizer (statuses, truncated-last files, canaries)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    r = subprocess.run([sys.executable, CASE], capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    _check_case_output(out)
