"""The reference's own test suite (pkg/tests) run against this package with
``meshplan`` aliased to it (tools/reference_suite.py): every test that is not
about the out-of-scope CLI, text mesh I/O, P100 cost model or arbitrary
Python element functions (tools/reference_suite_deselect.txt, each with its
reason) must pass on the GPU.  Needs the staged copy of the reference tests
(baseline/_ref_tests, tools/stage_reference.sh); skipped without it."""

import re
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu
STAGED = REPO / "baseline" / "_ref_tests"


@pytest.mark.skipif(not (STAGED / "conftest.py").exists(), reason="reference tests not staged")
def test_reference_suite_passes_against_this_package():
    r = subprocess.run([sys.executable, str(REPO / "tools" / "reference_suite.py"), "--", "-q", "--tb=short",
                        "-p", "no:randomly"], capture_output=True, text=True, timeout=1800, cwd=REPO)
    tail = r.stdout[-4000:]
    m = re.search(r"(\d+) passed", r.stdout)
    assert r.returncode == 0, tail
    assert m and int(m.group(1)) >= 190, tail
