"""The reference's hot-path unit tests re-run against the C++ host mirror
(paper_2207_06374_b200/csrc/host/trstmi_host.hpp) on the GPU — the same
assertions the reference's Catch2 suites make, through the C ABI."""
import os
import subprocess

import pytest

from paper_2207_06374_b200 import build

pytestmark = pytest.mark.gpu


def test_reference_unit_tests_through_cpp_host_mirror():
    exe = build.HOST_TEST_BIN
    if not os.path.exists(exe):
        build.build_host_tests()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout
