"""Runs the C++ parity suite (tests/cpp/test_dump.cpp over include/posdump.hpp,
written like the reference's Catch2 suites): [cpu] cases here, [gpu] cases on
the B200.  The binary is built by __graft_entry__.build()."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_dump")


def _run(tag):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} missing: run __graft_entry__.build()")
    r = subprocess.run([BIN, tag], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    return r.stdout


def test_cpp_suite_cpu_cases():
    import re
    out = _run("[cpu]")
    m = re.search(r"(\d+)/(\d+) passed", out)
    assert m and m.group(1) == m.group(2) and int(m.group(2)) >= 6, out


@pytest.mark.gpu
def test_cpp_suite_gpu_cases():
    out = _run("[gpu]")
    assert "passed" in out
