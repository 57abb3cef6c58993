"""The C++ drop-in (include/sslic_b200.hpp over the C ABI) against the
unmodified reference headers: oracle/_ref/adapter_test compares
sslic::run_slic / enforce_connectivity with sslic::b200::run_slic /
enforce_connectivity on 40 acceptance-corpus cases (bitwise labels, centres,
connectivity) and checks the exception class of a parameter error."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_dropin_matches_reference():
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_test")
    if not os.path.exists(exe):
        pytest.skip("adapter_test not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
