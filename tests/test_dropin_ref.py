"""The drop-in from the reference's side (tests/cpp/test_dropin_ref.cpp,
compiled against the unmodified reference headers by oracle/Makefile): a
reference OperatorSetup adopted through the C ABI, the device apply inside the
reference's own cg and ConstrainedOperator, restriction validation."""
import os
import subprocess

import pytest

import oracle

HAVE_BIN = os.path.exists(oracle.DROPIN_BIN)


@pytest.mark.skipif(not os.path.isdir("/root/reference"), reason="reference absent (the GPU box runs the prebuilt binary)")
def test_dropin_binary_built_from_the_reference_headers():
    oracle.build()
    assert os.path.exists(oracle.DROPIN_BIN)


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_BIN, reason="oracle/_ref/test_dropin_ref not built")
def test_dropin_through_the_reference_api():
    out = subprocess.run([oracle.DROPIN_BIN], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout
