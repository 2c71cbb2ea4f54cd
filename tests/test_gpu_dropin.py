"""GPU: the reference's OWN public-API unit tests (test_params.cpp,
test_partition.cpp, test_format.cpp, test_decoder.cpp from
/root/reference/proj/tests, unmodified) compiled against the B200 drop-in
headers include/plz/*.hpp and linked with libplzgpu.so (oracle/Makefile
target dropin-tests; the binary is built in the development container and
travels to the GPU box)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "ref_tests_on_b200")


@pytest.mark.skipif(not os.path.exists(BIN), reason="ref_tests_on_b200 not built")
def test_reference_public_api_suite_passes_on_the_b200_dropin():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "failed: 0" in r.stdout
