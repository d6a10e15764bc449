"""GPU: the reference's OWN doctest files (test_nufft.cpp, test_fft.cpp, test_grid.cpp, test_eig.cpp),
compiled unchanged against include/nuspectral/*.hpp and linked to libnuspectral_b200.so
(build recipe: `make reftests`; binaries in oracle/_ref/dropin, built where the
reference tree exists and shipped with the repo snapshot)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin")


@pytest.mark.parametrize("window", ["gaussian", "es"])
@pytest.mark.parametrize("name", ["test_nufft", "test_fft", "test_grid", "test_eig"])
def test_reference_doctest_file_passes_against_dropin(name, window):
    """Under the reference's Gaussian window and under the default ES window (NUS_KERNEL)."""
    exe = os.path.join(DROPIN, name)
    if not os.path.exists(exe):
        pytest.skip("drop-in reference tests not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, NUS_KERNEL=window))
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout
