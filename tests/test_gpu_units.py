"""Pair-pass unit sizes (stencil.cuh): the default 2x2x1 cell units, and the 2x1x1 and
single-cell fallbacks selected with SPH_UNIT_BITS, each checked against the oracle in
a fresh process (the unit size is read once per process).  The parity cases cover
uniform and variable h, periodic and open boxes, and the neighbour-list decode."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ubits", ["0", "1"])
def test_parity_with_other_unit_sizes(ubits):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, SPH_UNIT_BITS=ubits)
    sel = ("test_config1_square_patch_per_call or test_jittered_shuffled_patch or "
           "test_evrard_shaped_variable_h or test_pressure_ics_and_half_cells or "
           "test_brute_force_small_and_ragged or test_shadowed_multistep_config1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", sel],
                       env=env, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-3000:]
