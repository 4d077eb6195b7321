"""The expansion's three write paths and the launch modes give the same bit-exact tile lists:
dense chunks through expand_dense_kernel (RS_EXPAND_DENSE=0: every chunk dense), the
transposed walk column-centric only (RS_EXPAND_MAJOR=1000) or column-major only
(RS_EXPAND_MAJOR=0), stream launches without programmatic dependent launch (RS_PDL=0), and
both depth sorts at every size (RS_DSORT=0: the onesweep launches, 2: the cooperative kernel,
with the next pass's histograms by scatter atomics or by a second barrier: RS_DSORT_RED_MAX, and
4 passes of 8-bit digits where 3 of 9 bits would do: RS_DSORT_BINS=256).
The knobs are read once per process, so each case runs tests/gpu_binning_variant.py."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"RS_EXPAND_DENSE": "0"}, {"RS_EXPAND_DENSE": "1000", "RS_EXPAND_MAJOR": "1000"},
                                 {"RS_EXPAND_DENSE": "1000", "RS_EXPAND_MAJOR": "0"}, {"RS_PDL": "0"},
                                 {"RS_DSORT": "0"}, {"RS_DSORT": "2"}, {"RS_DSORT": "2", "RS_DSORT_RED_MAX": "0"},
                                 {"RS_DSORT": "2", "RS_DSORT_RED_MAX": "4294967295"},
                                 {"RS_DSORT": "2", "RS_DSORT_BINS": "256"}],
                         ids=["all-dense", "column-centric", "column-major", "no-pdl", "onesweep-sort", "coop-sort",
                              "coop-sort-barrier-hist", "coop-sort-atomic-hist", "coop-sort-8bit-digits"])
def test_expand_paths_bit_exact(env):
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "gpu_binning_variant.py")], cwd=ROOT,
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
