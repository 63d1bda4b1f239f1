"""Full-config parity on the GPU: EVERY entry of cfg1 (both orderings), cfg2, cfg3, cfg4 (Gram),
cfg4d (direct) and cfg5, and their float32 twins, through the CUDA path against the CPU oracle on
the same inputs (tools/parity_full.py: sigma normwise <= 1e-12 / 1e-5, U/V equal up to sign,
converged/sweeps rules, residual maxima no worse than the oracle's -- and for float32 the
reference's own -- maxima on the batch). Committed records: profiles/parity_r02.json,
profiles/parity_f32_r02.json."""

import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

import parity_full  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(parity_full.CONFIGS))
def test_full_config_parity(name):
    rec = parity_full.run_config(name, parity_full.host_threads())
    failed = parity_full.check(rec)
    assert not failed, failed
