"""The CUDA sampler's log1p / log1pf restatement (csrc/libm_log1p.h) equals the host C library
bit for bit -- numpy's ziggurat tail returns r - log1p(-U)/r, so this is what makes the device
Gaussian stream bitwise numpy's (rsvd.py:42-53). The header is compiled here with gcc and every
float tail argument (2^24) plus random doubles are compared with glibc's results. CPU only."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_log1p_restatement_matches_host_libm(tmp_path):
    exe = tmp_path / "libm_check"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "paper_1707_05141_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "libm_check.cpp"), "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe), "2000000"], check=True, capture_output=True, text=True).stdout
    rows = {ln.split()[0]: (int(ln.split()[1]), int(ln.split()[2])) for ln in out.strip().splitlines()}
    assert set(rows) == {"log1pf_tail_grid", "log1pf_all_strided", "log1p_tail_random", "log1p_all_random"}
    for name, (bad, n) in rows.items():
        assert n > 100000, name
        assert bad == 0, f"{name}: {bad} of {n} results differ from the host libm"
