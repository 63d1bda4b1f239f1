"""The full-config parity gates themselves (tools/parity_full.py check()), on synthetic records:
float64 rules (sigma 1e-12, residual maxima <= the oracle's, flags / sweeps +-1 with the Gram
chaos exception) and the float32 twins' rules anchored on the reference's own run (sigma within
1e-5 or closer to exact than the oracle, sweeps +-2, residual maxima within 2 % of
max(oracle, reference)). No GPU needed."""

import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

import parity_full as pf  # noqa: E402


def res(g, o):
    return {"gpu_max": g, "oracle_max": o}


def svd_rec(name, dtype="f64", **kw):
    r = {"config": name, "batch": 1000, "dtype": dtype, "sigma_normwise": {"max": 1e-14},
         "u_mismatch_ratio": {"max": 0.1}, "v_mismatch_ratio": {"max": 0.1},
         "orth_u": res(1.0, 1.0), "orth_v": res(0.5, 1.0), "recon": res(0.5, 1.0),
         "flag_or_sweep_outliers": []}
    r.update(kw)
    return r


def test_f64_gates():
    assert pf.check(svd_rec("cfg3")) == []
    assert pf.check(svd_rec("cfg3", sigma_normwise={"max": 2e-12}))
    assert pf.check(svd_rec("cfg3", orth_v=res(1.01, 1.0)))  # no tolerance band in float64
    out = [{"index": 3, "sweeps_gpu": 9, "sweeps_oracle": 11, "conv_gpu": True, "conv_oracle": True}]
    assert pf.check(svd_rec("cfg3", flag_or_sweep_outliers=out))
    # block Gram: entries marked chaotic (e hovering at tol) are accepted, capped at 10 %
    chaotic = [dict(o, marginal=True) for o in out]
    assert pf.check(svd_rec("cfg4", flag_or_sweep_outliers=chaotic)) == []
    assert pf.check(svd_rec("cfg4", flag_or_sweep_outliers=chaotic * 101))


def test_f32_gates():
    ok = svd_rec("cfg3f32", dtype="f32", sigma_normwise={"max": 2e-6}, sigma_f32_fail=0,
                 vs_reference={"full_batch": True, "ref_max": {"orth_u": 1.0, "orth_v": 1.0, "recon": 1.0}})
    assert pf.check(ok) == []
    # sigma: judged per matrix by sigma_f32_fail (beyond 1e-5 AND farther from exact than the oracle)
    assert pf.check(dict(ok, sigma_f32_fail=1))
    assert pf.check(dict(ok, sigma_normwise={"max": 1.7e-5})) == []
    # residuals: 2 % band over max(oracle, reference)
    assert pf.check(dict(ok, orth_u=res(1.015, 1.0))) == []
    assert pf.check(dict(ok, orth_u=res(1.03, 1.0)))
    assert pf.check(dict(ok, orth_u=res(1.03, 0.9),
                         vs_reference={"full_batch": True, "ref_max": {"orth_u": 1.02, "orth_v": 1, "recon": 1}})) == []
    # sweeps: +-2 accepted in float32, flags must agree
    two = [{"index": 1, "sweeps_gpu": 9, "sweeps_oracle": 11, "conv_gpu": True, "conv_oracle": True}]
    assert pf.check(dict(ok, flag_or_sweep_outliers=two)) == []
    three = [dict(two[0], sweeps_oracle=12)]
    assert pf.check(dict(ok, flag_or_sweep_outliers=three))
    flag = [dict(two[0], conv_gpu=False)]
    assert pf.check(dict(ok, flag_or_sweep_outliers=flag))


def test_f32_configs_mirror_f64():
    for k in ("cfg1", "cfg1rr", "cfg2", "cfg3", "cfg4d", "cfg5"):
        c32 = pf.CONFIGS[k + "f32"]
        assert c32["dtype"] == "f32"
        assert {kk: v for kk, v in c32.items() if kk not in ("dtype", "tol")} == \
            {kk: v for kk, v in pf.CONFIGS[k].items() if kk != "tol"}
