"""float32 entry points on both of their paths (api.cu "float32 on the float64 tiers"):

  * default: float32 storage, computed on the float64 register QR / rr / register SVD tiers, the
    DMMA block pipeline (direct method) and the rsvd built on them (faster on B200, more accurate);
  * BF_F32_NATIVE=1: the float32 CUDA-core tiers.

Both against the oracle's float32 run (the reference algorithm in float32) at the north-star
float32 gate (sigma normwise <= 1e-5), vectors up to sign, flags equal, sweeps within +-2 (float32
converges at its rounding noise floor: the reference and its restatement differ by 2 sweeps on
some entries, profiles/f32_ref_r02.json), and residuals of the float32 outputs.
"""

import ctypes

import numpy as np
import pytest
import torch

import paper_1707_05141_b200 as bf
from helpers import sigma_normwise, vec_mismatch
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    orc.build()


@pytest.fixture(params=["promoted", "native"])
def mode(request, monkeypatch):
    if request.param == "native":
        monkeypatch.setenv("BF_F32_NATIVE", "1")
    else:
        monkeypatch.delenv("BF_F32_NATIVE", raising=False)
    return request.param


def f32_inputs(B, m, n, seed):
    a = bf.gaussian_tensor(B, m, n, seed, seed_mode="add", dtype=torch.float32)
    return a, np.ascontiguousarray(a.transpose(1, 2).cpu().numpy())  # device (B, m, n); oracle column-major


def res(u, s, v, a):
    u, s, v, a = (torch.as_tensor(np.asarray(x), dtype=torch.float64) for x in (u, s, v, a))
    e = torch.eye(u.shape[2], dtype=torch.float64)
    ou = (u.transpose(1, 2) @ u - e).norm(dim=(1, 2))
    ov = (v.transpose(1, 2) @ v - torch.eye(v.shape[2], dtype=torch.float64)).norm(dim=(1, 2))
    rc = (a - (u * s[:, None, :]) @ v.transpose(1, 2)).norm(dim=(1, 2)) / a.norm(dim=(1, 2))
    return float(ou.max()), float(ov.max()), float(rc.max())


@pytest.mark.parametrize("m,n,ordering", [(64, 64, "round_robin"), (32, 32, "serial"), (32, 32, "round_robin"),
                                          (48, 40, "round_robin")])
def test_svd_f32(mode, m, n, ordering):
    B = 64
    a, a3 = f32_inputs(B, m, n, 6_100_000 + m + n)
    r = bf.svd_tensor(a, bf.JacobiOptions(ordering=ordering, accumulate_v=True))
    assert r["u"].dtype == torch.float32 and r["sigma"].dtype == torch.float32
    o = orc.batch_svd_stacked(a3, m, n, ordering=ordering, accumulate_v=True, threads=8)
    s, sw, cv = r["sigma"].cpu().numpy(), r["sweeps"].cpu().numpy(), r["converged"].cpu().numpy()
    u, v = r["u"].cpu().numpy(), r["v"].cpu().numpy()
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-5
        assert bool(cv[b]) == bool(o["converged"][b])
        assert abs(int(sw[b]) - int(o["sweeps"][b])) <= 2
        assert vec_mismatch(u[b], o["u"][b].T, o["s"][b], np.float32, factor=256.0) <= 1.0
        assert vec_mismatch(v[b], o["v"][b].T, o["s"][b], np.float32, factor=256.0) <= 1.0
    g = res(u, s, v, a.cpu().numpy())
    ref = res(o["u"].transpose(0, 2, 1), o["s"], o["v"].transpose(0, 2, 1), a.cpu().numpy())
    # U orthogonality sits at the stopping tolerance for both (~1 % noise between implementations)
    assert g[0] <= 1.05 * ref[0] and g[1] <= 1.05 * ref[1] and g[2] <= 1.05 * ref[2]


@pytest.mark.parametrize("m,n", [(64, 32), (128, 40), (64, 16)])
def test_qr_f32(mode, m, n):
    B = 256
    a, a3 = f32_inputs(B, m, n, 6_200_000 + m + n)
    q, r = bf.qr_tensor(a)
    assert q.dtype == torch.float32
    qo, ro, bad = orc.batch_qr_stacked(a3, m, n, 16, threads=8)
    assert bad == -1
    an = a.cpu().numpy().astype(np.float64)
    scale = np.sqrt(np.sum(an * an, axis=(1, 2)))[:, None, None]
    eps = np.finfo(np.float32).eps
    assert np.max(np.abs(q.cpu().numpy() - qo.transpose(0, 2, 1)) / (eps * scale)) <= 64
    assert np.max(np.abs(r.cpu().numpy() - ro.transpose(0, 2, 1)) / (eps * scale)) <= 64
    assert np.all(np.tril(r.cpu().numpy(), -1) == 0)


@pytest.mark.parametrize("method", ["direct", "gram"])
def test_block_f32(mode, method):
    B, m, n = 6, 192, 160
    a, a3 = f32_inputs(B, m, n, 6_300_000)
    r = bf.block_svd_tensor(a, bf.BlockJacobiOptions(method=method, block_width=32, accumulate_v=True))
    o = orc.batch_block_svd_stacked(a3, m, n, block_width=32, method=method, accumulate_v=True, threads=B)
    s, cv, sw = r["sigma"].cpu().numpy(), r["converged"].cpu().numpy(), r["sweeps"].cpu().numpy()
    assert r["e_history"].dtype == torch.float32
    lap = np.linalg.svd(a.cpu().numpy().astype(np.float64), compute_uv=False)
    for b in range(B):
        ge = np.max(np.abs(s[b] - lap[b])) / lap[b, 0]
        oe = np.max(np.abs(o["s"][b] - lap[b])) / lap[b, 0]
        # within 1e-5 of the oracle, or closer to the exact values than the oracle
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-5 or ge <= oe
        if method == "direct":
            assert bool(cv[b]) == bool(o["converged"][b])
            assert abs(int(sw[b]) - int(o["sweeps"][b])) <= 2
        # float32 Gram: e hovers at its float32 floor (~ tol), so its sweep count is decided by
        # rounding (the reference vs its own restatement included); it always runs on the float32
        # tiers (api.cu block_promote) and is gated on sigma and the reconstruction only
    g = res(r["u"].cpu().numpy(), s, r["v"].cpu().numpy(), a.cpu().numpy())
    assert g[2] < 1e-4


def test_rsvd_f32_paths(mode):
    B, m, n, k, p = 128, 128, 128, 32, 8
    a64, _ = bf.make_matrix_tensor(B, m, n, 1e16, rank=64, seed=6_400_000)
    a = a64.transpose(1, 2).float().contiguous().transpose(1, 2)
    r = bf.rsvd_tensor(a, bf.RsvdOptions(k=k, p=p, seed=9), index_base=3)
    assert r["s"].dtype == torch.float32
    o = orc.batch_rsvd_stacked(np.ascontiguousarray(a.transpose(1, 2).cpu().numpy()), m, n, k, p, seed=9,
                               index_base=3, threads=8)
    s = r["s"].cpu().numpy()
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-5


def test_f32_promotion_engaged(monkeypatch):
    """The default float32 path really runs on the float64 tiers: its workspace holds the widened
    copies (A, U in float64), the native one does not."""
    L = bf._lib.load()
    opts = bf._lib._Opts(0.0, 30, 1, 1, 0)
    monkeypatch.delenv("BF_F32_NATIVE", raising=False)
    promoted = L.bf_svd_workspace_size(1000, 64, 64, 4, ctypes.byref(opts))
    monkeypatch.setenv("BF_F32_NATIVE", "1")
    native = L.bf_svd_workspace_size(1000, 64, 64, 4, ctypes.byref(opts))
    assert promoted >= 2 * 1000 * 64 * 64 * 8 > native


def _edge_batch(m, n, rng):
    a = rng.standard_normal((4, m, n)).astype(np.float32)
    a[0] = 0.0                       # zero matrix: sigma 0, U completed (jacobi.py:189-209)
    a[1][:, 3] = 0.0                 # one zero column
    a[2][:, 5] = a[2][:, 1]          # duplicate columns (rank deficient)
    a[3][:, :] *= np.float32(1e-6)   # small scale (squared dot products still normal in float32)
    return a


@pytest.mark.parametrize("m,n,ordering", [(32, 32, "serial"), (32, 32, "round_robin"), (64, 64, "round_robin")])
def test_svd_f32_edge_cases(mode, m, n, ordering):
    a = _edge_batch(m, n, np.random.default_rng(3))
    r = bf.svd_tensor(torch.as_tensor(a).cuda(), bf.JacobiOptions(ordering=ordering, accumulate_v=True))
    o = orc.batch_svd_stacked(np.ascontiguousarray(a.transpose(0, 2, 1)), m, n, ordering=ordering, accumulate_v=True,
                              threads=4)
    s, cv = r["sigma"].cpu().numpy(), r["converged"].cpu().numpy()
    u = r["u"].cpu().numpy().astype(np.float64)
    for b in range(4):
        assert bool(cv[b]) == bool(o["converged"][b])
        if o["s"][b][0] > 0:
            assert sigma_normwise(s[b], o["s"][b]) <= 1e-5
        else:
            assert np.all(s[b] == 0)
        # U stays orthonormal, zero directions completed
        assert np.abs(u[b].T @ u[b] - np.eye(n)).max() < 1e-4


@pytest.mark.parametrize("m,n", [(64, 32), (128, 40)])
def test_qr_f32_edge_cases(mode, m, n):
    a = _edge_batch(m, n, np.random.default_rng(4))
    q, rr = bf.qr_tensor(torch.as_tensor(a).cuda())
    qo, ro, bad = orc.batch_qr_stacked(np.ascontiguousarray(a.transpose(0, 2, 1)), m, n, 16, threads=4)
    eps = np.finfo(np.float32).eps
    qg, rg = q.cpu().numpy().astype(np.float64), rr.cpu().numpy().astype(np.float64)
    for b in range(4):
        scale = float(np.linalg.norm(a[b].astype(np.float64)))
        # orthonormal Q, QR = A, exact zeros below the diagonal: every entry
        assert np.abs(qg[b].T @ qg[b] - np.eye(n)).max() < 1e-5
        assert np.abs(qg[b] @ rg[b] - a[b]).max() <= 64 * eps * max(scale, np.finfo(np.float32).tiny)
        assert np.all(np.tril(rg[b], -1) == 0)
        # elementwise against the oracle where the factorisation is unique (full column rank; the
        # duplicate-column entry's trailing reflectors are built from rounding noise)
        if b != 2:
            assert np.abs(qg[b] - qo[b].T).max() <= 64 * eps * max(scale, 1.0)
            assert np.abs(rg[b] - ro[b].T).max() <= 64 * eps * max(scale, 1.0)
