"""GPU parity: the CUDA path (through the C ABI) against the reference's golden outputs
and the CPU oracle, plus size-independent properties at the BASELINE config shapes.

Gates (north star / SURVEY.md §8c): sigma normwise max|ds|/s1 <= 1e-12 (f64) / 1e-5 (f32);
U, V equal up to column sign at a sigma_1/gap-scaled tolerance; converged flags equal and
sweeps within +-1 for the same ordering; QR elementwise at ~64 eps ||A||.
"""

import numpy as np
import pytest
import torch

import paper_1707_05141_b200 as bf
from helpers import case, golden, names, orth_residual, recon_residual, sigma_normwise, vec_mismatch
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def gate(dtype):
    return 1e-12 if np.dtype(dtype) == np.float64 else 1e-5


@pytest.fixture(scope="module", autouse=True)
def _setup():
    orc.build()
    torch.cuda.init()


def dev_gauss(batch, m, n, seed0):
    """Device Gaussian batch (B, m, n) with keys seed0 + i (bench/test input convention)."""
    return bf.gaussian_tensor(batch, m, n, seed0, seed_mode="add")


def stack_np(t):
    """(B, m, n) device tensor -> (B, n, m) C-contiguous numpy (per-matrix column-major)."""
    return t.transpose(-1, -2).contiguous().cpu().numpy()


# ------------------------------------------------------------------ Gaussian sampler


def test_gaussian_bitwise_vs_reference():
    """gaussian_matrix == the reference's own draws (golden), bit for bit, float64 and float32."""
    g = golden("gauss_testmat")
    for j in range(int(g["g_count"])):
        seed = int(g[f"g{j}/seed_lo"]) | (int(g[f"g{j}/seed_hi"]) << 64)
        x = bf.gaussian_matrix(128, 40, seed)
        assert x.dtype == np.float64 and np.array_equal(x, g[f"g{j}/x"]), f"f64 seed {seed}"
        x32 = bf.gaussian_matrix(128, 40, seed, np.float32)
        assert x32.dtype == np.float32 and np.array_equal(x32, g[f"g{j}/x32"]), f"f32 seed {seed}"


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_gaussian_batch_bitwise_vs_oracle(dtype):
    """10^4 cfg5 sketches (128 x 40, keys 5 ^ i) against the oracle (numpy's stream restated in C,
    pinned to numpy above): array_equal. ~1.3 ziggurat-tail samples per matrix, so the tail
    (log1p) and wedge paths are exercised thousands of times; asserted below."""
    B = 10_000
    t = bf.gaussian_tensor(B, 128, 40, 5, seed_mode="xor", dtype=dtype)
    got = stack_np(t)  # (B, 40, 128): per-matrix column-major
    npd = np.float64 if dtype == torch.float64 else np.float32
    ref = np.stack([orc.gaussian_matrix(128, 40, 5 ^ b, npd).T for b in range(B)])
    assert got.dtype == ref.dtype
    bad = np.flatnonzero(np.any(got != ref, axis=(1, 2)))
    assert bad.size == 0, f"{bad.size} matrices differ, first {bad[:8]}"
    tails = int(np.sum(np.abs(got) > 3.6541528853610088))  # ziggurat tail samples exceed r
    assert tails > 5000, tails


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_gaussian_long_streams_bitwise(dtype):
    """Long streams (Philox block boundaries, many slow-path events per matrix), C-order and
    column-major stores, 128-bit keys."""
    npd = np.float64 if dtype == torch.float64 else np.float32
    for seed in (0, (1 << 64) + 9, (1 << 127) + 12345):
        t = bf.gaussian_tensor(2, 700, 301, seed, seed_mode="add", dtype=dtype)
        got = stack_np(t)
        for b in range(2):
            ref = orc.gaussian_matrix(700, 301, seed + b, npd)
            assert np.array_equal(got[b].T, ref), (seed, b)


# ------------------------------------------------------------------ QR


@pytest.mark.parametrize("nm", names(golden("qr")))
def test_qr_golden(nm):
    c = case(golden("qr"), nm)
    a = c["a"]
    res = bf.qr(a, int(c["pw"]))
    scale = max(np.linalg.norm(a), 1.0)
    tol = 64 * np.finfo(a.dtype).eps * scale
    d = np.abs(np.diag(c["r"])).astype(np.float64)
    ok = np.cumprod(d > 1e3 * np.finfo(a.dtype).eps * scale).astype(bool)
    assert res.q.dtype == a.dtype and res.r.dtype == a.dtype
    assert np.max(np.abs(res.q - c["q"])[:, ok], initial=0.0) <= 4 * tol
    assert np.max(np.abs(res.r - c["r"])[ok, :], initial=0.0) <= tol
    assert np.all(np.tril(res.r, -1) == 0)
    assert orth_residual(res.q) <= (1e-13 if a.dtype == np.float64 else 1e-5)


def test_qr_cfg2_batch_vs_oracle():
    a = dev_gauss(512, 64, 32, 2_000_000)
    q, r = bf.qr_tensor(a)
    a3 = stack_np(a)
    qo, ro, bad = orc.batch_qr_stacked(a3, 64, 32, 16, threads=8)
    assert bad == -1
    assert np.max(np.abs(stack_np(q) - qo)) < 1e-13
    assert np.max(np.abs(stack_np(r) - ro)) < 1e-13


def test_qr_errors_and_batch_index():
    with pytest.raises(bf.BatchError) as ei:
        bf.batch_qr([np.ones((4, 2)), np.ones((2, 3)), np.ones((3, 2)), np.ones((1, 5))])
    assert ei.value.index == 1
    with pytest.raises(ValueError):
        bf.qr(np.ones((2, 3)))
    # heterogeneous batch keeps per-entry order
    res = bf.batch_qr([np.eye(3), np.array([[3.0], [4.0]])])
    assert np.allclose(res[1].r, [[-5.0]]) and np.allclose(res[1].q.ravel(), [-0.6, -0.8])


# ------------------------------------------------------------------ Jacobi SVD


def _svd_case(nm, tier="auto"):
    c = case(golden("svd"), nm)
    tol = float(c["tolerance"])
    opts = bf.JacobiOptions(
        tolerance=None if tol < 0 else tol,
        max_sweeps=int(c["max_sweeps"]),
        ordering=str(c["ordering"]),
        accumulate_v=bool(c["accumulate_v"]),
        tier=tier,
    )
    return c, bf.svd(c["a"], opts)


@pytest.mark.parametrize("tier", ["auto", "shared"])
@pytest.mark.parametrize("nm", names(golden("svd")))
def test_svd_golden(nm, tier):
    c, r = _svd_case(nm, tier)
    a = c["a"]
    assert r.u.dtype == a.dtype and r.sigma.dtype == a.dtype
    assert sigma_normwise(r.sigma, c["sigma"]) <= gate(a.dtype)
    assert r.converged == bool(c["converged"])
    assert abs(r.sweeps - int(c["sweeps"])) <= 1
    assert np.all(np.diff(r.sigma.astype(np.float64)) <= 0)
    assert vec_mismatch(r.u, c["u"], c["sigma"], a.dtype) <= 1.0
    if bool(c["accumulate_v"]):
        assert vec_mismatch(r.v, c["v"], c["sigma"], a.dtype) <= 1.0
        if a.size and c["sigma"][0] > 0:
            assert recon_residual(a, r.u, r.sigma, r.v) <= 64 * np.finfo(a.dtype).eps * a.shape[1]
    if a.shape[1] and a.dtype == np.float64 and c["sigma"].size and c["sigma"][0] > 0:
        # residuals no worse than the reference's own on the same matrix (north star). U's
        # orthogonality is set by the convergence tolerance, not rounding: equal to ~1 %.
        eps_n = np.finfo(np.float64).eps * a.shape[1]
        assert orth_residual(r.u) <= 1.02 * orth_residual(c["u"]) + eps_n
        if bool(c["accumulate_v"]):
            assert orth_residual(r.v) <= orth_residual(c["v"]) + eps_n
            assert recon_residual(a, r.u, r.sigma, r.v) <= recon_residual(a, c["u"], c["sigma"], c["v"]) + eps_n


@pytest.mark.parametrize("ordering", ["serial", "round_robin"])
@pytest.mark.parametrize("shape,tier", [((32, 32), "auto"), ((32, 32), "shared"), ((64, 64), "auto"),
                                        ((40, 40), "auto"), ((48, 20), "auto")])
def test_svd_batch_vs_oracle(shape, tier, ordering):
    m, n = shape
    B = 48
    a = dev_gauss(B, m, n, 1_000_000 + 7 * m + n)
    opts = bf.JacobiOptions(ordering=ordering, accumulate_v=True, tier=tier)
    r = bf.svd_tensor(a, opts, rotations=True)
    a3 = stack_np(a)
    o = orc.batch_svd_stacked(a3, m, n, ordering=ordering, accumulate_v=True, threads=8)
    s = r["sigma"].cpu().numpy()
    u = stack_np(r["u"])
    v = stack_np(r["v"])
    sw = r["sweeps"].cpu().numpy()
    cv = r["converged"].cpu().numpy()
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-12
        assert abs(int(sw[b]) - int(o["sweeps"][b])) <= 1
        assert bool(cv[b]) == bool(o["converged"][b])
        assert vec_mismatch(u[b].T, o["u"][b].T, o["s"][b], np.float64) <= 1.0
        assert vec_mismatch(v[b].T, o["v"][b].T, o["s"][b], np.float64) <= 1.0


@pytest.mark.parametrize("shape", [(128, 122), (200, 100), (300, 180)])
def test_svd_shared_tier_v_in_global(shape):
    """Shapes whose W fits shared memory but W + V does not (W in smem, V in global/L2), and
    one (300 x 180) where neither fits (everything in the global workspace)."""
    m, n = shape
    B = 6
    a = dev_gauss(B, m, n, 2_000_000 + m + n)
    r = bf.svd_tensor(a, bf.JacobiOptions(ordering="round_robin", accumulate_v=True))
    a3 = stack_np(a)
    o = orc.batch_svd_stacked(a3, m, n, ordering="round_robin", accumulate_v=True, threads=8)
    s = r["sigma"].cpu().numpy()
    u, v = stack_np(r["u"]), stack_np(r["v"])
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-12
        assert vec_mismatch(u[b].T, o["u"][b].T, o["s"][b], np.float64) <= 1.0
        assert vec_mismatch(v[b].T, o["v"][b].T, o["s"][b], np.float64) <= 1.0


@pytest.mark.parametrize("ordering", ["serial", "round_robin"])
def test_svd_f32_shared_tier_vs_oracle(ordering):
    """f32 through the shared-memory tier (96 x 80: beyond the register tier) vs the oracle."""
    B, m, n = 8, 96, 80
    a = np.random.default_rng(11).standard_normal((B, m, n)).astype(np.float32)
    r = bf.svd_tensor(torch.as_tensor(a).cuda(), bf.JacobiOptions(ordering=ordering, accumulate_v=True))
    o = orc.batch_svd_stacked(np.ascontiguousarray(a.transpose(0, 2, 1)), m, n, ordering=ordering,
                              accumulate_v=True, threads=8)
    s = r["sigma"].cpu().numpy()
    sw = r["sweeps"].cpu().numpy()
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-5
        assert abs(int(sw[b]) - int(o["sweeps"][b])) <= 1
    ad = torch.as_tensor(a, dtype=torch.float64)
    rec = (r["u"].cpu().double() * r["sigma"].cpu().double()[:, None, :]) @ r["v"].cpu().double().transpose(1, 2)
    assert float(((ad - rec).norm(dim=(1, 2)) / ad.norm(dim=(1, 2))).max()) < 1e-5


@pytest.mark.parametrize("ordering", ["serial", "round_robin"])
def test_svd_cfg1_full_batch_properties(ordering):
    """All 1,000 cfg1 matrices: the residual maxima are no worse than the oracle's own maxima on
    the same batch, and below SURVEY §8c's bars (7.0e-14 / 1.6e-14 / 2.9e-15)."""
    a = dev_gauss(1000, 32, 32, 1_000_000)
    r = bf.svd_tensor(a, bf.JacobiOptions(ordering=ordering, accumulate_v=True))
    u, s, v = r["u"], r["sigma"], r["v"]
    eye = torch.eye(32, dtype=torch.float64, device=a.device)
    assert torch.all(r["converged"])
    o = orc.batch_svd_stacked(stack_np(a), 32, 32, ordering=ordering, accumulate_v=True, threads=8)
    ao = torch.as_tensor(stack_np(a)).transpose(1, 2)
    uo, vo = torch.as_tensor(o["u"]).transpose(1, 2), torch.as_tensor(o["v"]).transpose(1, 2)
    so = torch.as_tensor(o["s"])
    e = torch.eye(32, dtype=torch.float64)
    ou_o = float((uo.transpose(1, 2) @ uo - e).norm(dim=(1, 2)).max())
    ov_o = float((vo.transpose(1, 2) @ vo - e).norm(dim=(1, 2)).max())
    rc_o = float(((ao - (uo * so[:, None, :]) @ vo.transpose(1, 2)).norm(dim=(1, 2)) / ao.norm(dim=(1, 2))).max())
    ou = float((u.transpose(1, 2) @ u - eye).norm(dim=(1, 2)).max())
    ov = float((v.transpose(1, 2) @ v - eye).norm(dim=(1, 2)).max())
    rec = (u * s[:, None, :]) @ v.transpose(1, 2)
    rc = float(((a - rec).norm(dim=(1, 2)) / a.norm(dim=(1, 2))).max())
    assert ou <= ou_o and ou <= 7.1e-14, (ou, ou_o)
    assert ov <= ov_o and ov <= 1.6e-14, (ov, ov_o)
    assert rc <= rc_o and rc <= 2.9e-15, (rc, rc_o)
    assert bool(torch.all(s[:, :-1] >= s[:, 1:]))


def test_svd_errors():
    with pytest.raises(ValueError):
        bf.svd(np.ones((2, 3)))
    with pytest.raises(bf.BatchError) as ei:
        bf.batch_svd([np.ones((3, 3)), np.ones((3, 3)), np.ones((1, 2))])
    assert ei.value.index == 2
    r = bf.svd(np.zeros((5, 0)))
    assert r.u.shape == (5, 0) and r.sigma.shape == (0,) and r.converged and r.sweeps == 0


def test_empty_batches():
    """Empty batches return empty results through every entry point (core.py:97-123: a batch
    is a list; the reference maps over zero entries)."""
    assert bf.batch_svd([]) == [] and bf.batch_qr([]) == [] and bf.batch_block_svd([]) == []
    assert bf.batch_rsvd([], bf.RsvdOptions(k=2)) == []
    z = torch.empty((0, 8, 6), dtype=torch.float64, device="cuda")
    r = bf.svd_tensor(z, bf.JacobiOptions(accumulate_v=True))
    assert r["u"].shape == (0, 8, 6) and r["sigma"].shape == (0, 6)
    q, rr = bf.qr_tensor(z)
    assert q.shape == (0, 8, 6) and rr.shape == (0, 6, 6)
    z64 = torch.empty((0, 64, 64), dtype=torch.float64, device="cuda")
    rb = bf.block_svd_tensor(z64, bf.BlockJacobiOptions(accumulate_v=True))
    assert rb["sigma"].shape == (0, 64)
    rs = bf.rsvd_tensor(z64, bf.RsvdOptions(k=8, p=8))
    assert rs["s"].shape == (0, 16)


# ------------------------------------------------------------------ block Jacobi


@pytest.mark.parametrize("nm", names(golden("block")))
def test_block_golden(nm):
    c = case(golden("block"), nm)
    a = c["a"]
    tol = float(c["tolerance"])
    opts = bf.BlockJacobiOptions(
        block_width=int(c["block_width"]),
        method=str(c["method"]),
        tolerance=None if tol < 0 else tol,
        accumulate_v=bool(c["accumulate_v"]),
    )
    r = bf.block_svd(a, opts)
    sref = c["sigma"].astype(np.float64)
    if str(c["method"]) == "gram" and not bool(c["converged"]):
        # Gram squares the condition number: values below sqrt(eps)*s1 are rounding noise in the
        # reference itself (blockjacobi.py:3-5), so only the resolvable part is compared
        floor = 64 * np.sqrt(np.finfo(a.dtype).eps) * sref[0]
        keep = sref > floor
        assert sigma_normwise(r.sigma[keep], sref[keep]) <= gate(a.dtype)
        assert np.all(np.abs(r.sigma[~keep]) <= 4 * floor)
    else:
        assert sigma_normwise(r.sigma, sref) <= gate(a.dtype)
    assert r.converged == bool(c["converged"])
    assert abs(r.sweeps - int(c["sweeps"])) <= 1
    eh = c["e_history"]
    k = min(len(eh), len(r.e_history))
    big = (eh[:k] > 1e-8) & (a.dtype == np.float64)
    assert np.allclose(np.array(r.e_history[:k])[big], eh[:k][big], rtol=1e-3)
    if not bool(c["converged"]):
        return
    if "u" in c:
        assert vec_mismatch(r.u, c["u"], c["sigma"], a.dtype, factor=4096.0) <= 1.0
    if "v" in c:
        assert vec_mismatch(r.v, c["v"], c["sigma"], a.dtype, factor=4096.0) <= 1.0


def test_block_cfg4_gram_vs_oracle():
    B = 6
    a = dev_gauss(B, 256, 256, 4_000_000)
    opts = bf.BlockJacobiOptions(method="gram", block_width=32, tolerance=1e-11, accumulate_v=True)
    r = bf.block_svd_tensor(a, opts)
    o = orc.batch_block_svd_stacked(stack_np(a), 256, 256, block_width=32, method="gram", tol=1e-11,
                                    accumulate_v=True, threads=B)
    s = r["sigma"].cpu().numpy()
    sw = r["sweeps"].cpu().numpy()
    eh = r["e_history"].cpu().numpy()
    tol = 1e-11
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-12
        so = int(o["sweeps"][b])
        eo = o["e_history"][b, :so]
        k = min(so, int(sw[b]))
        big = eo[:k] > 1e-8
        assert np.allclose(eh[b, :k][big], eo[:k][big], rtol=1e-3)
        # Gram's e stalls near eps*kappa^2: when the oracle only crossed tol inside that
        # noise band, the sweep at which either side dips below tol is chaotic -- skip the count there
        decisive = so < 2 or (eo[-1] < tol and eo[-2] > 3 * tol)
        if decisive:
            assert abs(int(sw[b]) - so) <= 1
    u, v = r["u"], r["v"]
    rec = (u * r["sigma"][:, None, :]) @ v.transpose(1, 2)
    rel = (a - rec).norm(dim=(1, 2)) / a.norm(dim=(1, 2))
    assert float(rel.max()) < 1e-12


@pytest.mark.parametrize("method", ["gram", "direct"])
@pytest.mark.parametrize("m,n,bw,dtype", [(256, 256, 64, np.float64), (200, 150, 48, np.float64),
                                          (160, 120, 40, np.float32), (130, 130, 100, np.float64)])
def test_block_wide_width_vs_oracle(method, m, n, bw, dtype):
    """block_width > 32 (pair width 2k > 64; the reference accepts any width, blockjacobi.py:98-104):
    the staged wide-pair pipeline against the oracle -- sigma, vectors, flags, sweeps, e_history."""
    B = 3
    a = dev_gauss(B, m, n, 4_200_000 + m + n + bw)
    if dtype == np.float32:
        a = a.float()
    tol = 1e-11 if method == "gram" and dtype == np.float64 else None
    opts = bf.BlockJacobiOptions(method=method, block_width=bw, tolerance=tol, accumulate_v=True)
    r = bf.block_svd_tensor(a, opts)
    otol = tol if tol is not None else (1e-13 if dtype == np.float64 else 1e-5)
    o = orc.batch_block_svd_stacked(stack_np(a), m, n, block_width=bw, method=method, tol=otol,
                                    accumulate_v=True, threads=B)
    s = r["sigma"].cpu().numpy()
    sw = r["sweeps"].cpu().numpy()
    cv = r["converged"].cpu().numpy()
    eh = r["e_history"].cpu().numpy()
    u, v = stack_np(r["u"]), stack_np(r["v"])
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= gate(dtype)
        so = int(o["sweeps"][b])
        eo = o["e_history"][b, :so]
        k = min(so, int(sw[b]))
        big = eo[:k] > (1e-8 if dtype == np.float64 else 1e-3)
        assert np.allclose(eh[b, :k][big], eo[:k][big], rtol=1e-3 if dtype == np.float64 else 1e-2)
        decisive = so < 2 or (eo[-1] < otol and eo[-2] > 3 * otol)
        if decisive:
            assert abs(int(sw[b]) - so) <= 1
            assert bool(cv[b]) == bool(o["converged"][b])
        if dtype == np.float64 and bool(o["converged"][b]):
            assert vec_mismatch(u[b].T, o["u"][b].T, o["s"][b], np.float64, factor=4096.0) <= 1.0
            assert vec_mismatch(v[b].T, o["v"][b].T, o["s"][b], np.float64, factor=4096.0) <= 1.0
    ad = a.double()
    rec = (r["u"].double() * r["sigma"].double()[:, None, :]) @ r["v"].double().transpose(1, 2)
    rel = (ad - rec).norm(dim=(1, 2)) / ad.norm(dim=(1, 2))
    assert float(rel.max()) < (1e-12 if dtype == np.float64 else 1e-4)


@pytest.mark.parametrize("m,n", [(256, 256), (200, 128), (300, 128)])
def test_block_direct_bw32_vs_oracle(m, n):
    """Direct method at the BASELINE block width (pair 2k = 64): register pair QR for m <= 256,
    shared-memory pair QR above; sigma, vectors, sweeps and flags against the oracle."""
    B = 4
    a = dev_gauss(B, m, n, 4_100_000 + m + n)
    opts = bf.BlockJacobiOptions(method="direct", block_width=32, accumulate_v=True)
    r = bf.block_svd_tensor(a, opts)
    o = orc.batch_block_svd_stacked(stack_np(a), m, n, block_width=32, method="direct", tol=1e-13,
                                    accumulate_v=True, threads=B)
    s = r["sigma"].cpu().numpy()
    sw = r["sweeps"].cpu().numpy()
    cv = r["converged"].cpu().numpy()
    u, v = stack_np(r["u"]), stack_np(r["v"])
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-12
        assert abs(int(sw[b]) - int(o["sweeps"][b])) <= 1
        assert bool(cv[b]) == bool(o["converged"][b])
        assert vec_mismatch(u[b].T, o["u"][b].T, o["s"][b], np.float64) <= 1.0
        assert vec_mismatch(v[b].T, o["v"][b].T, o["s"][b], np.float64) <= 1.0


@pytest.mark.parametrize("method", ["gram", "direct"])
@pytest.mark.parametrize("m,n", [(129, 72), (255, 200)])
def test_block_odd_rows_vs_oracle(method, m, n):
    """Odd row counts (columns 8-byte aligned only: the 16-byte cp.async / tensor-map TMA staging
    falls back to plain loads) through the batched DMMA pipelines, against the oracle."""
    B = 3
    a = dev_gauss(B, m, n, 4_300_000 + m + n)
    tol = 1e-11 if method == "gram" else None
    r = bf.block_svd_tensor(a, bf.BlockJacobiOptions(method=method, block_width=32, tolerance=tol, accumulate_v=True))
    o = orc.batch_block_svd_stacked(stack_np(a), m, n, block_width=32, method=method,
                                    tol=tol if tol is not None else 1e-13, accumulate_v=True, threads=B)
    s = r["sigma"].cpu().numpy()
    u, v = stack_np(r["u"]), stack_np(r["v"])
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-12
        assert vec_mismatch(u[b].T, o["u"][b].T, o["s"][b], np.float64, factor=4096.0) <= 1.0
        assert vec_mismatch(v[b].T, o["v"][b].T, o["s"][b], np.float64, factor=4096.0) <= 1.0


@pytest.mark.parametrize("method", ["gram", "direct"])
def test_block_f32_vs_oracle(method):
    """f32 block Jacobi (one-CTA-per-pair f32 steps) vs the oracle at the f32 gates."""
    B, m, n = 4, 160, 128
    a = np.random.default_rng(13).standard_normal((B, m, n)).astype(np.float32)
    opts = bf.BlockJacobiOptions(method=method, block_width=32, accumulate_v=True)
    r = bf.block_svd_tensor(torch.as_tensor(a).cuda(), opts)
    o = orc.batch_block_svd_stacked(np.ascontiguousarray(a.transpose(0, 2, 1)), m, n, block_width=32, method=method,
                                    accumulate_v=True, threads=B)
    s = r["sigma"].cpu().numpy()
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-5
    ad = torch.as_tensor(a, dtype=torch.float64)
    rec = (r["u"].cpu().double() * r["sigma"].cpu().double()[:, None, :]) @ r["v"].cpu().double().transpose(1, 2)
    assert float(((ad - rec).norm(dim=(1, 2)) / ad.norm(dim=(1, 2))).max()) < 1e-4


# ------------------------------------------------------------------ randomized SVD


@pytest.mark.parametrize("nm", names(golden("rsvd")))
def test_rsvd_golden(nm):
    c = case(golden("rsvd"), nm)
    a = c["a"]
    seed = int(c["seed"]) ^ int(c["index"])
    r = bf.rsvd(a, bf.RsvdOptions(k=int(c["k"]), p=int(c["p"]), seed=seed))
    assert r.s.dtype == a.dtype
    assert sigma_normwise(r.s, c["s"]) <= gate(a.dtype)
    k = int(c["k"])
    assert vec_mismatch(r.u[:, :k], c["u"][:, :k], c["s"][:k], a.dtype, factor=4096.0) <= 1.0
    assert vec_mismatch(r.v[:, :k], c["v"][:, :k], c["s"][:k], a.dtype, factor=4096.0) <= 1.0


def test_rsvd_f32_with_caller_omega_vs_oracle():
    """f32 rsvd (the caller supplies the sketch: numpy's float32 ziggurat is a different stream)
    against the oracle on the same Omega; gate 1e-5 normwise (north star, f32)."""
    B, m, n, k, p = 16, 128, 96, 24, 8
    rng = np.random.default_rng(7)
    a = rng.standard_normal((B, m, n)).astype(np.float32)
    om = rng.standard_normal((B, n, k + p)).astype(np.float32)
    r = bf.rsvd_tensor(torch.as_tensor(a).cuda(), bf.RsvdOptions(k=k, p=p, seed=3), omega=torch.as_tensor(om).cuda())
    o = orc.batch_rsvd_stacked(np.ascontiguousarray(a.transpose(0, 2, 1)), m, n, k, p, seed=3,
                               omega3=np.ascontiguousarray(om.transpose(0, 2, 1)), threads=8)
    s = r["s"].cpu().numpy()
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-5
    u = r["u"].cpu().double()
    orth = (u.transpose(1, 2) @ u - torch.eye(k + p, dtype=torch.float64)).abs().max()
    assert float(orth) < 1e-4


def test_rsvd_f32_device_omega_vs_oracle():
    """f32 rsvd drawing its own sketch on the device -- numpy's float32 stream, as the reference
    does for float32 input (rsvd.py:65) -- against the oracle (same stream, drawn in C)."""
    B, m, n, k, p = 64, 96, 80, 16, 8
    a64, _ = bf.make_matrix_tensor(B, m, n, 1e5, rank=n, seed=5_200_000)
    a = a64.float()
    r = bf.rsvd_tensor(a, bf.RsvdOptions(k=k, p=p, seed=21), index_base=7)
    o = orc.batch_rsvd_stacked(stack_np(a), m, n, k, p, seed=21, index_base=7, threads=8)
    s = r["s"].cpu().numpy()
    assert s.dtype == np.float32
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-5


def test_rsvd_omega_validation():
    a = torch.randn(4, 32, 24, dtype=torch.float64, device="cuda")
    opts = bf.RsvdOptions(k=4, p=2)
    with pytest.raises(ValueError):
        bf.rsvd_tensor(a, opts, omega=torch.randn(4, 24, 4, dtype=torch.float64, device="cuda"))  # k, not k+p
    with pytest.raises(ValueError):
        bf.rsvd_tensor(a, opts, omega=torch.randn(4, 24, 6, dtype=torch.float64))  # host tensor
    with pytest.raises(ValueError):
        bf.rsvd_tensor(a, opts, omega=torch.randn(4, 24, 6, dtype=torch.float32, device="cuda"))


def test_rsvd_cfg5_batch_vs_oracle():
    B = 64
    a, sig = bf.make_matrix_tensor(B, 128, 128, 1e16, rank=64, seed=5_000_000)
    opts = bf.RsvdOptions(k=32, p=8, seed=5)
    r = bf.rsvd_tensor(a, opts)
    o = orc.batch_rsvd_stacked(stack_np(a), 128, 128, 32, 8, seed=5, threads=8)
    s = r["s"].cpu().numpy()
    for b in range(B):
        assert sigma_normwise(s[b], o["s"][b]) <= 1e-12
    # truncated spectrum recovers the constructed sigma as well as the reference algorithm does
    sg = sig.cpu().numpy()
    eg = np.max(np.abs(s[:, :32] - sg[None, :32]) / sg[None, :32], axis=1)
    eo = np.max(np.abs(o["s"][:, :32] - sg[None, :32]) / sg[None, :32], axis=1)
    assert np.all(eg <= 1.01 * eo + 1e-6)
    assert np.median(eg) < 1e-4


def test_make_matrix_matches_reference():
    g = golden("gauss_testmat")
    a, sig = bf.make_matrix_tensor(1, 128, 128, 1e16, rank=64, seed=5_000_000)
    assert np.array_equal(sig.cpu().numpy(), g["tm/sigma"])
    assert np.max(np.abs(a[0].cpu().numpy() - g["tm/a"])) < 1e-14


def test_rsvd_errors():
    with pytest.raises(ValueError):
        bf.rsvd(np.ones((8, 6)), bf.RsvdOptions(k=5, p=2))


def test_host_pipeline_matches_single_call():
    """Chunked host-buffer pipeline (stream.py) == one device call, bitwise, incl. rsvd seeds."""
    from paper_1707_05141_b200.jacobi import svd_colmajor
    from paper_1707_05141_b200.rsvd import rsvd_colmajor
    from paper_1707_05141_b200.stream import run_host_pipelined

    a = dev_gauss(37, 24, 24, 77_000)
    st = a.transpose(1, 2).contiguous()
    opts = bf.JacobiOptions(ordering="round_robin", accumulate_v=True)
    ref = svd_colmajor(st, 24, 24, opts)
    host_in = st.cpu().pin_memory()
    outs = [torch.empty(ref[k].shape, dtype=ref[k].dtype).pin_memory() for k in ("u", "s", "v", "sweeps")]

    def op(x, ib):
        r = svd_colmajor(x, 24, 24, opts)
        return [r["u"], r["s"], r["v"], r["sweeps"]]

    run_host_pipelined(op, host_in, outs, chunks=5)
    for k, h in zip(("u", "s", "v", "sweeps"), outs):
        assert torch.equal(h, ref[k].cpu()), k
    ro = bf.RsvdOptions(k=4, p=2, seed=11)
    rref = rsvd_colmajor(st, 24, 24, ro, index_base=3)
    outs = [torch.empty(rref["s"].shape, dtype=torch.float64).pin_memory()]
    run_host_pipelined(lambda x, ib: [rsvd_colmajor(x, 24, 24, ro, index_base=ib)["s"]], host_in, outs, chunks=4,
                       index_base=3)
    assert torch.equal(outs[0], rref["s"].cpu())


# ------------------------------------------------------------------ devices= sharding


def test_devices_sharding_is_shard_invariant():
    """devices= cuts each shape group into contiguous pieces, one batched call per device
    (SURVEY §8b); the per-entry results are bitwise those of the single-device call (core.py:97-103),
    including rsvd's seed ^ global index (rsvd.py:82-85). One GPU here: the same device twice."""
    rng = np.random.default_rng(5)
    mats = [rng.standard_normal((24, 16)) for _ in range(7)] + [rng.standard_normal((20, 20)) for _ in range(4)]
    devs = ["cuda:0", "cuda:0", "cuda:0"]
    for fn, kw in ((bf.batch_svd, dict(opts=bf.JacobiOptions(accumulate_v=True))), (bf.batch_qr, {}),
                   (bf.batch_block_svd, dict(opts=bf.BlockJacobiOptions(block_width=4, accumulate_v=True))),
                   (bf.batch_rsvd, dict(opts=bf.RsvdOptions(k=4, p=2, seed=77)))):
        one = fn(mats, **kw)
        many = fn(mats, devices=devs, **kw)
        assert len(one) == len(many)
        for x, y in zip(one, many):
            for f in x.__dataclass_fields__:
                a, b = getattr(x, f), getattr(y, f)
                if isinstance(a, np.ndarray):
                    assert np.array_equal(a, b), (fn.__name__, f)
                else:
                    assert a == b, (fn.__name__, f)
    with pytest.raises(ValueError):
        bf.batch_svd(mats, device="cuda:0", devices=devs)


# ------------------------------------------------------------------ reference helper re-exports


def test_helper_reexports_vs_oracle():
    """householder_vector, jacobi_rotation, off_orthogonality, scaled_offdiag, syrk, gemm and
    frobenius (the names batchfact exports, __init__.py:3-23, + blockjacobi.scaled_offdiag) run on
    the device and agree with the oracle's restatements / the reference's formulas."""
    from paper_1707_05141_b200.blockjacobi import scaled_offdiag

    rng = np.random.default_rng(3)
    eps = np.finfo(np.float64).eps
    for x in (rng.standard_normal(17), np.array([2.0]), np.array([3.0, 0.0, 0.0]), rng.standard_normal(64) * 1e-200):
        v, tau = bf.householder_vector(x)
        vo, to = orc.householder(x)
        assert v.dtype == x.dtype and v[0] == 1.0
        assert abs(tau - to) <= 4 * eps * max(abs(to), 1.0)
        assert np.allclose(v, vo, rtol=8 * eps, atol=0)
    v32, t32 = bf.householder_vector(rng.standard_normal(9).astype(np.float32))
    assert v32.dtype == np.float32
    with pytest.raises(ValueError):
        bf.householder_vector(np.zeros((2, 2)))
    for g in ((2.0, 0.5, 1.0), (1.0, 0.0, 3.0), (1.0, 1e-300, 1.0 + 1e-15), (5.0, -2.0, 5.0), (1e200, 1e199, 3e200)):
        c, s = bf.jacobi_rotation(*g)
        co, so = orc.rotation(*g)
        assert abs(c - co) <= 2 * eps and abs(s - so) <= 2 * eps * max(abs(so), 1e-300)
    a = rng.standard_normal((30, 12))
    a[:, 3] = 0.0
    assert abs(bf.off_orthogonality(a) - orc.off_orthogonality(a)) <= 64 * eps
    assert bf.off_orthogonality(a[:, :1]) == 0.0
    g = a.T @ a
    assert abs(scaled_offdiag(g) - orc.scaled_offdiag(g)) <= 64 * eps
    z = np.array([[0.0, 1.0], [1.0, 1.0]])
    assert scaled_offdiag(z) == np.inf and bf.scaled_offdiag(np.zeros((2, 2))) == 0.0
    with pytest.raises(ValueError):
        scaled_offdiag(np.ones((2, 3)))
    gs = bf.syrk(a)
    assert np.array_equal(gs, gs.T) and np.allclose(gs, orc.syrk(a), rtol=0, atol=64 * eps * np.abs(gs).max())
    b = rng.standard_normal((12, 7))
    cc = rng.standard_normal((30, 7))
    assert np.allclose(bf.gemm(a, b), a @ b, atol=1e-13)
    assert np.allclose(bf.gemm(a, b, cc, alpha=2.0, beta=-0.5), 2.0 * (a @ b) - 0.5 * cc, atol=1e-13)
    assert np.allclose(bf.gemm(b, a, trans_a=True, trans_b=True), b.T @ a.T, atol=1e-13)
    nan_c = np.full((30, 7), np.nan)
    assert np.all(np.isfinite(bf.gemm(a, b, nan_c, beta=0.0)))  # beta == 0 ignores c (core.py:37-40)
    assert np.all(bf.gemm(a, b, alpha=0.0) == 0.0)
    with pytest.raises(ValueError):
        bf.gemm(a, a)
    with pytest.raises(ValueError):
        bf.gemm(a, b, beta=1.0)
    assert abs(bf.frobenius(a) - np.linalg.norm(a)) <= 8 * eps * np.linalg.norm(a)
    assert bf.frobenius(np.zeros((0, 3))) == 0.0
    assert bf.frobenius(np.array([[1e300, 1e300]])) == pytest.approx(np.sqrt(2) * 1e300, rel=1e-15)


def test_rr_log_chunking_is_invisible():
    """With V the round-robin tier logs rotations per matrix, sized for max_sweeps; a call whose
    logs exceed the per-launch budget (svd_rr.cu kRRLogBudget) runs in chunks of whole CTA waves.
    max_sweeps = 300 forces 3 chunks for 1 300 64x64 matrices; every matrix converges far below 30
    sweeps, so the result must equal the unchunked max_sweeps = 30 call bit for bit."""
    a = dev_gauss(1300, 64, 64, 3_100_000)
    r30 = bf.svd_tensor(a, bf.JacobiOptions(ordering="round_robin", accumulate_v=True, max_sweeps=30))
    r300 = bf.svd_tensor(a, bf.JacobiOptions(ordering="round_robin", accumulate_v=True, max_sweeps=300))
    assert bool(torch.all(r30["converged"])) and int(r30["sweeps"].max()) < 30
    for k in ("u", "sigma", "v", "sweeps", "converged"):
        assert torch.equal(r30[k], r300[k]), k


@pytest.mark.parametrize("entry", ["svd", "qr", "block", "rsvd"])
def test_dropin_input_layouts_identical(entry):
    """The drop-in batch calls stage C-ordered, Fortran-ordered, strided and mixed entry lists
    differently (core.stack_to_device: host stack + device transpose / plain stack / per-entry);
    the results must be bitwise identical, and the inputs untouched (core.py:26-33)."""
    rng = np.random.default_rng(21)
    m, n = (96, 64) if entry != "block" else (128, 96)
    base = [rng.standard_normal((m, n)) for _ in range(6)]
    layouts = {
        "c": [np.ascontiguousarray(a) for a in base],
        "f": [np.asfortranarray(a) for a in base],
        "strided": [np.repeat(a, 2, axis=1)[:, ::2] for a in base],
        "mixed": [np.asfortranarray(a) if i % 2 else np.ascontiguousarray(a) for i, a in enumerate(base)],
    }
    keep = [a.copy() for a in layouts["c"]]

    def run(batch):
        if entry == "svd":
            return [(r.u, r.sigma, r.v) for r in bf.batch_svd(batch, bf.JacobiOptions(accumulate_v=True))]
        if entry == "qr":
            return [(r.q, r.r) for r in bf.batch_qr(batch)]
        if entry == "block":
            return [(r.u, r.sigma, r.v) for r in
                    bf.batch_block_svd(batch, bf.BlockJacobiOptions(block_width=16, accumulate_v=True))]
        return [(r.u, r.s, r.v) for r in bf.batch_rsvd(batch, bf.RsvdOptions(k=8, p=4, seed=3))]

    ref = run(layouts["c"])
    for name, batch in layouts.items():
        got = run(batch)
        for x, y in zip(ref, got):
            for p, q in zip(x, y):
                assert np.array_equal(p, q), name
    for a, b in zip(layouts["c"], keep):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("entry", ["svd", "qr", "rsvd", "block"])
@pytest.mark.parametrize("order", ["c", "f"])
def test_dropin_pipelined_matches_tensor_api(entry, order):
    """Large drop-in groups run the chunked host pipeline (stream.run_entries_pipelined: host
    staging, H2D, kernels and D2H overlapped); results bitwise equal to one tensor-API call."""
    B, m, n = (1100, 64, 48) if entry != "block" else (1030, 72, 64)
    a = dev_gauss(B, m, n, 7_700_000 + m)
    host = a.cpu().numpy()
    ents = [np.ascontiguousarray(x) if order == "c" else np.asfortranarray(x) for x in host]
    if entry == "svd":
        opts = bf.JacobiOptions(ordering="round_robin", accumulate_v=True)
        got = bf.batch_svd(ents, opts)
        r = bf.svd_tensor(a, opts)
        pairs = [("u", "u"), ("sigma", "sigma"), ("v", "v")]
    elif entry == "qr":
        got = bf.batch_qr(ents)
        q, rr = bf.qr_tensor(a)
        r = {"q": q, "r": rr}
        pairs = [("q", "q"), ("r", "r")]
    elif entry == "block":
        opts = bf.BlockJacobiOptions(block_width=16, accumulate_v=True, max_sweeps=4)
        got = bf.batch_block_svd(ents, opts)
        r = bf.block_svd_tensor(a, opts)
        pairs = [("u", "u"), ("sigma", "sigma"), ("v", "v")]
    else:
        opts = bf.RsvdOptions(k=8, p=4, seed=11)
        got = bf.batch_rsvd(ents, opts)
        r = bf.rsvd_tensor(a, opts)
        pairs = [("u", "u"), ("s", "s"), ("v", "v")]
    for attr, key in pairs:
        ref = r[key].cpu().numpy()
        for i in (0, 1, B // 2, B - 1):
            assert np.array_equal(getattr(got[i], attr), ref[i]), (attr, i)
