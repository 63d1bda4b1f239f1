"""H^2 compression driver: construction and matvec on the host, the batched
GPU compression against the per-node CPU oracle (oracle/h2_ref.py), and the SPEC.md examples."""

import math

import numpy as np
import pytest
import torch

from paper_1707_05141_b200 import h2
from oracle import h2_ref


@pytest.fixture(scope="module")
def fix1024():
    pts = h2.perturbed_grid(1024, seed=1)
    return pts, h2.build_h2(pts, 0.1, 8, 1.0, 64)


# ------------------------------------------------------------------ SPEC examples (host)


def test_exp_kernel_examples():
    p = np.array([0.3, 0.4])
    assert h2.exp_kernel(p, p, 0.1) == 1.0
    q = p + np.array([0.06, 0.08])  # distance 0.1 = ell
    assert abs(h2.exp_kernel(p, q, 0.1) - math.exp(-1.0)) < 1e-15
    vals = [h2.exp_kernel(p, p + np.array([d, 0.0]), 0.1) for d in (0.1, 0.5, 1.0, 5.0)]
    assert all(a > b for a, b in zip(vals, vals[1:])) and vals[-1] < 1e-20
    with pytest.raises(ValueError):
        h2.exp_kernel(p, q, 0.0)


def test_chebyshev_grid_examples():
    assert np.array_equal(h2.chebyshev_grid(1), [0.0])
    np.testing.assert_allclose(h2.chebyshev_grid(3), [math.sqrt(3) / 2, 0.0, -math.sqrt(3) / 2], atol=1e-15)
    g = h2.chebyshev_grid(8)
    assert len(set(g)) == 8 and np.all(np.abs(g) < 1) and np.allclose(g, -g[::-1], atol=1e-15)


def test_cluster_tree_examples():
    t = h2.build_cluster_tree(h2.perturbed_grid(64, seed=0), 64)
    assert t.num_nodes == 1 and t.is_leaf(0)
    g = np.array([(i, j) for j in range(4) for i in range(4)], dtype=float)
    t = h2.build_cluster_tree(g, 4)
    assert t.depth() == 2 and len(t.leaves()) == 4
    assert all(t.hi[i] - t.lo[i] == 4 for i in t.leaves())
    # each leaf of the regular grid is a 2x2 quadrant (mean splits are midlines)
    for i in t.leaves():
        q = t.points[t.lo[i] : t.hi[i]]
        assert np.ptp(q[:, 0]) == 1 and np.ptp(q[:, 1]) == 1
    same = np.full((100, 2), 0.5)
    t = h2.build_cluster_tree(same, 8)
    assert all(t.hi[i] - t.lo[i] <= 8 for i in t.leaves())


def test_cluster_tree_invariants(fix1024):
    _, H = fix1024
    t = H.tree
    assert sorted(t.perm.tolist()) == list(range(t.n))
    for i in range(t.num_nodes):
        q = t.points[t.lo[i] : t.hi[i]]
        b = t.box[i]
        assert q[:, 0].min() >= b[0] and q[:, 0].max() <= b[1] and q[:, 1].min() >= b[2] and q[:, 1].max() <= b[3]
        if t.is_leaf(i):
            assert t.hi[i] - t.lo[i] <= t.leaf_size
        else:
            c0, c1 = t.children[i]
            assert t.lo[c0] == t.lo[i] and t.hi[c0] == t.lo[c1] and t.hi[c1] == t.hi[i]


def test_single_dense_root_exact():
    pts = h2.perturbed_grid(50, seed=2)
    H = h2.build_h2(pts, 0.1, 4, 1.0, 64)
    assert len(H.dense["t"]) == 1 and not H.coupling
    x = np.random.default_rng(0).standard_normal(50)
    y = h2.h2_matvec(H.to(), torch.as_tensor(x)).numpy()
    np.testing.assert_allclose(y, h2_ref.dense_kernel(pts, 0.1) @ x, rtol=0, atol=1e-14)
    assert np.all(h2.h2_matvec(H.to(), torch.zeros(50)).numpy() == 0)
    m = h2.memory_report(H)
    assert m["dense"] == 50 * 50 * 8 and m["lowrank"] == 50 * 16 * 8  # one leaf basis, no coupling


def test_memory_single_leaf_example():
    H = h2.build_h2(h2.perturbed_grid(64, seed=3), 0.1, 8, 1.0, 64)
    assert h2.memory_report(H)["dense"] == 64 * 64 * 8 == 32768


def test_matvec_matches_dense_and_oracle(fix1024):
    pts, H = fix1024
    x = np.random.default_rng(1).standard_normal((1024, 3))
    A = h2_ref.dense_kernel(pts, 0.1)
    y = h2.h2_matvec(H.to(), torch.as_tensor(x)).numpy()
    assert np.linalg.norm(y - A @ x) / np.linalg.norm(A @ x) <= 1e-7
    yr = h2_ref.matvec_ref(H, x)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) <= 1e-14


def test_dense_assembly_matches_kernel(fix1024):
    pts, H = fix1024
    A_h = h2.dense_assembly(H.to()).numpy()
    A = h2_ref.dense_kernel(pts, 0.1)
    assert np.linalg.norm(A - A_h) / np.linalg.norm(A) <= 1e-7


def test_lowrank_blocks_accurate(fix1024):
    """Every admissible block to 1e-6; well-separated ones (diam <= dist / 2) to 1e-7."""
    pts, H = fix1024
    tree = H.tree
    seen = 0
    for g in H.coupling.values():
        for b in range(0, len(g["t"]), 7):
            t, s = g["t"][b], g["s"][b]
            blk = h2.kernel_block(tree.points[tree.lo[t] : tree.hi[t]], tree.points[tree.lo[s] : tree.hi[s]], 0.1)
            approx = h2.explicit_basis(H, t) @ g["S"][b] @ h2.explicit_basis(H, s).T
            err = np.linalg.norm(blk - approx) / np.linalg.norm(blk)
            assert err <= 1e-6
            if h2.admissible(tree.box[t], tree.box[s], 0.5):
                assert err <= 1e-7
                seen += 1
    assert seen > 0


def test_nested_basis_identity(fix1024):
    _, H = fix1024
    tree = H.tree
    for i in range(tree.num_nodes):
        if tree.is_leaf(i):
            continue
        B = h2.explicit_basis(H, i)
        direct = h2.lagrange_2d(tree.box[i], H.order, tree.points[tree.lo[i] : tree.hi[i]])
        assert np.abs(B - direct).max() <= 1e-12


def test_oracle_compress_error_and_memory():
    pts = h2.perturbed_grid(6000, seed=1)
    H = h2.build_h2(pts, 0.1, 8, 1.0, 64)
    Hc, k = h2_ref.compress_ref(H, 1e-7)
    assert k[-1] < H.ranks[-1]  # ragged leaves compress (leaves with < 64 points)
    assert h2.estimate_error(H.to(), Hc.to()) <= 1e-7
    m0, m1 = h2.memory_report(H), h2.memory_report(Hc)
    assert m1["lowrank"] < m0["lowrank"] and m1["dense"] == m0["dense"]


def _constructed_single_leaf():
    """One leaf, order 2 (rank 4) with leaf basis of spectrum (1, 1e-9, 1e-10, 1e-11)."""
    H = h2.build_h2(h2.perturbed_grid(4, seed=4), 0.1, 2, 1.0, 64)
    rng = np.random.default_rng(0)
    q1, _ = np.linalg.qr(rng.standard_normal((4, 4)))
    q2, _ = np.linalg.qr(rng.standard_normal((4, 4)))
    H.leaf_U[0] = (q1 @ np.diag([1, 1e-9, 1e-10, 1e-11]) @ q2.T)[None]
    return H


def test_oracle_constructed_spectrum_rank1():
    _, k = h2_ref.compress_ref(_constructed_single_leaf(), 1e-7)
    assert k == [1]


def test_compress_cli_usage(tmp_path):
    from paper_1707_05141_b200 import cli

    assert cli.main(["compress", "--n", "0"]) == 1


# ------------------------------------------------------------------ GPU compression vs oracle


def _cuda(H):
    return H.to("cuda")


def _compare(Hc_gpu, Hc_ref, n, tol=1e-12):
    x = np.random.default_rng(5).standard_normal((n, 4))
    y = h2.h2_matvec(Hc_gpu, torch.as_tensor(x)).cpu().numpy()
    yr = h2_ref.matvec_ref(Hc_ref, x)
    return np.linalg.norm(y - yr) / np.linalg.norm(yr)


@pytest.mark.gpu
def test_bmm_matches_torch():
    g = torch.Generator(device="cuda").manual_seed(0)
    for B, M, N, K in ((7, 64, 64, 64), (5, 30, 121, 64), (3, 128, 40, 17), (4, 1, 1, 1)):
        a = torch.randn(B, M, K, device="cuda", dtype=torch.float64, generator=g)
        b = torch.randn(B, K, N, device="cuda", dtype=torch.float64, generator=g)
        ref = a @ b
        assert (h2.bmm(a, b) - ref).abs().max() <= 1e-12 * K
        assert (h2.bmm(a.transpose(1, 2).contiguous(), b, ta=True) - ref).abs().max() <= 1e-12 * K
        assert (h2.bmm(a, b.transpose(1, 2).contiguous(), tb=True) - ref).abs().max() <= 1e-12 * K
        af, bf_ = a.float(), b.float()
        assert (h2.bmm(af, bf_) - ref).abs().max() <= 1e-4 * K


@pytest.mark.gpu
@pytest.mark.parametrize("n,order,eta", [(1024, 8, 1.0), (6000, 8, 1.0), (2500, 11, 2.0)])
def test_compress_matches_oracle(n, order, eta):
    pts = h2.perturbed_grid(n, seed=1)
    H = h2.build_h2(pts, 0.1, order, eta, 64)
    Hc, rep = h2.compress(_cuda(H), 1e-7)
    Hr, k = h2_ref.compress_ref(H, 1e-7)
    assert rep["ranks_after"] == k
    assert _compare(Hc, Hr, n) <= 1e-12
    assert h2.estimate_error(_cuda(H), Hc) <= 1e-7
    m0, m1 = h2.memory_report(H), h2.memory_report(Hc)
    assert m1["dense"] == m0["dense"] and m1["lowrank"] <= m0["lowrank"]
    if k != H.ranks:
        assert m1["lowrank"] < m0["lowrank"]


@pytest.mark.gpu
def test_compressed_basis_nested_and_orthonormal():
    H = h2.build_h2(h2.perturbed_grid(2500, seed=1), 0.1, 11, 2.0, 64)
    Hc, _ = h2.compress(_cuda(H), 1e-7)
    tree = Hc.tree
    for i in range(tree.num_nodes):
        B = h2.explicit_basis(Hc, i)
        G = B.T @ B
        nz = np.abs(np.diag(G)) > 0.5  # zero-padded columns are exactly zero
        assert np.abs(G[np.ix_(nz, nz)] - np.eye(nz.sum())).max() <= 1e-12
        assert np.all(B[:, ~nz] == 0)


@pytest.mark.gpu
def test_compress_constructed_spectrum_rank1():
    Hc, rep = h2.compress(_cuda(_constructed_single_leaf()), 1e-7)
    assert rep["ranks_after"] == [1]


@pytest.mark.gpu
def test_compress_idempotent_and_machine_eps():
    H = h2.build_h2(h2.perturbed_grid(6000, seed=1), 0.1, 8, 1.0, 64)
    Hc, rep = h2.compress(_cuda(H), 1e-7)
    Hcc, rep2 = h2.compress(Hc, 1e-7)
    assert rep2["ranks_after"] == rep["ranks_after"]
    assert h2.estimate_error(Hc, Hcc) <= 1e-12
    _, rep3 = h2.compress(_cuda(H), np.finfo(np.float64).eps)
    assert rep3["ranks_after"] == H.ranks or rep3["ranks_after"] == rep["ranks_after"]


@pytest.mark.gpu
def test_projection_identity_is_bitwise():
    H = _cuda(h2.build_h2(h2.perturbed_grid(2000, seed=1), 0.1, 8, 1.0, 64))
    st = h2._level_struct(H)
    T = [torch.eye(H.ranks[l], dtype=torch.float64, device="cuda").expand(st["nnodes"][l], -1, -1).contiguous()
         for l in range(H.tree.num_levels)]
    out = h2.project_coupling(H, T)
    for key, g in H.coupling.items():
        assert torch.equal(out[key]["S"], g["S"])


@pytest.mark.gpu
def test_rsvd_truncation_matches_full_ranks():
    H = h2.build_h2(h2.perturbed_grid(2500, seed=1), 0.1, 11, 2.0, 64)
    _, full = h2.compress(_cuda(H), 1e-7)
    # leaf level: rank 121 -> <= 64; a 64-sample budget covers the post-truncation rank
    Hc, rs = h2.compress(_cuda(H), 1e-7, h2.SvdChoice(kind="rsvd", samples=121, oversample=8))
    assert rs["ranks_after"] == full["ranks_after"]
    assert h2.estimate_error(_cuda(H), Hc) <= 1e-7


@pytest.mark.gpu
def test_compress_f32():
    H = h2.build_h2(h2.perturbed_grid(2500, seed=1), 0.1, 11, 2.0, 64)
    Hc, rep = h2.compress(H.to("cuda", torch.float32), 1e-5)
    assert rep["ranks_after"][-1] <= 64
    assert h2.estimate_error(_cuda(H), Hc) <= 1e-5


@pytest.mark.gpu
def test_compress_cli(tmp_path):
    import json

    from paper_1707_05141_b200 import cli

    out = tmp_path / "r.json"
    rc = cli.main(["compress", "--n", "2500", "--cheb-order", "11", "--eta", "2", "--report", str(out)])
    assert rc == 0
    rec = json.loads(out.read_text().splitlines()[-1])
    assert rec["ranks_after"][-1] <= 64 and rec["error_estimate"] <= 1e-7
    assert rec["memory_after"]["dense"] == rec["memory_before"]["dense"]


@pytest.mark.gpu
def test_projection_tree_norm_on_orthonormal_basis():
    """||T||_2 <= 1 + 1e-12 when T projects an orthonormal basis (a compressed H)."""
    H = h2.build_h2(h2.perturbed_grid(2500, seed=1), 0.1, 11, 2.0, 64)
    Hc, _ = h2.compress(_cuda(H), 1e-7)
    _, _, _, T, _ = h2.truncate_basis(Hc, 1e-7)
    for t in T:
        if t is not None and t.numel():
            assert float(torch.linalg.matrix_norm(t.double().cpu(), ord=2).max()) <= 1 + 1e-12


def test_degenerate_points_build_and_matvec():
    """All points identical (SPEC.md:554 ledger): the tree halves by index, nothing is
    admissible, the operator is the exact dense kernel (all ones)."""
    pts = np.full((300, 2), 0.25)
    H = h2.build_h2(pts, 0.1, 4, 1.0, 64)
    assert not H.coupling and all(H.tree.hi[i] - H.tree.lo[i] <= 64 for i in H.tree.leaves())
    x = np.random.default_rng(2).standard_normal(300)
    y = h2.h2_matvec(H.to(), torch.as_tensor(x)).numpy()
    np.testing.assert_allclose(y, np.full(300, x.sum()), rtol=1e-12, atol=1e-12)
