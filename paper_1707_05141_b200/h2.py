"""H^2-matrix compression driver: the batched SVD's real caller.

The reference declares the H^2 module (the CLI ``compress`` of SPEC.md:573-614)
but ships no code for it (its package, /root/reference/pkg/src/batchfact, stops at the batched
factorisations), so this module follows the specification:

  * construction (host, numpy): perturbed-grid points, KD-tree with mean split
    (SPEC.md:468-474), tensor Chebyshev interpolation bases and transfer matrices
    (SPEC.md:475-486), dual traversal with the max-diameter admissibility;
  * compression (device): level by level, bottom-up, ONE batched Jacobi SVD (or batched
    randomized SVD) per level over all of the level's nodes -- leaf bases U and the stacked
    [T_c1 E_c1; T_c2 E_c2] of inner nodes (§8.2) -- then the
    per-level-pair batched projections S~ = T_t S T_s^T. The SVDs are the
    library's register/shared tiers (bf_svd_batched_*, bf_rsvd_batched_*), the products are
    bf_gemm_batched_* (FP64 tensor cores);
  * matvec (device or host torch; verification plumbing), the 30-vector
    error estimator and the memory report.

Layout. Everything is grouped per tree level so a level is one batch: ``leaf_U[l]`` is
(leaves at l, leaf_rows, k_l) with zero rows past each leaf's point count; ``transfer[l]`` is
(nodes at l, k_l, k_{l-1}) in the level's node order (E_c of U_parent = [U_c1 E_c1; U_c2 E_c2]);
``coupling[(lt, ls)]`` holds the (blocks, k_lt, k_ls) coupling matrices of the low-rank leaves
whose row/column clusters sit at levels lt/ls; ``dense`` the (blocks, leaf_rows, leaf_rows)
near-field blocks. Ranks are uniform per level: after truncation the level rank is
the level's maximum and nodes below it carry zero columns.
"""

import math
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import ptr, resolve_device, stream_handle

# ---------------------------------------------------------------- kernel, points, Chebyshev


def exp_kernel(p, q, ell):
    """exp(-||p - q||_2 / ell), broadcasting over leading dims of (…, 2) arrays."""
    if not ell > 0:
        raise ValueError("ell must be > 0")
    d = np.asarray(p, dtype=np.float64) - np.asarray(q, dtype=np.float64)
    return np.exp(-np.sqrt(np.sum(d * d, axis=-1)) / ell)


def kernel_block(P, Q, ell):
    """K(P_i, Q_j) for point arrays P (..., m, 2), Q (..., n, 2) -> (..., m, n)."""
    dx = P[..., :, None, 0] - Q[..., None, :, 0]
    dy = P[..., :, None, 1] - Q[..., None, :, 1]
    return np.exp(-np.sqrt(dx * dx + dy * dy) / ell)


def chebyshev_grid(order):
    """The ``order`` Chebyshev points cos(pi (2i+1) / (2 order)) on [-1, 1]."""
    if order < 1:
        raise ValueError("order must be >= 1")
    i = np.arange(order, dtype=np.float64)
    x = np.cos(np.pi * (2.0 * i + 1.0) / (2.0 * order))
    x[np.abs(x) < 1e-15] = 0.0  # cos(pi/2) is 6e-17 in floating point
    return x


def perturbed_grid(n, seed=0, amplitude=0.25):
    """n points of a regular nx x ny grid on the unit square (cell centres), each moved by a
    uniform +-amplitude grid spacing per axis ("random perturbation of a regular
    discretization"). nx = ceil(sqrt(n)), rows filled in order, so n need not be a square."""
    if n < 1:
        raise ValueError("n must be >= 1")
    nx = int(math.ceil(math.sqrt(n)))
    ny = int(math.ceil(n / nx))
    rng = np.random.default_rng(seed)
    j, i = np.divmod(np.arange(n), nx)
    hx, hy = 1.0 / nx, 1.0 / ny
    pert = rng.uniform(-amplitude, amplitude, size=(n, 2))
    return np.stack([(i + 0.5 + pert[:, 0]) * hx, (j + 0.5 + pert[:, 1]) * hy], axis=1)


def lagrange_1d(nodes, t):
    """(len(t), len(nodes)) Lagrange polynomials of ``nodes`` evaluated at ``t``."""
    nodes = np.asarray(nodes, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    out = np.ones(t.shape + (len(nodes),))
    for j in range(len(nodes)):
        for m in range(len(nodes)):
            if m != j:
                out[..., j] *= (t - nodes[m]) / (nodes[j] - nodes[m])
    return out


# ---------------------------------------------------------------- cluster tree


@dataclass
class ClusterTree:
    """Binary KD-tree over point index ranges. Nodes are numbered breadth-first,
    so each level is a contiguous id range; ``perm[k]`` is the original index of tree-ordered point k."""

    points: np.ndarray  # (n, 2) in tree order
    perm: np.ndarray  # (n,)
    lo: np.ndarray
    hi: np.ndarray
    box: np.ndarray  # (nodes, 4): xmin, xmax, ymin, ymax (tight)
    parent: np.ndarray
    children: np.ndarray  # (nodes, 2), -1 for leaves
    level: np.ndarray
    leaf_size: int

    @property
    def n(self):
        return len(self.perm)

    @property
    def num_nodes(self):
        return len(self.lo)

    @property
    def num_levels(self):
        return int(self.level.max()) + 1

    def is_leaf(self, i):
        return self.children[i, 0] < 0

    def level_nodes(self, l):
        return np.nonzero(self.level == l)[0]

    def pos_in_level(self):
        """pos[i] = index of node i inside its level's node list."""
        pos = np.empty(self.num_nodes, dtype=np.int64)
        for l in range(self.num_levels):
            ids = self.level_nodes(l)
            pos[ids] = np.arange(len(ids))
        return pos

    def leaves(self):
        return np.nonzero(self.children[:, 0] < 0)[0]

    def depth(self):
        return self.num_levels - 1


def build_cluster_tree(points, leaf_size):
    """KD-tree with a mean split along the wider bounding-box axis.

    Degenerate clusters: a mean split that leaves one side empty falls back to a
    median split (by stable sort order); a cluster of identical points is halved by index."""
    if leaf_size < 1:
        raise ValueError("leaf_size must be >= 1")
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 2 or len(pts) == 0:
        raise ValueError("points must be a non-empty (n, 2) array")
    if not np.all(np.isfinite(pts)):
        raise ValueError("point coordinates must be finite")
    n = len(pts)
    perm = np.arange(n)
    lo, hi, parent, level, children = [0], [n], [-1], [0], [[-1, -1]]
    queue = deque([0])
    while queue:
        i = queue.popleft()
        a, b = lo[i], hi[i]
        if b - a <= leaf_size:
            continue
        idx = perm[a:b]
        p = pts[idx]
        ext = p.max(axis=0) - p.min(axis=0)
        ax = 0 if ext[0] >= ext[1] else 1
        c = p[:, ax]
        left = c < c.mean()
        if left.all() or not left.any():
            left = np.zeros(b - a, dtype=bool)
            if ext.max() == 0.0:
                left[: (b - a) // 2] = True
            else:
                left[np.argsort(c, kind="stable")[: (b - a) // 2]] = True
        perm[a:b] = np.concatenate([idx[left], idx[~left]])
        mid = a + int(left.sum())
        kids = []
        for x, y in ((a, mid), (mid, b)):
            kids.append(len(lo))
            lo.append(x)
            hi.append(y)
            parent.append(i)
            level.append(level[i] + 1)
            children.append([-1, -1])
            queue.append(kids[-1])
        children[i] = kids
    tp = pts[perm]
    lo_a, hi_a = np.array(lo, dtype=np.int64), np.array(hi, dtype=np.int64)
    box = np.empty((len(lo), 4))
    for i in range(len(lo)):
        q = tp[lo_a[i] : hi_a[i]]
        box[i] = (q[:, 0].min(), q[:, 0].max(), q[:, 1].min(), q[:, 1].max())
    return ClusterTree(
        points=tp,
        perm=perm,
        lo=lo_a,
        hi=hi_a,
        box=box,
        parent=np.array(parent, dtype=np.int64),
        children=np.array(children, dtype=np.int64),
        level=np.array(level, dtype=np.int64),
        leaf_size=int(leaf_size),
    )


def box_diameter(box):
    return np.hypot(box[..., 1] - box[..., 0], box[..., 3] - box[..., 2])


def box_distance(b1, b2):
    dx = np.maximum(0.0, np.maximum(b1[..., 0] - b2[..., 1], b2[..., 0] - b1[..., 1]))
    dy = np.maximum(0.0, np.maximum(b1[..., 2] - b2[..., 3], b2[..., 2] - b1[..., 3]))
    return np.hypot(dx, dy)


def admissible(b1, b2, eta):
    """max(diam t, diam s) <= eta * dist(t, s), bounding boxes, dist > 0."""
    dist = box_distance(b1, b2)
    return bool(dist > 0.0 and max(box_diameter(b1), box_diameter(b2)) <= eta * dist)


def dual_traversal(tree, eta):
    """Matrix tree leaves from the dual traversal of (root, root): admissible pairs
    become LOWRANK, pairs of leaves DENSE; otherwise the non-leaf side(s) split. Returns
    (lowrank [(t, s)], dense [(t, s)]), each sorted."""
    low, dense = [], []
    stack = [(0, 0)]
    while stack:
        t, s = stack.pop()
        if admissible(tree.box[t], tree.box[s], eta):
            low.append((t, s))
            continue
        lt, ls = tree.is_leaf(t), tree.is_leaf(s)
        if lt and ls:
            dense.append((t, s))
        elif lt:
            stack.extend((t, c) for c in tree.children[s])
        elif ls:
            stack.extend((c, s) for c in tree.children[t])
        else:
            stack.extend((c, d) for c in tree.children[t] for d in tree.children[s])
    return sorted(low), sorted(dense)


# ---------------------------------------------------------------- interpolation bases


def _box_map(box):
    """Centre and half-width per axis; degenerate widths get a tiny positive half-width."""
    box = np.asarray(box, dtype=np.float64)
    cx, cy = 0.5 * (box[..., 0] + box[..., 1]), 0.5 * (box[..., 2] + box[..., 3])
    hx, hy = 0.5 * (box[..., 1] - box[..., 0]), 0.5 * (box[..., 3] - box[..., 2])
    tiny = 1e-12
    hx = np.where(hx > tiny * np.maximum(1.0, np.abs(cx)), hx, tiny * np.maximum(1.0, np.abs(cx)))
    hy = np.where(hy > tiny * np.maximum(1.0, np.abs(cy)), hy, tiny * np.maximum(1.0, np.abs(cy)))
    return cx, cy, hx, hy


def interp_points(box, order):
    """(order^2, 2) tensor Chebyshev grid on ``box``; index b = jx * order + jy."""
    c = chebyshev_grid(order)
    cx, cy, hx, hy = _box_map(box)
    gx, gy = np.meshgrid(cx + hx * c, cy + hy * c, indexing="ij")
    return np.stack([gx.ravel(), gy.ravel()], axis=1)


def lagrange_2d(box, order, pts):
    """(len(pts), order^2) tensor Lagrange polynomials of ``box``'s grid at ``pts``."""
    c = chebyshev_grid(order)
    cx, cy, hx, hy = _box_map(box)
    lx = lagrange_1d(c, (pts[:, 0] - cx) / hx)
    ly = lagrange_1d(c, (pts[:, 1] - cy) / hy)
    return (lx[:, :, None] * ly[:, None, :]).reshape(len(pts), order * order)


# ---------------------------------------------------------------- H^2 matrix


@dataclass
class H2Matrix:
    """Symmetric H^2 matrix (V = U). Arrays are numpy (host) or torch (device)."""

    tree: ClusterTree
    ell: float
    order: int
    eta: float
    ranks: list  # k_l per level
    leaf_U: list  # per level: (leaves at l, leaf_rows, k_l) or None
    transfer: list  # per level: (nodes at l, k_l, k_{l-1}); None at level 0
    coupling: dict  # (lt, ls) -> dict(t=ids, s=ids, S=(blocks, k_lt, k_ls))
    dense: dict  # dict(t=ids, s=ids, D=(blocks, rows, rows))
    meta: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.tree.n

    @property
    def leaf_rows(self):
        return self.meta["leaf_rows"]

    def arrays_on(self):
        a = self.dense["D"]
        return a.device if isinstance(a, torch.Tensor) else None

    def to(self, device=None, dtype=torch.float64):
        """Copy every array to a torch device (``dtype`` float64 or float32)."""
        dev = torch.device(device) if device is not None else None

        def conv(x):
            if x is None:
                return None
            if isinstance(x, np.ndarray) and x.dtype.kind == "f":
                return torch.as_tensor(x).to(device=dev, dtype=dtype)
            if isinstance(x, torch.Tensor) and x.is_floating_point():
                return x.to(device=dev, dtype=dtype)
            return x

        return H2Matrix(
            tree=self.tree,
            ell=self.ell,
            order=self.order,
            eta=self.eta,
            ranks=list(self.ranks),
            leaf_U=[conv(u) for u in self.leaf_U],
            transfer=[conv(e) for e in self.transfer],
            coupling={k: dict(t=g["t"], s=g["s"], S=conv(g["S"])) for k, g in self.coupling.items()},
            dense=dict(t=self.dense["t"], s=self.dense["s"], D=conv(self.dense["D"])),
            meta=dict(self.meta),
        )

    def numpy(self):
        """Host float64 numpy copy (for the oracle)."""

        def conv(x):
            if isinstance(x, torch.Tensor):
                return x.detach().to("cpu", torch.float64).numpy()
            return x

        return H2Matrix(
            tree=self.tree,
            ell=self.ell,
            order=self.order,
            eta=self.eta,
            ranks=list(self.ranks),
            leaf_U=[conv(u) for u in self.leaf_U],
            transfer=[conv(e) for e in self.transfer],
            coupling={k: dict(t=g["t"], s=g["s"], S=conv(g["S"])) for k, g in self.coupling.items()},
            dense=dict(t=self.dense["t"], s=self.dense["s"], D=conv(self.dense["D"])),
            meta=dict(self.meta),
        )


def _leaf_index(tree, rows):
    """(nodes, rows) tree-order point indices of each leaf, padded with n (a zero row)."""
    idx = np.full((tree.num_nodes, rows), tree.n, dtype=np.int64)
    for i in tree.leaves():
        m = tree.hi[i] - tree.lo[i]
        idx[i, :m] = np.arange(tree.lo[i], tree.hi[i])
    return idx


def build_h2(points, ell=0.1, cheb_order=8, eta=1.0, leaf_size=64, *, chunk=2048):
    """Chebyshev-interpolation H^2 matrix of the exponential kernel.

    Leaf U = Lagrange-Chebyshev polynomials of the leaf's bounding box at its points; transfer
    E_c = the parent's polynomials at the child's grid points; LOWRANK coupling S = kernel at
    (row grid x column grid); DENSE leaves = exact kernel evaluation. Host (numpy)."""
    if not (ell > 0 and cheb_order >= 1 and eta > 0 and leaf_size >= 1):
        raise ValueError("ell, cheb_order, eta and leaf_size must be positive")
    tree = build_cluster_tree(points, leaf_size)
    r = cheb_order * cheb_order
    L = tree.num_levels
    rows = int(max(tree.hi[i] - tree.lo[i] for i in tree.leaves()))
    pos = tree.pos_in_level()
    grids = np.stack([interp_points(tree.box[i], cheb_order) for i in range(tree.num_nodes)])  # (nodes, r, 2)

    leaf_U, transfer = [], []
    for l in range(L):
        ids = tree.level_nodes(l)
        lv = [i for i in ids if tree.is_leaf(i)]
        if lv:
            U = np.zeros((len(lv), rows, r))
            for j, i in enumerate(lv):
                U[j, : tree.hi[i] - tree.lo[i]] = lagrange_2d(tree.box[i], cheb_order,
                                                              tree.points[tree.lo[i] : tree.hi[i]])
            leaf_U.append(U)
        else:
            leaf_U.append(None)
        if l == 0:
            transfer.append(None)
        else:
            E = np.stack([lagrange_2d(tree.box[tree.parent[i]], cheb_order, grids[i]) for i in ids])
            transfer.append(E)

    low, dense = dual_traversal(tree, eta)
    coupling = {}
    groups = {}
    for t, s in low:
        groups.setdefault((int(tree.level[t]), int(tree.level[s])), []).append((t, s))
    for key, pairs in sorted(groups.items()):
        t = np.array([p[0] for p in pairs], dtype=np.int64)
        s = np.array([p[1] for p in pairs], dtype=np.int64)
        S = np.empty((len(pairs), r, r))
        for a in range(0, len(pairs), chunk):
            S[a : a + chunk] = kernel_block(grids[t[a : a + chunk]], grids[s[a : a + chunk]], ell)
        coupling[key] = dict(t=t, s=s, S=S)

    lidx = _leaf_index(tree, rows)
    pts_pad = np.concatenate([tree.points, np.zeros((1, 2))])
    dt = np.array([p[0] for p in dense], dtype=np.int64)
    ds = np.array([p[1] for p in dense], dtype=np.int64)
    D = np.zeros((len(dense), rows, rows))
    for a in range(0, len(dense), chunk):
        ti, si = lidx[dt[a : a + chunk]], lidx[ds[a : a + chunk]]
        blk = kernel_block(pts_pad[ti], pts_pad[si], ell)
        blk *= (ti < tree.n)[:, :, None] & (si < tree.n)[:, None, :]
        D[a : a + chunk] = blk
    meta = dict(leaf_rows=rows, leaf_index=lidx, pos=pos, cheb_rank=r)
    return H2Matrix(tree=tree, ell=float(ell), order=int(cheb_order), eta=float(eta), ranks=[r] * L,
                    leaf_U=leaf_U, transfer=transfer, coupling=coupling,
                    dense=dict(t=dt, s=ds, D=D), meta=meta)


# ---------------------------------------------------------------- matvec (torch, any device)


def _level_struct(H):
    """Cached per-level index tensors on the arrays' device."""
    dev = H.arrays_on() or torch.device("cpu")
    key = ("struct", str(dev))
    if key in H.meta:
        return H.meta[key]
    tree, pos = H.tree, H.meta["pos"]
    L = tree.num_levels
    st = dict(leafpos=[], leafidx=[], parentpos=[], slot=[], nnodes=[])
    lidx = H.meta["leaf_index"]
    for l in range(L):
        ids = tree.level_nodes(l)
        st["nnodes"].append(len(ids))
        lv = np.array([i for i in ids if tree.is_leaf(i)], dtype=np.int64)
        st["leafpos"].append(torch.as_tensor(pos[lv] if len(lv) else np.zeros(0, np.int64), device=dev))
        st["leafidx"].append(torch.as_tensor(lidx[lv] if len(lv) else np.zeros((0, H.leaf_rows), np.int64),
                                             device=dev))
        if l > 0:
            par = tree.parent[ids]
            st["parentpos"].append(torch.as_tensor(pos[par], device=dev))
            st["slot"].append(torch.as_tensor((tree.children[par, 1] == ids).astype(np.int64), device=dev))
        else:
            st["parentpos"].append(None)
            st["slot"].append(None)
    st["cpl"] = {k: (torch.as_tensor(pos[g["t"]], device=dev), torch.as_tensor(pos[g["s"]], device=dev))
                 for k, g in H.coupling.items()}
    st["dense"] = (torch.as_tensor(lidx[H.dense["t"]], device=dev), torch.as_tensor(lidx[H.dense["s"]], device=dev))
    st["perm"] = torch.as_tensor(tree.perm, device=dev)
    H.meta[key] = st
    return st


def h2_matvec(H, x):
    """y = A_H x for x (n,) or (n, nrhs), original point order: upward pass
    x^ = U^T x through the transfer matrices, coupling y^_t += S_ts x^_s, downward pass, dense
    near field. H's arrays must be torch tensors; x is moved to their device/dtype."""
    if isinstance(H.dense["D"], np.ndarray):
        raise TypeError("h2_matvec needs a torch H2Matrix; call H.to(device)")
    D = H.dense["D"]
    x = torch.as_tensor(x)
    vec = x.dim() == 1
    if x.shape[0] != H.n:
        raise ValueError(f"x has {x.shape[0]} rows, H is {H.n} x {H.n}")
    x = x.to(device=D.device, dtype=D.dtype).reshape(H.n, -1)
    nrhs = x.shape[1]
    st = _level_struct(H)
    L = H.tree.num_levels
    xt = torch.zeros(H.n + 1, nrhs, dtype=D.dtype, device=D.device)
    xt[: H.n] = x[st["perm"]]
    xhat = [None] * L
    for l in range(L - 1, -1, -1):
        xl = torch.zeros(st["nnodes"][l], H.ranks[l], nrhs, dtype=D.dtype, device=D.device)
        if H.leaf_U[l] is not None:
            xl[st["leafpos"][l]] = H.leaf_U[l].transpose(1, 2) @ xt[st["leafidx"][l]]
        if l + 1 < L:
            xl.index_add_(0, st["parentpos"][l + 1], H.transfer[l + 1].transpose(1, 2) @ xhat[l + 1])
        xhat[l] = xl
    yhat = [torch.zeros_like(xh) for xh in xhat]
    for (lt, ls), g in H.coupling.items():
        tp, sp = st["cpl"][(lt, ls)]
        yhat[lt].index_add_(0, tp, g["S"] @ xhat[ls][sp])
    for l in range(1, L):
        yhat[l] += H.transfer[l] @ yhat[l - 1][st["parentpos"][l]]
    yt = torch.zeros(H.n + 1, nrhs, dtype=D.dtype, device=D.device)
    for l in range(L):
        if H.leaf_U[l] is not None:
            li = st["leafidx"][l]
            yt.index_add_(0, li.reshape(-1), (H.leaf_U[l] @ yhat[l][st["leafpos"][l]]).reshape(-1, nrhs))
    ti, si = st["dense"]
    if len(ti):
        yt.index_add_(0, ti.reshape(-1), (D @ xt[si]).reshape(-1, nrhs))
    y = torch.empty(H.n, nrhs, dtype=D.dtype, device=D.device)
    y[st["perm"]] = yt[: H.n]
    return y[:, 0] if vec else y


def estimate_error(H, Hc, nvec=30, seed=0):
    """||(A_H - A~_H) X||_F / ||A_H X||_F over ``nvec`` Gaussian vectors."""
    g = torch.Generator().manual_seed(seed)
    X = torch.randn(H.n, nvec, generator=g, dtype=torch.float64)
    y1, y2 = h2_matvec(H, X).double(), h2_matvec(Hc, X).double()
    return float((y1 - y2).norm() / y1.norm().clamp_min(1e-300))


def memory_report(H, element_bytes=None):
    """Bytes for dense leaves, basis (leaf U + transfer E) and coupling S;
    counts the stored (unpadded) entries: a leaf with m points costs m x k_l."""
    if element_bytes is None:
        D = H.dense["D"]
        element_bytes = D.element_size() if isinstance(D, torch.Tensor) else D.dtype.itemsize
    tree, k = H.tree, H.ranks
    cnt = tree.hi - tree.lo
    dense = int(sum(int(cnt[t]) * int(cnt[s]) for t, s in zip(H.dense["t"], H.dense["s"])))
    basis = 0
    for i in range(tree.num_nodes):
        l = int(tree.level[i])
        if tree.is_leaf(i):
            basis += int(cnt[i]) * k[l]
        if l > 0:
            basis += k[l] * k[l - 1]
    coupling = sum(len(g["t"]) * k[lt] * k[ls] for (lt, ls), g in H.coupling.items())
    out = dict(dense=dense * element_bytes, basis=basis * element_bytes, coupling=coupling * element_bytes)
    out["lowrank"] = out["basis"] + out["coupling"]
    out["total"] = out["dense"] + out["lowrank"]
    return out


# ---------------------------------------------------------------- batched GEMM over the C ABI


def bmm(a, b, *, ta=False, tb=False, out=None):
    """Batched op(a) @ op(b) of row-major (B, ., .) CUDA tensors on bf_gemm_batched_* (our DMMA /
    CUDA-core kernels). Row-major C = op(A) op(B) is the column-major C^T = op(B)^T op(A)^T."""
    L = _lib.load()
    if a.device.type != "cuda":
        raise _lib.BackendUnavailable("bmm runs on CUDA tensors only (no CPU fallback)")
    a = a.contiguous()
    b = b.contiguous()
    B = a.shape[0]
    M = a.shape[2] if ta else a.shape[1]
    K = a.shape[1] if ta else a.shape[2]
    N = b.shape[1] if tb else b.shape[2]
    if (b.shape[2] if tb else b.shape[1]) != K or b.shape[0] != B:
        raise ValueError(f"bmm shape mismatch {tuple(a.shape)} x {tuple(b.shape)}")
    if out is None:
        out = torch.empty(B, M, N, dtype=a.dtype, device=a.device)
    # column-major view: stored row-major X (r x c) == X^T column-major with ld c
    fn = L.bf_gemm_batched_f64 if a.dtype == torch.float64 else L.bf_gemm_batched_f32
    with torch.cuda.device(a.device):
        rc = fn(B, N, M, K,
                ptr(b), b.shape[2], b.shape[1] * b.shape[2], int(tb),
                ptr(a), a.shape[2], a.shape[1] * a.shape[2], int(ta),
                ptr(out), N, M * N, stream_handle(a.device))
    _lib.check(rc, "gemm")
    return out


# ---------------------------------------------------------------- compression (device)


@dataclass
class SvdChoice:
    """Per-node factorisation for the truncation: ``full`` one-sided Jacobi (bf_svd_batched),
    ``block`` block Jacobi (direct method) for more than 64 columns, or ``rsvd`` with a
    ``samples`` = k + p budget ("randomized SVD with 32 samples")."""

    kind: str = "full"
    samples: int = 32
    oversample: int = 8
    seed: int = 0


# converged flags of the batched Jacobi factorisations inside one compress() call (None outside);
# rsvd reports none (the reference drops the inner flag, rsvd.py:70-76)
_CONV_TALLY = None


def _tally(conv):
    if _CONV_TALLY is not None:
        _CONV_TALLY.append(conv)


def _factor(A, choice, level, need_v=True):
    """Batched SVD of (B, M, N), M >= N: returns u (B, M, w), s (B, w) descending, v (B, N, w)
    (v is None for ``full`` when not ``need_v``: the Jacobi sweeps then skip V entirely).

    ``full``: the one-sided Jacobi tiers (bf_svd_batched: register tier up to 64 columns, else
    the shared-memory tier); ``block``: block Jacobi, direct method (bf_block_svd_batched, the
    paper's "direct block Jacobi kernels" for the rank-121 fixture), columns zero-padded to a
    multiple of the block width; ``rsvd``: bf_rsvd_batched with a k + p = samples budget."""
    from .blockjacobi import BlockJacobiOptions, block_svd_tensor
    from .jacobi import JacobiOptions, svd_tensor
    from .rsvd import RsvdOptions, rsvd_tensor

    B, M, N = A.shape
    if choice.kind == "rsvd":
        w = min(choice.samples, N)
        p = min(choice.oversample, w - 1)
        r = rsvd_tensor(A, RsvdOptions(k=w - p, p=p, seed=choice.seed + level))
        return r["u"], r["s"], r["v"]
    if choice.kind == "block" and N > 64:
        bw = 32
        Np = -(-N // bw) * bw
        Mp = max(M, Np)
        Ap = torch.zeros(B, Mp, Np, dtype=A.dtype, device=A.device)
        Ap[:, :M, :N] = A
        r = block_svd_tensor(Ap, BlockJacobiOptions(block_width=bw, method="direct", accumulate_v=True))
        _tally(r["converged"])
        # the padded columns are exactly zero: their sigma are 0 and sort last
        return r["u"][:, :M, :N], r["sigma"][:, :N], r["v"][:, :N, :N]
    if M > N and (N > 64 or M > 64):
        # QR preconditioning (bf_qr_batched): the Jacobi sweeps then run on the N x N triangle,
        # whose columns fit shared memory; the left vectors are Q U_R (bf_gemm_batched)
        from .qr import qr_tensor

        q, rr = qr_tensor(A)
        r = svd_tensor(rr.contiguous(), JacobiOptions(ordering="round_robin", accumulate_v=need_v))
        _tally(r["converged"])
        return bmm(q.contiguous(), r["u"].contiguous()), r["sigma"], r["v"]
    r = svd_tensor(A, JacobiOptions(ordering="round_robin", accumulate_v=need_v))
    _tally(r["converged"])
    return r["u"], r["sigma"], r["v"]


def _node_svd(A, nz, k, choice, level):
    """SVD of every node matrix of a level, returned in a common padded form.

    A: (nn, R, k) node matrices with zero rows; nz: (nn, R) bool, the rows that may be nonzero.
    A node with fewer than k nonzero rows is rank deficient: one-sided Jacobi on it would chase
    the rounding noise of its null columns forever (the reference's criterion, jacobi.py:145-150,
    never accepts them), so it is factored as the transpose of its compacted nonzero rows
    (k x r_i, full column rank) and the roles of the singular vector sets are swapped back.
    Returns u (nn, R, w), s (nn, w), v (nn, k, w) with w = max width, zero-padded."""
    nn, R, _ = A.shape
    dev, dt = A.device, A.dtype
    cnt = nz.sum(dim=1)
    cnt_h = cnt.cpu().numpy()
    wide = np.nonzero(cnt_h < k)[0]
    tall = np.nonzero(cnt_h >= k)[0]
    parts = []
    if len(tall):
        idx = torch.as_tensor(tall, device=dev)
        At = A[idx]
        u, s, v = _factor(At, choice, level, need_v=False)
        if v is None:
            # T = diag(sigma) W^T = U^T A: the right vectors are never needed on their own, so the
            # sweeps skip V and W diag(sigma) = A^T U comes from one batched GEMM
            vs = bmm(At, u.contiguous(), ta=True)  # (b, k, w)
            v = vs / torch.where(s > 0, s, torch.ones_like(s))[:, None, :]
        parts.append((idx, u, s, v))
    if len(wide):
        idx = torch.as_tensor(wide, device=dev)
        C = int(cnt_h[wide].max())
        # compacted nonzero rows first (stable), C of them
        order = torch.argsort((~nz[idx]).to(torch.int8), dim=1, stable=True)[:, :C]  # (b, C)
        Ac = torch.gather(A[idx], 1, order[:, :, None].expand(-1, -1, k))  # (b, C, k)
        valid = torch.gather(nz[idx], 1, order)
        Ac = Ac * valid[:, :, None]
        if C == 0:
            ut = torch.zeros(len(wide), k, 0, dtype=dt, device=dev)
            st = torch.zeros(len(wide), 0, dtype=dt, device=dev)
            vt = torch.zeros(len(wide), 0, 0, dtype=dt, device=dev)
        else:
            ut, st, vt = _factor(Ac.transpose(1, 2).contiguous(), choice, level)  # Ac^T = ut diag(st) vt^T
        w = st.shape[1]
        # left vectors of A: vt (C x w) scattered back to the node's row positions
        uu = torch.zeros(len(wide), R, w, dtype=dt, device=dev)
        src = vt * valid[:, :, None]
        uu.scatter_(1, order[:, :, None].expand(-1, -1, w), src)
        parts.append((idx, uu, st, ut))
    w = max(p[2].shape[1] for p in parts)
    U = torch.zeros(nn, R, w, dtype=dt, device=dev)
    S = torch.zeros(nn, w, dtype=dt, device=dev)
    V = torch.zeros(nn, k, w, dtype=dt, device=dev)
    for idx, u, s, v in parts:
        ww = s.shape[1]
        U[idx, :, :ww] = u
        S[idx, :ww] = s
        V[idx, :, :ww] = v
    return U, S, V


def truncate_basis(H, eps, svd=None):
    """Bottom-up batched-SVD truncation of the basis tree (§8.2).

    Level l is one batched factorisation (two when it mixes full-rank and rank-deficient nodes,
    see _node_svd): leaves contribute their U (leaf_rows x k_l), inner nodes the stacked
    TE = [T_c1 E_c1; T_c2 E_c2] (2 k~_{l+1} x k_l, formed by bf_gemm_batched). Columns with
    sigma_j >= eps sigma_1 are kept per node (rank floor 1); the level rank is the max and the
    nodes below it get zero columns. New leaf bases / transfer matrices are the kept left vectors
    (block rows of Q~ for the children), and T = diag(sigma~) W~^T (= U~^T U). Returns
    (new_ranks, new_leaf_U, new_transfer, T per level, info)."""
    choice = svd or SvdChoice()
    if not eps > 0:
        raise ValueError("eps must be > 0")
    D = H.dense["D"]
    if not isinstance(D, torch.Tensor) or D.device.type != "cuda":
        raise _lib.BackendUnavailable("compress runs on the GPU: move the H2Matrix with H.to('cuda')")
    dev, dt = D.device, D.dtype
    st = _level_struct(H)
    tree = H.tree
    L = tree.num_levels
    rows = H.leaf_rows
    cnt = torch.as_tensor(tree.hi - tree.lo, device=dev)
    newk = [0] * L
    keeps = [None] * L
    new_U = [None] * L
    new_E = [None] * L
    T = [None] * L
    info = []
    for l in range(L - 1, -1, -1):
        nn, k = st["nnodes"][l], H.ranks[l]
        inner = l + 1 < L and st["nnodes"][l + 1] > 0
        kc = newk[l + 1] if inner else 0
        R = max(rows if H.leaf_U[l] is not None else 0, 2 * kc, 1)
        A = torch.zeros(nn, R, k, dtype=dt, device=dev)
        nz = torch.zeros(nn, R, dtype=torch.bool, device=dev)
        ar = torch.arange(R, device=dev)
        if H.leaf_U[l] is not None:
            lp = st["leafpos"][l]
            A[lp, :rows] = H.leaf_U[l]
            nz[lp] = ar[None, :] < cnt[torch.as_tensor(tree.level_nodes(l), device=dev)[lp]][:, None]
        if inner:
            TE = bmm(T[l + 1], H.transfer[l + 1])  # (nodes at l+1, kc, k)
            pp, sl = st["parentpos"][l + 1], st["slot"][l + 1]
            kk = keeps[l + 1]
            for j in (0, 1):
                sel = torch.nonzero(sl == j).flatten()
                A[pp[sel], j * kc : (j + 1) * kc] = TE[sel]
                nz[pp[sel], j * kc : (j + 1) * kc] = ar[None, :kc] < kk[sel][:, None]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        u, s, v = _node_svd(A, nz, k, choice, l)
        e1.record()
        s_host = s.double().cpu().numpy()  # the level rank is decided on the host (one small copy)
        keep = np.maximum(1, np.sum(s_host >= eps * s_host[:, :1], axis=1)) if s_host.shape[1] else np.ones(nn, int)
        kl = min(int(keep.max()) if nn else 1, s.shape[1]) if s.shape[1] else 1
        newk[l] = kl
        keeps[l] = torch.as_tensor(np.minimum(keep, kl), device=dev)
        mask = (torch.arange(kl, device=dev)[None, :] < keeps[l][:, None]).to(dt)
        if u.shape[2] < kl:  # a 0-width factorisation (all-zero nodes): pad
            u = torch.nn.functional.pad(u, (0, kl - u.shape[2]))
            s = torch.nn.functional.pad(s, (0, kl - s.shape[1]))
            v = torch.nn.functional.pad(v, (0, kl - v.shape[2]))
        Q = u[:, :, :kl] * mask[:, None, :]
        T[l] = ((s[:, :kl] * mask)[:, :, None] * v[:, :, :kl].transpose(1, 2)).contiguous()
        if H.leaf_U[l] is not None:
            new_U[l] = Q[st["leafpos"][l], :rows].contiguous()
        if inner:
            pp, sl = st["parentpos"][l + 1], st["slot"][l + 1]
            E = torch.empty(st["nnodes"][l + 1], kc, kl, dtype=dt, device=dev)
            for j in (0, 1):
                sel = torch.nonzero(sl == j).flatten()
                E[sel] = Q[pp[sel], j * kc : (j + 1) * kc]
            new_E[l + 1] = E
        info.append(dict(level=l, nodes=nn, rows=R, cols=k, rank_before=k, rank_after=kl,
                         svd_ms=round(e0.elapsed_time(e1), 3), wide_nodes=int((nz.sum(1) < k).sum()),
                         node_ranks_max=int(keep.max()) if nn else 0, node_ranks_min=int(keep.min()) if nn else 0))
    return newk, new_U, new_E, T, info[::-1]


def project_coupling(H, T, new_ranks=None):
    """S~_ts = T_t S_ts T_s^T for every LOWRANK leaf, one pair of batched GEMMs per (level_t,
    level_s) group; DENSE leaves untouched."""
    st = _level_struct(H)
    out = {}
    for key, g in H.coupling.items():
        lt, ls = key
        tp, sp = st["cpl"][key]
        X = bmm(T[lt][tp], g["S"])  # (blocks, k~_t, k_s)
        out[key] = dict(t=g["t"], s=g["s"], S=bmm(X, T[ls][sp], tb=True))
    return out


def compress(H, eps=1e-7, svd=None, *, sync_timing=True):
    """truncate_basis then project_coupling, assembled into a new H2Matrix.
    Returns (H~, report) with per-level ranks and the device time of each phase."""
    choice = svd or SvdChoice()
    dev = H.dense["D"].device if isinstance(H.dense["D"], torch.Tensor) else None
    if dev is None or dev.type != "cuda":
        raise _lib.BackendUnavailable("compress runs on the GPU: move the H2Matrix with H.to('cuda')")
    _level_struct(H)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    global _CONV_TALLY
    _CONV_TALLY = []
    t0 = time.perf_counter()
    ev[0].record()
    try:
        newk, U, E, T, info = truncate_basis(H, eps, choice)
    finally:
        flags, _CONV_TALLY = _CONV_TALLY, None
    ev[1].record()
    cpl = project_coupling(H, T, newk)
    ev[2].record()
    if sync_timing:
        torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    Hc = H2Matrix(tree=H.tree, ell=H.ell, order=H.order, eta=H.eta, ranks=newk, leaf_U=U, transfer=E,
                  coupling=cpl, dense=H.dense, meta={k: v for k, v in H.meta.items() if k in
                                                     ("leaf_rows", "leaf_index", "pos", "cheb_rank")})
    report = dict(
        eps=eps,
        svd=choice.kind,
        samples=choice.samples if choice.kind != "full" else None,
        ranks_before=list(H.ranks),
        ranks_after=newk,
        levels=info,
        truncation_ms=ev[0].elapsed_time(ev[1]) if sync_timing else None,
        projection_ms=ev[1].elapsed_time(ev[2]) if sync_timing else None,
        wall_s=wall,
        svd_calls=len(flags),
        nonconverged_entries=int(sum(int((~f.bool()).sum()) for f in flags)),
    )
    return Hc, report


def dense_assembly(H, chunk=512):
    """A_H materialised by matvecs against identity columns (n <= 2048)."""
    D = H.dense["D"]
    cols = []
    for a in range(0, H.n, chunk):
        e = torch.zeros(H.n, min(chunk, H.n - a), dtype=D.dtype, device=D.device)
        e[torch.arange(a, a + e.shape[1]), torch.arange(e.shape[1])] = 1
        cols.append(h2_matvec(H, e))
    return torch.cat(cols, dim=1)


def explicit_basis(H, node):
    """Explicit basis of ``node`` from the nested representation: leaves their U, inner nodes
    [U_c1 E_c1; U_c2 E_c2], rows in tree order over the node's points."""
    tree, pos = H.tree, H.meta["pos"]
    l = int(tree.level[node])
    to_np = (lambda x: x.detach().cpu().double().numpy()) if isinstance(H.dense["D"], torch.Tensor) else (lambda x: x)
    if tree.is_leaf(node):
        lv = [i for i in tree.level_nodes(l) if tree.is_leaf(i)]
        j = lv.index(node)
        m = tree.hi[node] - tree.lo[node]
        return to_np(H.leaf_U[l][j])[:m]
    parts = [explicit_basis(H, c) @ to_np(H.transfer[l + 1][pos[c]]) for c in tree.children[node]]
    return np.vstack(parts)


def level_summary(H):
    tree = H.tree
    return [dict(level=l, nodes=int(np.sum(tree.level == l)),
                 leaves=int(sum(1 for i in tree.level_nodes(l) if tree.is_leaf(i))), rank=H.ranks[l])
            for l in range(tree.num_levels)]


def require_cuda_device(device=None):
    return resolve_device(device)
