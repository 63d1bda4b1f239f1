"""CPU restatement of the H^2 compression. TEST INFRASTRUCTURE ONLY.

Importable only from tests/ (and bench-side checkers) -- never from the product package.
Per-node Python/numpy loops over a host H2Matrix (paper_1707_05141_b200.h2.build_h2 output):

  * matvec_ref       -- SPEC.md:488-494 (upward pass, coupling, downward pass, dense leaves);
  * compress_ref     -- SPEC.md:507-534 / PAPER.md §8.2: per node LAPACK SVD (np.linalg.svd,
                        the checker, not the thing measured), keep sigma_j >= eps * sigma_1 with
                        a rank floor of 1, level rank = max with zero columns below it, new
                        transfer matrices = block rows of Q~, T = diag(sigma~) W~^T, projection
                        S~ = T_t S T_s^T;
  * dense_kernel     -- the exact kernel matrix (SPEC.md:535's dense oracle).

Parity status: the reference ships no H^2 code (its package stops at the batched
factorisations, /root/reference/pkg/src/batchfact), so this restatement is pinned only to the
SPEC.md examples (tests/test_h2.py) -- "parity unpinned" against reference outputs.
"""

import numpy as np


def dense_kernel(points, ell):
    d = points[:, None, :] - points[None, :, :]
    return np.exp(-np.sqrt(np.sum(d * d, axis=-1)) / ell)


def _leaf_pos(H):
    """node -> index inside its level's leaf list."""
    tree = H.tree
    out = {}
    for l in range(tree.num_levels):
        lv = [i for i in tree.level_nodes(l) if tree.is_leaf(i)]
        for j, i in enumerate(lv):
            out[int(i)] = j
    return out


def matvec_ref(H, x):
    """y = A_H x, original point order, one node at a time."""
    tree, pos = H.tree, H.meta["pos"]
    lp = _leaf_pos(H)
    x = np.asarray(x, dtype=np.float64)
    vec = x.ndim == 1
    x = x.reshape(H.n, -1)
    xt = x[tree.perm]
    nodes = range(tree.num_nodes)
    xhat = {}
    for i in sorted(nodes, key=lambda i: -tree.level[i]):  # children before parents
        l = int(tree.level[i])
        if tree.is_leaf(i):
            m = tree.hi[i] - tree.lo[i]
            xhat[i] = H.leaf_U[l][lp[i]][:m].T @ xt[tree.lo[i] : tree.hi[i]]
        else:
            xhat[i] = sum(H.transfer[l + 1][pos[c]].T @ xhat[c] for c in tree.children[i])
    yhat = {i: np.zeros_like(xhat[i]) for i in nodes}
    for g in H.coupling.values():
        for b, (t, s) in enumerate(zip(g["t"], g["s"])):
            yhat[t] += g["S"][b] @ xhat[s]
    for i in sorted(nodes, key=lambda i: tree.level[i]):  # parents before children
        if tree.level[i] > 0:
            yhat[i] += H.transfer[tree.level[i]][pos[i]] @ yhat[tree.parent[i]]
    yt = np.zeros_like(xt)
    for i in tree.leaves():
        l, m = int(tree.level[i]), tree.hi[i] - tree.lo[i]
        yt[tree.lo[i] : tree.hi[i]] += H.leaf_U[l][lp[int(i)]][:m] @ yhat[i]
    for b, (t, s) in enumerate(zip(H.dense["t"], H.dense["s"])):
        mt, ms = tree.hi[t] - tree.lo[t], tree.hi[s] - tree.lo[s]
        yt[tree.lo[t] : tree.hi[t]] += H.dense["D"][b][:mt, :ms] @ xt[tree.lo[s] : tree.hi[s]]
    y = np.empty_like(yt)
    y[tree.perm] = yt
    return y[:, 0] if vec else y


def _truncate(u, s, vt, eps, kl):
    """Kept columns: sigma_j >= eps sigma_1 (floor 1), zero-padded to the level rank kl."""
    keep = max(1, int(np.sum(s >= eps * s[0]))) if len(s) else 1
    keep = min(keep, len(s)) if len(s) else 0
    Q = np.zeros((u.shape[0], kl))
    T = np.zeros((kl, vt.shape[1]))
    Q[:, :keep] = u[:, :keep]
    T[:keep] = s[:keep, None] * vt[:keep]
    return Q, T


def compress_ref(H, eps):
    """Returns (new H2Matrix on the host, new ranks). SPEC.md:507-534."""
    from paper_1707_05141_b200.h2 import H2Matrix

    tree, pos = H.tree, H.meta["pos"]
    lp = _leaf_pos(H)
    L = tree.num_levels
    rows = H.leaf_rows
    newk = [0] * L
    T = {}
    new_U = [None] * L
    new_E = [None] * L
    for l in range(L - 1, -1, -1):
        ids = tree.level_nodes(l)
        fac = {}
        keeps = []
        for i in ids:
            if tree.is_leaf(i):
                m = tree.hi[i] - tree.lo[i]
                A = H.leaf_U[l][lp[int(i)]][:m]
            else:
                A = np.vstack([T[c] @ H.transfer[l + 1][pos[c]] for c in tree.children[i]])
            u, s, vt = np.linalg.svd(A, full_matrices=False)
            fac[i] = (u, s, vt)
            keeps.append(max(1, int(np.sum(s >= eps * s[0]))) if len(s) else 1)
        kl = max(keeps)
        newk[l] = kl
        Q = {}
        for i in ids:
            Q[i], T[i] = _truncate(*fac[i], eps, kl)
        lv = [i for i in ids if tree.is_leaf(i)]
        if lv:
            new_U[l] = np.zeros((len(lv), rows, kl))
            for j, i in enumerate(lv):
                new_U[l][j, : Q[i].shape[0]] = Q[i]
        if l + 1 < L:
            kc = newk[l + 1]
            ch = tree.level_nodes(l + 1)
            E = np.zeros((len(ch), kc, kl))
            for c in ch:
                p = tree.parent[c]
                j = 0 if tree.children[p, 0] == c else 1
                E[pos[c]] = Q[p][j * kc : (j + 1) * kc]
            new_E[l + 1] = E
    cpl = {}
    for key, g in H.coupling.items():
        S = np.stack([T[t] @ g["S"][b] @ T[s].T for b, (t, s) in enumerate(zip(g["t"], g["s"]))])
        cpl[key] = dict(t=g["t"], s=g["s"], S=S)
    meta = {k: v for k, v in H.meta.items() if k in ("leaf_rows", "leaf_index", "pos", "cheb_rank")}
    Hc = H2Matrix(tree=tree, ell=H.ell, order=H.order, eta=H.eta, ranks=newk, leaf_U=new_U, transfer=new_E,
                  coupling=cpl, dense=H.dense, meta=meta)
    return Hc, newk
