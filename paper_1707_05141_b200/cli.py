"""Command-line front end with JSON-lines records (the reference declares
``batchfact = "batchfact.cli:entry"`` in pkg/pyproject.toml:15-16 but ships no module).

    python -m paper_1707_05141_b200 gen --m 64 --n 32 --seed 3 --out a.txt
    python -m paper_1707_05141_b200 bench svd --m 32 --n 32 --batch 10 --precision f64
    python -m paper_1707_05141_b200 bench qr|block-svd|rsvd ... [--report path] [--strict]

Every record echoes the fully resolved configuration (defaults included), the seed, the
precision, wall time, and the per-batch metrics (sweeps, convergence flags, residuals). Exit
codes: 0 success, 1 invalid arguments (usage text), 2 numerical non-convergence with --strict.
``compress`` runs the H^2 workflow (h2.py): build the covariance H^2 matrix on
the host, compress it on the GPU, report per-level ranks, memory and the error estimate.
Inputs are the reference's synthetic matrices: ``gaussian_matrix`` (rsvd.py:42-53) with key
``seed + i``, or ``testmat.make_matrix`` spectra for ``--cond``.
"""

import argparse
import json
import sys
import time

import numpy as np

USAGE_EXIT, NONCONV_EXIT = 1, 2


def write_matrix_text(path, a):
    """Write a matrix as text: a ``rows cols`` header, then row-major values (core.py:126-134)."""
    from .core import as_matrix

    a = as_matrix(a)
    with open(path, "w") as fh:
        fh.write(f"{a.shape[0]} {a.shape[1]}\n")
        for i in range(a.shape[0]):
            fh.write(" ".join(repr(float(x)) for x in a[i, :]))
            fh.write("\n")


def read_matrix_text(path, dtype=np.float64):
    """Read a matrix written by :func:`write_matrix_text` (column-major result, core.py:137-147)."""
    with open(path) as fh:
        header = fh.readline().split()
        if len(header) != 2:
            raise ValueError(f"{path}: bad header {header!r}")
        rows, cols = int(header[0]), int(header[1])
        data = fh.read().split()
    if len(data) != rows * cols:
        raise ValueError(f"{path}: expected {rows * cols} values, got {len(data)}")
    a = np.array([float(x) for x in data], dtype=dtype).reshape(rows, cols)
    return np.asfortranarray(a)


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _UsageError(f"{self.prog}: {message}\n{self.format_usage()}")


class _UsageError(Exception):
    pass


def _parser():
    p = _Parser(prog="batchfact_b200", description="B200 batched QR / Jacobi SVD / randomized SVD")
    sub = p.add_subparsers(dest="cmd")

    def common(q):
        q.add_argument("--m", type=int, default=32)
        q.add_argument("--n", type=int, default=32)
        q.add_argument("--batch", type=int, default=10)
        q.add_argument("--seed", type=int, default=0)
        q.add_argument("--precision", choices=("f64", "f32"), default="f64")
        q.add_argument("--cond", type=float, default=None, help="testmat geometric spectrum instead of Gaussian")
        q.add_argument("--report", default=None, help="append the JSON line here instead of stdout")
        q.add_argument("--strict", action="store_true", help="exit 2 if any entry did not converge")
        q.add_argument("--threads", type=int, default=None, help="accepted for compatibility (no effect)")
        q.add_argument("--device", default=None)

    g = sub.add_parser("gen", help="write one synthetic matrix in the text format")
    g.add_argument("--m", type=int, default=32)
    g.add_argument("--n", type=int, default=32)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--cond", type=float, default=None)
    g.add_argument("--rank", type=int, default=None)
    g.add_argument("--out", required=True)

    b = sub.add_parser("bench", help="run one batched workflow and emit a JSON-lines record")
    bs = b.add_subparsers(dest="op")
    q = bs.add_parser("qr")
    common(q)
    q.add_argument("--panel-width", type=int, default=16)
    s = bs.add_parser("svd")
    common(s)
    s.add_argument("--ordering", choices=("serial", "round_robin"), default="serial")
    s.add_argument("--tolerance", type=float, default=None)
    s.add_argument("--max-sweeps", type=int, default=30)
    k = bs.add_parser("block-svd")
    common(k)
    k.add_argument("--block-width", type=int, default=32)
    k.add_argument("--method", choices=("gram", "direct"), default="direct")
    k.add_argument("--tolerance", type=float, default=None)
    k.add_argument("--max-sweeps", type=int, default=30)
    r = bs.add_parser("rsvd")
    common(r)
    r.add_argument("--k", type=int, default=8)
    r.add_argument("--p", type=int, default=8)

    c = sub.add_parser("compress", help="H^2 covariance matrix: build, batched-SVD compression, report")
    c.add_argument("--n", type=int, default=4096)
    c.add_argument("--ell", type=float, default=0.1)
    c.add_argument("--cheb-order", type=int, default=8)
    c.add_argument("--leaf-size", type=int, default=64)
    c.add_argument("--eta", type=float, default=1.0)
    c.add_argument("--eps", type=float, default=1e-7)
    c.add_argument("--svd", choices=("full", "rsvd"), default="full")
    c.add_argument("--samples", type=int, default=32)
    c.add_argument("--oversample", type=int, default=8)
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--precision", choices=("f64", "f32"), default="f64")
    c.add_argument("--error-vectors", type=int, default=30)
    c.add_argument("--report", default=None)
    c.add_argument("--device", default=None)
    c.add_argument("--strict", action="store_true",
                   help=f"exit {NONCONV_EXIT} when a batched Jacobi SVD of the truncation did not converge")
    return p


def _compress(args):
    """per-level ranks before/after, memory before/after, error estimate,
    wall time per phase (truncation vs projection)."""
    import torch

    from . import h2

    if args.n < 1 or args.leaf_size < 1 or args.cheb_order < 1 or not (args.ell > 0 and args.eta > 0 and args.eps > 0):
        raise ValueError("compress: --n, --leaf-size, --cheb-order, --ell, --eta and --eps must be positive")
    if args.samples < 2 or args.oversample < 0:
        raise ValueError("compress: --samples must be >= 2 and --oversample >= 0")
    from .core import resolve_device

    dev = resolve_device(args.device)
    t0 = time.perf_counter()
    H = h2.build_h2(h2.perturbed_grid(args.n, seed=args.seed), args.ell, args.cheb_order, args.eta, args.leaf_size)
    t_build = time.perf_counter() - t0
    dt = torch.float64 if args.precision == "f64" else torch.float32
    Hd = H.to(dev, dt)
    choice = h2.SvdChoice(kind=args.svd, samples=args.samples, oversample=args.oversample, seed=args.seed)
    h2.compress(Hd, args.eps, choice)  # warm-up (library load, allocator)
    Hc, rep = h2.compress(Hd, args.eps, choice)
    ref = H.to(dev, torch.float64)
    err = h2.estimate_error(ref, Hc, nvec=args.error_vectors, seed=args.seed)
    cfg = {k: v for k, v in vars(args).items() if k not in ("report", "cmd")}
    rec = dict(command="compress", config=cfg, precision=args.precision, seed=args.seed, build_s=t_build,
               levels=h2.level_summary(H), error_estimate=err,
               memory_before=h2.memory_report(Hd), memory_after=h2.memory_report(Hc))
    rec.update({k: v for k, v in rep.items() if k != "levels"})
    rec["truncation_levels"] = rep["levels"]
    return rec


def _inputs(args):
    """(B, m, n) host batch: gaussian_matrix(m, n, seed + i) or testmat make_matrix spectra."""
    import torch

    from .rsvd import gaussian_tensor
    from .testmat import make_matrix_tensor

    if args.cond is not None:
        a, _ = make_matrix_tensor(args.batch, args.m, args.n, args.cond, seed=args.seed, device=args.device)
    else:
        a = gaussian_tensor(args.batch, args.m, args.n, args.seed, seed_mode="add", device=args.device)
    if args.precision == "f32":
        a = a.to(torch.float32)
    return a


def _residuals(a, u, s, v):
    import torch

    a = a.double()
    u, s = u.double(), s.double()
    eye_n = torch.eye(u.shape[-1], dtype=torch.float64, device=u.device)
    out = {"orth_u_max": float((u.transpose(1, 2) @ u - eye_n).norm(dim=(1, 2)).max())}
    if v is not None:
        v = v.double()
        eye_v = torch.eye(v.shape[-1], dtype=torch.float64, device=v.device)
        out["orth_v_max"] = float((v.transpose(1, 2) @ v - eye_v).norm(dim=(1, 2)).max())
        rec = (u * s[:, None, :]) @ v.transpose(1, 2)
        out["recon_rel_max"] = float(((a - rec).norm(dim=(1, 2)) / a.norm(dim=(1, 2)).clamp_min(1e-300)).max())
    return out


def _bench(args):
    import torch

    from . import BlockJacobiOptions, JacobiOptions, RsvdOptions, block_svd_tensor, qr_tensor, rsvd_tensor, svd_tensor

    a = _inputs(args)
    cfg = {k: v for k, v in vars(args).items() if k not in ("report", "cmd")}
    rec = {"command": f"bench {args.op}", "config": cfg, "precision": args.precision, "seed": args.seed}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    conv_all = True
    if args.op == "qr":
        q, r = qr_tensor(a, args.panel_width)
        torch.cuda.synchronize()
        rec["wall_s"] = time.perf_counter() - t0
        qd, rd, ad = q.double(), r.double(), a.double()
        eye = torch.eye(q.shape[-1], dtype=torch.float64, device=q.device)
        rec["orth_q_max"] = float((qd.transpose(1, 2) @ qd - eye).norm(dim=(1, 2)).max())
        rec["recon_rel_max"] = float(((ad - qd @ rd).norm(dim=(1, 2)) / ad.norm(dim=(1, 2)).clamp_min(1e-300)).max())
        rec["bytes"] = int(a.numel() * a.element_size() + q.numel() * q.element_size() + r.numel() * r.element_size())
    elif args.op == "svd":
        o = JacobiOptions(tolerance=args.tolerance, max_sweeps=args.max_sweeps, ordering=args.ordering,
                          accumulate_v=True)
        out = svd_tensor(a, o)
        torch.cuda.synchronize()
        rec["wall_s"] = time.perf_counter() - t0
        sw = out["sweeps"].double()
        rec.update(sweeps_mean=float(sw.mean()), sweeps_max=int(sw.max()),
                   converged=[bool(x) for x in out["converged"].cpu()])
        conv_all = all(rec["converged"])
        rec.update(_residuals(a, out["u"], out["sigma"], out["v"]))
    elif args.op == "block-svd":
        o = BlockJacobiOptions(block_width=args.block_width, method=args.method, tolerance=args.tolerance,
                               max_sweeps=args.max_sweeps, accumulate_v=True)
        out = block_svd_tensor(a, o)
        torch.cuda.synchronize()
        rec["wall_s"] = time.perf_counter() - t0
        sw = out["sweeps"].double()
        rec.update(sweeps_mean=float(sw.mean()), sweeps_max=int(sw.max()),
                   converged=[bool(x) for x in out["converged"].cpu()])
        conv_all = all(rec["converged"])
        rec.update(_residuals(a, out["u"], out["sigma"], out["v"]))
    else:
        out = rsvd_tensor(a, RsvdOptions(k=args.k, p=args.p, seed=args.seed))
        torch.cuda.synchronize()
        rec["wall_s"] = time.perf_counter() - t0
        rec.update(_residuals(a, out["u"], out["s"], out["v"]))
    for key, val in list(rec.items()):
        if isinstance(val, float) and not np.isfinite(val):
            rec[key] = None
            rec.setdefault("nonfinite", []).append(key)
    return rec, conv_all


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    try:
        args = _parser().parse_args(argv)
        if args.cmd is None or (args.cmd == "bench" and args.op is None):
            raise _UsageError(_parser().format_help())
    except _UsageError as exc:
        sys.stderr.write(str(exc))
        return USAGE_EXIT
    except SystemExit as exc:  # --help
        return int(exc.code or 0)
    if args.cmd == "gen":
        from .rsvd import gaussian_matrix

        if args.cond is not None:
            from .testmat import make_matrix_tensor

            a, _ = make_matrix_tensor(1, args.m, args.n, args.cond, rank=args.rank, seed=args.seed)
            a = a[0].cpu().numpy()
        else:
            a = gaussian_matrix(args.m, args.n, args.seed)
        write_matrix_text(args.out, a)
        return 0
    try:
        if args.cmd == "compress":
            rec = _compress(args)
            conv_all = rec.get("nonconverged_entries", 0) == 0
        else:
            rec, conv_all = _bench(args)
    except ValueError as exc:
        sys.stderr.write(f"{exc}\n")
        return USAGE_EXIT
    line = json.dumps(rec, sort_keys=True)
    if args.report:
        with open(args.report, "a") as fh:
            fh.write(line + "\n")
    else:
        print(line)
    return NONCONV_EXIT if (getattr(args, "strict", False) and not conv_all) else 0


def entry():
    sys.exit(main())
