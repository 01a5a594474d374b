"""Command-line entry for the B200 path.

    python -m paper_2506_05617_b200.cli singvals --weights W.npy --height M --width N \
        [--values-only] [--dtype f64|f32] [--device cuda:0] [--out spectrum.csv] [--meta run.json]
    python -m paper_2506_05617_b200.cli gen-kernel --cout C --cin C [--kh 3 --kw 3 --seed 0] --out W.npy

``singvals`` is the reference's command (CS/cli.py:107-123) on the device:
NPY kernel in (read_npy_kernel), ``compute_spectrum`` on the GPU, the
spectrum CSV and optional metadata JSON out, the same one-line summary.
``--device`` and ``--dtype`` are added (fp64 by default, as the reference
computes).  ``--workers`` is accepted for compatibility and ignored.
Exit codes follow CS/cli.py:1-5: 0 success, 2 usage / validation, 3 resource
limits (memory budget, size cap, no CUDA device), 4 non-convergence.  The
reference's ``compare-boundary`` and ``bench`` commands drive its dense
Dirichlet oracle and its CPU timing grid; they are outside this package's
hot path.
"""

from __future__ import annotations

import argparse
import sys

from .errors import AllocationFailure, ConvergenceFailure, ConvSpectraError, SizeCapExceeded
from .kernels import SpatialDims, random_kernel
from .npyio import read_npy_kernel, write_npy_kernel, write_run_metadata_json, write_spectrum_csv


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="conv-spectra-b200",
                                 description="Singular value spectra of 2D multi-channel convolutions on a B200.")
    sub = ap.add_subparsers(dest="command", required=True)

    p = sub.add_parser("singvals", help="compute a spectrum on the GPU and write it as CSV")
    p.add_argument("--weights", required=True, help="kernel NPY file (c_out, c_in, k_h, k_w)")
    p.add_argument("--height", type=int, required=True, metavar="M")
    p.add_argument("--width", type=int, required=True, metavar="N")
    p.add_argument("--method", choices=("lfa", "fft"), default="lfa")
    p.add_argument("--boundary", choices=("periodic",), default="periodic")
    p.add_argument("--values-only", action="store_true", help="values only (the vectors solve may still run)")
    p.add_argument("--workers", type=int, default=0, help="accepted for compatibility; no host pool")
    p.add_argument("--dtype", choices=("f64", "f32"), default="f64")
    p.add_argument("--device", default="cuda:0")
    p.add_argument("--out", default="spectrum.csv")
    p.add_argument("--meta", default=None, help="optional metadata JSON path")
    p.add_argument("--size-cap", type=int, default=None)
    p.set_defaults(func=cmd_singvals)

    p = sub.add_parser("gen-kernel", help="write a seeded random kernel as NPY")
    p.add_argument("--cout", type=int, required=True)
    p.add_argument("--cin", type=int, required=True)
    p.add_argument("--kh", type=int, default=3)
    p.add_argument("--kw", type=int, default=3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--dist", choices=("normal", "uniform"), default="normal")
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_gen_kernel)
    return ap


def cmd_singvals(args) -> int:
    from .pipeline import compute_spectrum

    kernel = read_npy_kernel(args.weights)
    dims = SpatialDims(n=args.width, m=args.height)
    result = compute_spectrum(kernel, dims, method=args.method, boundary=args.boundary,
                              values_only=args.values_only, workers=args.workers,
                              size_cap=args.size_cap, device=args.device, dtype=args.dtype)
    write_spectrum_csv(result, args.out)
    if args.meta:
        write_run_metadata_json(result, args.meta, device=args.device, dtype=args.dtype)
    print(f"{len(result)} singular values ({args.method}, {args.boundary}, {args.dtype}, {args.device}) "
          f"-> {args.out}; sigma_max={result.values[0]:.6g}")
    return 0


def cmd_gen_kernel(args) -> int:
    kernel = random_kernel(args.cout, args.cin, args.kh, args.kw, seed=args.seed, dist=args.dist)
    write_npy_kernel(args.out, kernel)
    print(f"kernel ({args.cout}, {args.cin}, {args.kh}, {args.kw}) seed={args.seed} dist={args.dist} -> {args.out}")
    return 0


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return args.func(args)
    except (SizeCapExceeded, AllocationFailure) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except ConvergenceFailure as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 4
    except (ConvSpectraError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except RuntimeError as exc:  # no CUDA device / library: no CPU fallback
        print(f"error: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
