"""Command line for the B200 path: ``python -m paper_2502_06377_b200.cli``.

Mirrors the reference's solve-path subcommands (`/root/reference/pkg/src/ibmi/cli.py`):

* ``invert``  — approximate the inverse of a stored SPD matrix (cli.py:63-74, :145-166);
* ``compare`` — solve vs direct inversion on one matrix (cli.py:89-95, :206-211);
* ``gen``     — write one of the BASELINE problems (c1–c4) to an IBMI1/CSV file
  (the reference's grid-kernel ``gen`` is outside this path).

Flags, partition options (``--blocks/--overlap/--ordering/--partition-json``),
guess syntax (``mc:N:SEED``) and exit codes (0 ok, 1 error) follow the
reference.  IBMI1 inputs stream straight into HBM and Σ straight back to disk
(``ibmi_load_ibmi1`` / ``ibmi_save_sigma_ibmi1``); CSV goes through the host.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import matio
from .exceptions import InvalidOverlap
from .partition import contiguous_partition, contiguous_ranges, block_permutation, load_partition_json, \
    red_black_partition
from .solver import GUESS_CHOICES, GUESS_MONTE_CARLO, IbmiConfig

__all__ = ["main"]


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        return args.handler(args)
    except (OSError, ValueError, ArithmeticError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


def _parser():
    ap = argparse.ArgumentParser(prog="ibmi-b200", description="Iterative block inversion on a B200")
    sub = ap.add_subparsers(required=True)
    inv = sub.add_parser("invert", help="approximate the inverse of a stored matrix")
    inv.add_argument("--in", dest="input", required=True)
    inv.add_argument("--out", help="file for the approximate inverse")
    inv.add_argument("--tol", type=float, default=1e-8)
    inv.add_argument("--max-iters", type=int, default=500)
    _partition_flags(inv)
    inv.add_argument("--guess", default="identity", help="identity | local | mc:N:SEED | takahashi | jacobi")
    inv.add_argument("--stopping", default="estimate", choices=("estimate", "frobenius"))
    inv.add_argument("--report", help="write a JSON solve report here")
    inv.add_argument("--device", type=int, default=0)
    inv.set_defaults(handler=_cmd_invert)
    cmp_ = sub.add_parser("compare", help="solve vs direct inversion for one matrix")
    cmp_.add_argument("--in", dest="input", required=True)
    cmp_.add_argument("--tol", type=float, default=1e-8)
    cmp_.add_argument("--max-iters", type=int, default=500)
    _partition_flags(cmp_)
    cmp_.add_argument("--guess", default="identity")
    cmp_.add_argument("--device", type=int, default=0)
    cmp_.set_defaults(handler=_cmd_compare)
    gen = sub.add_parser("gen", help="write a BASELINE problem matrix")
    gen.add_argument("--config", choices=("c1", "c2", "c3", "c4"), required=True)
    gen.add_argument("--seed", type=int, default=0)
    gen.add_argument("--out", required=True)
    gen.set_defaults(handler=_cmd_gen)
    return ap


def _partition_flags(cmd):
    cmd.add_argument("--blocks", type=int, default=2)
    cmd.add_argument("--overlap", type=float, default=0.0)
    cmd.add_argument("--ordering", choices=("contiguous", "red-black"), default="contiguous")
    cmd.add_argument("--partition-json", help="custom partition file overriding the flags")


def _partition(args, p):
    if args.partition_json:
        return load_partition_json(args.partition_json)
    if args.ordering == "red-black":
        if args.overlap != 0.0:
            raise InvalidOverlap("red-black ordering does not support overlap")
        return red_black_partition(p)
    return contiguous_partition(p, args.blocks, args.overlap)


def _config(args) -> IbmiConfig:
    guess, mc_samples, mc_seed = args.guess, 100, 0
    if guess == GUESS_MONTE_CARLO or guess.startswith(GUESS_MONTE_CARLO + ":"):
        parts = guess.split(":")
        guess = GUESS_MONTE_CARLO
        if len(parts) > 1 and parts[1]:
            mc_samples = int(parts[1])
        if len(parts) > 2 and parts[2]:
            mc_seed = int(parts[2])
    if guess not in GUESS_CHOICES:
        raise ValueError(f"unknown guess {args.guess!r}")
    return IbmiConfig(tol=args.tol, max_iterations=args.max_iters, initial_guess=guess, mc_samples=mc_samples,
                      mc_seed=mc_seed, stopping=getattr(args, "stopping", "estimate"))


def _p_of(path) -> int:
    if matio.is_csv(path):
        return matio.load_csv(path).shape[0]
    rows, cols = matio.read_header(path)
    return rows


def _device_state(path, part, device):
    """DeviceSolver for the file: IBMI1 straight into HBM when no relabelling is needed."""
    from .device import DeviceSolver

    if not matio.is_csv(path) and (contiguous_ranges(part) is not None or block_permutation(part) is None):
        return DeviceSolver.from_ibmi1(path, part, device=device), None
    a = matio.load_matrix(path)
    return DeviceSolver(a, partition=part, device=device), a


def _cmd_invert(args) -> int:
    from .partition import validate
    from .solver import run_solve

    p = _p_of(args.input)
    part = _partition(args, p)
    validate(part)
    cfg = _config(args)
    t0 = time.perf_counter()
    ds, a = _device_state(args.input, part, args.device)
    with ds:
        rep = run_solve(ds, part, cfg, a=a, fetch_result=False)
        if args.out:
            if matio.is_csv(args.out):
                matio.save_csv(args.out, ds.sigma())
            else:
                ds.save_sigma_ibmi1(args.out)
    if args.report:
        payload = {"iterations": rep.iterations, "converged": rep.converged, "error_trace": rep.error_trace,
                   "wall_times": rep.wall_times, "total_seconds": rep.total_seconds,
                   "power_iterations": rep.power_iterations, "residual_trace": rep.residual_trace,
                   "setup_seconds": rep.setup_seconds, "end_to_end_seconds": time.perf_counter() - t0}
        with open(args.report, "w") as fh:
            json.dump(payload, fh, indent=2)
    status = "converged" if rep.converged else "NOT converged"
    print(f"{status} after {rep.iterations} iteration(s); last error estimate {rep.error_trace[-1]:.6e}")
    return 0


def _cmd_compare(args) -> int:
    """solve vs direct SPD inversion (reference bench.compare_direct, bench.py:135-159), both on the GPU."""
    from .linalg import spd_inverse, two_norm
    from .solver import solve

    a = matio.load_matrix(args.input)
    part = _partition(args, a.shape[0])
    cfg = _config(args)
    t0 = time.perf_counter()
    rep = solve(a, part, cfg, device=args.device)
    t_ibmi = time.perf_counter() - t0
    t0 = time.perf_counter()
    direct = spd_inverse(a)
    t_direct = time.perf_counter() - t0
    diff = two_norm(rep.result - direct)
    payload = {"p": int(a.shape[0]), "iterations": rep.iterations, "converged": rep.converged,
               "ibmi_seconds": t_ibmi, "direct_seconds": t_direct, "inverse_error_2norm": diff,
               "relative_error_2norm": diff / max(two_norm(direct), 1e-300)}
    print(json.dumps(payload))
    return 0


def _cmd_gen(args) -> int:
    from . import configs

    matio.save_matrix(args.out, configs.make_matrix(args.config, args.seed))
    return 0


if __name__ == "__main__":
    sys.exit(main())
