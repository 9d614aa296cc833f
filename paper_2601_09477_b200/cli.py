"""Command line: the reference's ``multiply`` workflow on the B200 path.

    python -m paper_2601_09477_b200 [--seed S] [--threads T] [--transform fwht|fft] \\
        [--format csv|json] [--max-mem BYTES] \\
        multiply A B -o OUT (--cd CD --cb CB | -b WIDTH -d DEPTH) [--save-sketch SKETCH]

Same global options, validation and exit codes as the reference (cli.py:133-199):
0 on success, 1 on runtime failures (I/O, formats, memory budget, no GPU), 2 on
usage or parameter errors.  ``--max-mem`` applies the reference's budget check
(cli.py:85-92: 1.25 x estimate_workspace_bytes against the budget) before any
work; ``--format`` only selects the result-table format of the reference's
experiment subcommands and is accepted for compatibility.  The estimate matrix and the ``.skch`` container are written in the
reference's formats.  The reference's generator / experiment subcommands are
outside this path.
"""

from __future__ import annotations

import functools
import re
import time

import click

from . import __version__
from .errors import InvalidParameterError, MemoryBudgetError, SketchmmError
from .matio import load_matrix, save_matrix
from .sketch import (SketchParams, compress, decompress_all, derive_params, effective_threads,
                     estimate_workspace_bytes, save_sketch)


def _parse_bytes(text: str) -> int:
    """Memory size with an optional K/M/G/T suffix (cli.py:62-67)."""
    m = re.fullmatch(r"\s*(\d+(?:\.\d+)?)\s*([kmgt]?)b?\s*", text, re.IGNORECASE)
    if not m:
        raise click.BadParameter(f"cannot parse memory size {text!r}")
    scale = {"": 1, "k": 1 << 10, "m": 1 << 20, "g": 1 << 30, "t": 1 << 40}
    return int(float(m.group(1)) * scale[m.group(2).lower()])


def _check_budget(cfg: dict, n: int, b: int, d: int, transform: str) -> None:
    """The reference's working-set check (cli.py:85-92), same estimate and margin."""
    if cfg["max_mem"] is None:
        return
    need = int(1.25 * estimate_workspace_bytes(n, b, d, transform, effective_threads(cfg["threads"])))
    if need > cfg["max_mem"]:
        raise MemoryBudgetError(f"estimated working set {need} bytes exceeds --max-mem {cfg['max_mem']}")


def _cli_errors(fn):
    """Map library errors onto the exit-code contract (cli.py:70-82)."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except InvalidParameterError as exc:
            raise click.UsageError(str(exc)) from exc
        except (SketchmmError, OSError, RuntimeError) as exc:
            raise click.ClickException(str(exc)) from exc

    return wrapper


@click.group(context_settings={"help_option_names": ["-h", "--help"]})
@click.version_option(__version__, prog_name="sketchmm-b200")
@click.option("--seed", type=click.IntRange(0, 2**64 - 1), default=0, show_default=True,
              help="Root seed; all randomness derives from it.")
@click.option("--threads", type=click.IntRange(min=1), default=None,
              help="Accepted for compatibility (device reduction order is fixed).")
@click.option("--transform", type=click.Choice(["fft", "fwht"]), default="fwht", show_default=True,
              help="Sketch convolution variant.")
@click.option("--format", "fmt", type=click.Choice(["csv", "json"]), default="csv", show_default=True,
              help="Result table format of the reference's experiment subcommands (compatibility).")
@click.option("--max-mem", type=str, default=None, metavar="BYTES",
              help="Refuse runs whose estimated working set exceeds this budget (accepts K/M/G/T suffixes).")
@click.pass_context
def main(ctx, seed, threads, transform, fmt, max_mem):
    """Sketched matrix products on B200: estimate entries of A @ B from a small sketch."""
    budget = _parse_bytes(max_mem) if max_mem is not None else None
    ctx.obj = {"seed": seed, "threads": threads, "transform": transform, "fmt": fmt, "max_mem": budget}


@main.command()
@click.argument("a_file", type=click.Path(dir_okay=False))
@click.argument("b_file", type=click.Path(dir_okay=False))
@click.option("-o", "--out", required=True, type=click.Path(dir_okay=False),
              help="Output matrix file (.csv for text, anything else binary).")
@click.option("--cd", type=float, default=None, help="Depth constant c_d.")
@click.option("--cb", type=float, default=None, help="Width constant c_b.")
@click.option("-b", "--buckets", type=int, default=None, help="Explicit sketch width b.")
@click.option("-d", "--depth", type=int, default=None, help="Explicit sketch depth d.")
@click.option("--save-sketch", "sketch_out", type=click.Path(dir_okay=False), default=None,
              help="Also write the sketch container to this path.")
@click.pass_obj
@_cli_errors
def multiply(cfg, a_file, b_file, out, cd, cb, buckets, depth, sketch_out):
    """Estimate A @ B through a sketch and write the full estimate matrix."""
    derived = cd is not None or cb is not None
    explicit = buckets is not None or depth is not None
    if derived == explicit or (derived and (cd is None or cb is None)) or (
            explicit and (buckets is None or depth is None)):
        raise click.UsageError("give either --cd with --cb, or --buckets with --depth")
    a = load_matrix(a_file)
    b = load_matrix(b_file)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape != b.shape:
        raise InvalidParameterError(f"operands must be square with matching size, got {a.shape} and {b.shape}")
    n = a.shape[0]
    if derived:
        params = derive_params(n, cd, cb, transform=cfg["transform"], seed=cfg["seed"])
    else:
        params = SketchParams(n=n, b=buckets, d=depth, transform=cfg["transform"], seed=cfg["seed"])
    _check_budget(cfg, n, params.b, params.d, params.transform)
    threads = effective_threads(cfg["threads"])
    t0 = time.perf_counter()
    sk = compress(a, b, params, threads=threads)
    est = decompress_all(sk)
    wall = time.perf_counter() - t0
    save_matrix(out, est)
    if sketch_out is not None:
        save_sketch(sketch_out, sk)
    click.echo(f"n={n} b={params.b} d={params.d} transform={params.transform} threads={threads} "
               f"seed={params.seed} wall={wall:.3f}s", err=True)


if __name__ == "__main__":  # pragma: no cover
    main()
