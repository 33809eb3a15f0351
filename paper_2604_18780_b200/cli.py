"""Command line: the reference's `decode` and `bench` subcommands (cli.py:42-53, 131-200,
390-440) on the device kernels.

    python -m paper_2604_18780_b200 decode --params p.json --emissions e.csv [--marginals m.json]
    python -m paper_2604_18780_b200 bench --T 1000 10000 --K 100 --C 24 --B 8 [--format csv]

Only the streaming backend exists here (the dense O(T K C^2) oracle is out of scope, §8);
`--backend dense` is rejected with the reference's JSON failure line on stderr.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time

BENCH_COLUMNS = (
    "backend", "T", "K", "C", "B", "wall_ms_forward", "wall_ms_backward", "peak_working_bytes",
    "positions_per_sec", "status",
)
# beside the reference's columns: fwd+bwd throughput (the BASELINE metric) and the device's peak
EXTRA_COLUMNS = ("positions_per_sec_fwd_bwd", "peak_device_bytes")


def _emit(args, text: str) -> None:
    if getattr(args, "out", None):
        with open(args.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def _emit_json(args, doc: dict) -> None:
    _emit(args, json.dumps(doc, indent=1) + "\n")


def _fail_stderr(command, reason: str) -> int:
    sys.stderr.write(json.dumps({"command": command, "status": "fail", "reason": reason}) + "\n")
    return 2


def _csv_cell(v) -> str:
    if v is None:
        return ""
    if isinstance(v, float):
        return repr(v)
    return str(v)


def _median_ms(fn, repeats: int) -> float:
    import torch

    fn()
    torch.cuda.synchronize()
    samples = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        samples.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(samples)


def cmd_bench(args) -> int:
    import torch

    from . import streaming as S
    from .accounting import MemoryLedger
    from .instances import equivalence_instance

    if args.backend == "dense":
        return _fail_stderr("bench", "the dense backend is not part of this build (streaming kernels only)")
    rows = []
    for T in args.T:
        _, params, cum = equivalence_instance(args.seed, T=T, K=args.K, C=args.C, B=args.B)
        row = dict.fromkeys(BENCH_COLUMNS + EXTRA_COLUMNS)
        row.update(backend="streaming", T=T, K=args.K, C=args.C, B=args.B, status="ok")
        torch.cuda.reset_peak_memory_stats()
        ledger = MemoryLedger()
        logZ, ckpts = S.streaming_forward(cum, params, args.delta, ledger=ledger)
        S.streaming_backward(cum, params, logZ, ckpts, ledger=ledger)
        fwd_ms = _median_ms(lambda: S.forward_logZ(cum, params, args.delta), args.repeats)

        def backward():
            z, ck = S.streaming_forward(cum, params, args.delta)
            S.streaming_backward(cum, params, z, ck)

        bwd_ms = _median_ms(backward, args.repeats)
        fb_ms = _median_ms(lambda: S.posterior(cum, params, args.delta), args.repeats)
        row.update(wall_ms_forward=fwd_ms, wall_ms_backward=bwd_ms, peak_working_bytes=ledger.total(),
                   positions_per_sec=args.B * T / (fwd_ms / 1e3),
                   positions_per_sec_fwd_bwd=args.B * T / (fb_ms / 1e3),
                   peak_device_bytes=int(torch.cuda.max_memory_allocated()))
        rows.append(row)
    if args.format == "csv":
        from .potentials import CSV_HEADER

        cols = BENCH_COLUMNS + EXTRA_COLUMNS
        lines = [CSV_HEADER, ",".join(cols)] + [",".join(_csv_cell(r[c]) for c in cols) for r in rows]
        _emit(args, "\n".join(lines) + "\n")
    else:
        _emit_json(args, {"command": "bench", "rows": rows})
    return 0


def cmd_decode(args) -> int:
    from . import streaming as S
    from .potentials import (CenteringMode, build_scores, load_emissions_csv, load_emissions_json,
                             load_params_json, segmentations_to_json)

    if args.backend == "dense":
        return _fail_stderr("decode", "the dense backend is not part of this build (streaming kernels only)")
    params = load_params_json(args.params)
    batch = load_emissions_json(args.emissions) if args.emissions.endswith(".json") else load_emissions_csv(args.emissions)
    cum = build_scores(batch, params, CenteringMode(args.centering))
    segs, score_arr = S.decode(cum, params)
    doc = {"command": "decode", "lengths": [int(v) for v in batch.lengths],
           "segmentations": segmentations_to_json(segs), "scores": [float(v) for v in score_arr]}
    if args.marginals:
        _, _, marg = S.posterior(cum, params, args.delta)
        lengths = [int(v) for v in marg.lengths]
        mdoc = {
            "lengths": lengths,
            "position_marginals": [marg.position_marginals[b, :L, :].tolist() for b, L in enumerate(lengths)],
            "boundary_posterior": [marg.boundary_posterior[b, :L].tolist() for b, L in enumerate(lengths)],
            "expected_segment_count": [float(v) for v in marg.expected_segment_count],
        }
        with open(args.marginals, "w") as fh:
            json.dump(mdoc, fh, indent=1)
    _emit_json(args, doc)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2604_18780_b200", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)
    sp = sub.add_parser("bench", help="wall time and working-set bytes (device streaming kernels)")
    sp.add_argument("--T", type=int, nargs="+", default=[1000, 10000])
    sp.add_argument("--K", type=int, default=100)
    sp.add_argument("--C", type=int, default=8)
    sp.add_argument("--B", type=int, default=4)
    sp.add_argument("--seed", type=int, default=0)
    sp.add_argument("--backend", choices=("dense", "streaming", "auto"), default="auto")
    sp.add_argument("--delta", type=int, default=None, help="checkpoint interval")
    sp.add_argument("--repeats", type=int, default=5, help="timed runs (median reported)")
    sp.add_argument("--format", choices=("json", "csv"), default="json")
    sp.add_argument("--out", default=None)
    sp = sub.add_parser("decode", help="best segmentations for stored inputs")
    sp.add_argument("--params", required=True, help="parameter JSON file")
    sp.add_argument("--emissions", required=True, help="emissions file (.csv or .json)")
    sp.add_argument("--centering", choices=("none", "mean", "shared_max"), default="none")
    sp.add_argument("--backend", choices=("dense", "streaming", "auto"), default="auto")
    sp.add_argument("--delta", type=int, default=None, help="checkpoint interval")
    sp.add_argument("--marginals", default=None, help="also write posterior marginals (JSON) here")
    sp.add_argument("--out", default=None)
    return ap


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return {"bench": cmd_bench, "decode": cmd_decode}[args.command](args)
    except ValueError as e:
        return _fail_stderr(args.command, str(e)) - 1


if __name__ == "__main__":  # pragma: no cover
    sys.exit(main())
