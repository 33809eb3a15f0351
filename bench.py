"""Benchmark: streaming semi-CRF forward+backward positions/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4]
                    [--scaling weak|strong] [--memory full|sublinear]

One step = one full forward + backward (logZ, all gradients, all marginals) of the batch of
BASELINE.json config 4 (B=8, T=100000, K=1000, C=24; synthetic instance
`equivalence_instance(seed, ..., mode=MEAN)`), followed -- for N > 1 -- by the path's only
cross-GPU exchange: the per-sequence grad_T / grad_B partials all-gathered in batch order and
reduced in a fixed order (bit-identical to one GPU). Weak scaling (default): every rank owns
its own B=8 batch. Strong scaling: one B=8 batch split across the ranks. `value` = all
ranks' positions / max-over-ranks device time.

`e2e` = the same metric through the public numpy API (`posterior`) with host inputs and host
outputs (H2D of S and parameters, D2H of logZ, gradients, marginals) inside the timed region.
`--impl reference` times the REAL reference (baseline/_ref, pip-installed from
/root/reference) on the host cores (steady-state positions, all cores); when baseline/_ref
is absent, the CPU oracle port of the reference algorithm.

The inputs (S: 8 x 100001 x 24 fp64 = 154 MB) are larger than the 126 MB L2, so no
explicit flush is done between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "positions/sec (B*T) for fwd+bwd at T=100k,K=1000,C=24"
UNIT = "positions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the forward-only and Viterbi throughputs (reported beside the headline, SURVEY 8(d))")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--memory", default="full", choices=["full", "sublinear"],
                    help="working-memory mode of the timed posterior (the other mode is reported in extras)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# CPU baseline: the reference on the host cores, steady-state sample

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "streamcrf"))


def _ref_worker(args):
    """Seconds per steady-state position of the REAL reference's streaming_forward +
    streaming_backward (one sequence): two runs of lengths K + n1 and K + n2 differenced, which
    cancels the t < K ramp (SURVEY §6.2 method)."""
    K, C, seed, n1, n2 = args
    sys.path.insert(0, REF_DIR)
    from streamcrf.potentials import CenteringMode as RMode
    from streamcrf.streaming import streaming_backward, streaming_forward
    from streamcrf.validation import equivalence_instance as ref_instance

    secs = []
    for n in (n1, n2):
        _, params, cum = ref_instance(seed, T=K + n, K=K, C=C, B=1, mode=RMode.MEAN)
        t0 = time.perf_counter()
        logZ, ck = streaming_forward(cum, params)
        streaming_backward(cum, params, logZ, ck)
        secs.append(time.perf_counter() - t0)
    return (secs[1] - secs[0]) / (n2 - n1)


def _port_worker(args):
    cfg, seed, n_steps = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import streaming_oracle as oracle

    from paper_2604_18780_b200.instances import equivalence_instance
    from paper_2604_18780_b200.potentials import CenteringMode

    K = cfg["K"]
    _, params, cum = equivalence_instance(seed, T=K + n_steps + 2, K=K, C=cfg["C"], B=1, mode=CenteringMode.MEAN)
    return oracle.steady_position_seconds(cum, params, n_steps)


def cpu_baseline(cfg: dict, budget_s: float) -> dict:
    """positions/s of the reference's fwd+bwd on all host cores (one sequence per core).

    The real reference (baseline/_ref) when installed -- kind "reference" -- else the oracle
    port (kind "port"). Per-position cost is constant once t >= K, so rate = cores / seconds
    per steady-state position; the sample is a few dozen positions per core."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    workers = max(1, min(cores, 8))
    K, C = cfg["K"], cfg["C"]
    t0 = time.perf_counter()
    if have_reference():
        n1, n2 = 8, 8 + max(64, min(256, int(16 * budget_s)))
        with mp.get_context("spawn").Pool(workers) as pool:
            secs = pool.map(_ref_worker, [(K, C, s, n1, n2) for s in range(workers)])
        kind = "reference"
        sample = (f"baseline/_ref streamcrf 0.1.0 (the reference, pip-installed from /root/reference): "
                  f"streaming_forward + streaming_backward of one sequence per process, lengths K+{n1} and "
                  f"K+{n2} differenced (steady state t >= K), K={K}, C={C}, {workers} processes")
    else:
        probe = _port_worker((cfg, 0, 2))
        n_steps = int(max(2, min(200, budget_s / max(probe, 1e-6) / 1.5)))
        with mp.get_context("spawn").Pool(workers) as pool:
            secs = pool.map(_port_worker, [(cfg, s, n_steps) for s in range(workers)])
        kind = "port"
        sample = (f"oracle/streaming_oracle.py (reference algorithm, fp64 numpy) steady-state fwd+replay+bwd, "
                  f"{n_steps} positions per process, K={K}, C={C}, {workers} processes")
    wall = time.perf_counter() - t0
    per_pos = float(np.mean(secs))
    return {"value": workers / per_pos, "unit": UNIT, "cores": workers, "kind": kind,
            "sample": sample + f"; {wall:.1f}s wall; value = processes / mean s-per-position",
            "seconds_per_position": per_pos}


# ---------------------------------------------------------------------------
# clocks sampling during the timed region


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) >= 7:
                for n, v in zip(names, s[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:  # noqa: BLE001
        return {}


def hbm_peak_gbs():
    """HBM copy peak: MEASURED_PEAKS.json (driver-written) or the profiling guide's fallback."""
    f = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(f):
        with open(f) as fh:
            d = json.load(fh)
        if "hbm_gbs" in d:
            return float(d["hbm_gbs"]), "of measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "of fallback (6.65 TB/s, B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def mufu_peak_per_s(sm_mhz: float | None) -> tuple[float, str]:
    """MUFU ex2 peak = 148 SMs x 16 / clk x f_SM (16/clk/SM measured: profiles/r01_microbench.jsonl)."""
    peaks = measured_peaks()
    mhz = sm_mhz or peaks.get("sm_max_mhz", 1965.0)
    return 148 * 16 * mhz * 1e6, f"148 SM x 16 ex2/clk (microbenchmarked) x {mhz:.0f} MHz (median SM clock in the timed region)"


def run_ours(args, rank, world, local):
    import torch

    import paper_2604_18780_b200 as scrf
    from paper_2604_18780_b200 import _lib
    from paper_2604_18780_b200 import streaming as S
    from paper_2604_18780_b200.dist import reduce_shared_grads_exact, shard_bounds
    from paper_2604_18780_b200.instances import CONFIGS

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    S.set_precision(args.precision)
    cfg = dict(CONFIGS[args.config])
    B, T, K, C = cfg["B"], cfg["T"], cfg["K"], cfg["C"]
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    # synthetic instance of the config's shape: weak scaling -> every rank its own B-sequence
    # batch (seed = rank); strong scaling -> one B-sequence batch, this rank's contiguous shard
    if args.scaling == "weak":
        _, params, cum = scrf.equivalence_instance(rank, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN)
        B_glob, lo = B * world, rank * B
    else:
        _, params, cum_all = scrf.equivalence_instance(0, T=T, K=K, C=C, B=B, mode=scrf.CenteringMode.MEAN)
        lo, hi = shard_bounds(B, rank, world)
        from dataclasses import replace

        cum = replace(cum_all, S=cum_all.S[lo:hi], lengths=np.asarray(cum_all.lengths)[lo:hi])
        B_glob = B
    B_loc = cum.batch_size
    prob = scrf.DeviceProblem.from_host(cum, params, device=dev)
    torch.cuda.synchronize()
    lib = _lib.load()

    def step():
        fwd, bw = S.device_posterior(prob, memory=args.memory)
        n = lib.scrf_last_launch_count()
        if world > 1:
            # the path's only collective: per-sequence grad_T / grad_B partials gathered in batch
            # order, fixed-order reduction (bit-identical to the single-GPU result)
            gT, gB = S.device_grad_partials(prob, fwd, bw)
            reduce_shared_grads_exact(gT, gB, B_glob)
            n += 3
        return n

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # live kernel timing (events around the fused alpha/beta sweep launch, on the launching stream)
    ev_main = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev_step = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for e in ev_main + ev_step:  # torch creates the CUDA event lazily on first record
        e.record()
    torch.cuda.synchronize()
    sweep_ms, step_ms = [], []
    for _ in range(min(2, args.steps)):
        lib.scrf_profile_events(ev_main[0].cuda_event, ev_main[1].cuda_event)
        ev_step[0].record()
        S.device_posterior(prob, memory=args.memory)
        ev_step[1].record()
        lib.scrf_profile_events(None, None)
        torch.cuda.synchronize()
        sweep_ms.append(ev_main[0].elapsed_time(ev_main[1]))
        step_ms.append(ev_step[0].elapsed_time(ev_step[1]))

    t_start = torch.cuda.Event(enable_timing=True)
    t_stop = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    torch.cuda.reset_peak_memory_stats(dev)
    with sampler:
        t_start.record()
        for _ in range(args.steps):
            launches += step()
        t_stop.record()
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = t_start.elapsed_time(t_stop) / args.steps
    if dist is not None:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    positions = B_glob * T
    value = positions / (ms / 1e3)
    clocks = sampler.summary()
    peak_mem = torch.cuda.max_memory_allocated(dev)

    out = None
    if rank == 0:
        # dominant kernel: the fused alpha+beta sweep (one launch per step): (K*C + C^2) exps per
        # position per direction in the factored recursion; the blocked tails
        # evaluate most of the K*C part as FMA against exp-space source blocks, so the MUFU pipe
        # is far from saturated -- the sweep is bound by the latency of its per-position chain
        # step (profiles/r02_sweep_summary.txt has the executed MUFU / FMA pipe rates)
        E_sweep = 2 * (K * C + C * C)
        sweep_avg = float(np.mean(sweep_ms))
        post_avg = float(np.mean(step_ms)) - sweep_avg
        peak, peak_note = mufu_peak_per_s(clocks["sm_mhz"])
        achieved = B_loc * T * E_sweep / (sweep_avg / 1e3)
        alg_bytes = 2 * B_loc * (T + 1) * C * 8 + 2 * 2 * B_loc * (T + 1) * C * 4 + B_loc * (T + 1) * 2 * 8
        traffic, executed = None, None
        tfile = os.path.join(ROOT, "profiles", "r02_sweep_traffic.json")
        if os.path.exists(tfile) and (B_loc, T, K, C) == (8, 100000, 1000, 24):
            with open(tfile) as fh:
                tj = json.load(fh)
            traffic = int(tj["bytes_per_launch"])
            executed = tj.get("executed")
        hbm_peak, hbm_src = hbm_peak_gbs()
        out = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": ("f32 log-semiring (fp64 prefix sums / normalisers / cut normalisers; fp64 outputs)"
                      if args.precision == "fp32" else "f64"),
            "data": f"synthetic: equivalence_instance(seed={'rank' if args.scaling == 'weak' else 0}, mode=MEAN) of "
                    f"config {args.config[1:]}",
            "config": {
                "workload": f"BASELINE config {args.config[1:]} fwd+bwd (logZ, grad_S/T/B, marginals), "
                            f"B={B_glob} T={T} K={K} C={C} in total ({B_loc} per GPU)",
                "B_total": B_glob, "B_per_gpu": B_loc, "T": T, "K": K, "C": C,
                "delta": S.choose_checkpoint_interval(T, K), "memory_mode": args.memory,
                "parallelism": f"batch-sharded dp{world}; grad_T/grad_B: per-sequence partials all-gathered "
                               f"in batch order + fixed-order reduce (bit-identical to 1 GPU)",
                "l2": "inputs larger than L2 (S = 154 MB fp64 per 8 sequences); no flush",
            },
            "roofline": {
                "bound": "sfu",
                "limiter": "latency of the per-position chain step of the alpha/beta recursions "
                           "(one dependent LSE + C x C GEMV per position); no pipe is saturated",
                "kernel": "sweep_kernel (alpha and beta message sweeps, one cluster per sequence and direction)",
                "achieved": achieved / 1e9,
                "peak": peak / 1e9,
                "unit": "Gexp2/s",
                "frac": achieved / peak,
                "traffic": traffic,
                "traffic_source": "profiles/r02_sweep_traffic.json (dram__bytes_read+write, ncu --set full)",
                "executed": executed,
                "hbm": {"algorithmic_bytes": alg_bytes, "achieved": alg_bytes / (sweep_avg / 1e3) / 1e9,
                        "peak": hbm_peak, "unit": "GB/s", "frac": alg_bytes / (sweep_avg / 1e3) / 1e9 / hbm_peak,
                        "peak_source": hbm_src},
                "algorithm": "factored: (K*C + C^2) exps per position per direction (algorithmic count)",
                "per_launch_exps": B_loc * T * E_sweep,
                "kernel_ms": sweep_avg,
                "post_ms": post_avg,
                "peak_note": peak_note,
            },
            "clocks": clocks,
            "peak_hbm_bytes": int(peak_mem),
            "gpu_launches": int(launches),
        }
    return out, (prob, cum, params, cfg, dev, lib, S, scrf, torch, dist, B_glob)


def e2e_measure(ctx, args):
    """The public numpy API end to end: host arrays in, host arrays out."""
    prob, cum, params, cfg, dev, lib, S, scrf, torch, dist, B_glob = ctx
    T, K = cfg["T"], cfg["K"]
    B = cum.batch_size
    # warm: two calls holding their results, as the timed loop does, so the pinned host blocks
    # of both live result sets are in torch's caching host allocator (steady state)
    for _ in range(3):
        res = scrf.posterior(cum, params, memory=args.memory)
    del res
    torch.cuda.synchronize()
    n = max(1, min(3, args.steps))
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    walls = []
    for _ in range(n):
        t1 = time.perf_counter()
        logZ, grads, marg = scrf.posterior(cum, params, memory=args.memory)
        walls.append(time.perf_counter() - t1)
    wall = (time.perf_counter() - t0) / n
    if dist is not None:  # every rank runs its shard through the API; the job takes the slowest
        tw = torch.tensor([wall], device=dev, dtype=torch.float64)
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        wall = float(tw.item())
    h2d = cum.S.nbytes + np.asarray(cum.lengths).nbytes + params.transition.nbytes + params.duration_bias.nbytes
    d2h = (logZ.nbytes + grads.grad_S.nbytes + grads.grad_T.nbytes + grads.grad_B.nbytes
           + marg.position_marginals.nbytes + marg.boundary_posterior.nbytes + marg.expected_segment_count.nbytes
           + B * 4 + B * 8 * (-(-T // S.choose_checkpoint_interval(T, K))))
    return {"value": B_glob * T / wall, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": "paper_2604_18780_b200.posterior (numpy in / numpy out, host wall clock, max over ranks)",
            "steps": n, "call_ms": [round(1e3 * w, 2) for w in walls]}


def _time_device(torch, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def extras_measure(ctx, args):
    """Beside the headline: forward only, Viterbi, the other memory mode (throughput and peak
    device memory of both), and the other BASELINE configs (fwd+bwd and Viterbi)."""
    prob, cum, params, cfg, dev, lib, S, scrf, torch, dist, B_glob = ctx
    B, T = prob.B, prob.T
    res = {}
    res["forward_positions_per_s"] = B * T / (_time_device(torch, lambda: S.device_forward(prob, sparse=True)) / 1e3)
    vit_ms = _time_device(torch, lambda: S.device_viterbi(prob))
    res["viterbi_positions_per_s"] = B * T / (vit_ms / 1e3)
    # Viterbi against the fp64 add pipe: (K*C + C^2) max-plus candidates per position (one fp64
    # add + one fp64 compare each, exact fp64 with the reference's tie rules); peak = measured
    # add.f64 rate (profiles/r01_microbench.jsonl: 18.1 T/s at 1965 MHz)
    K, C = prob.K, prob.C
    cand = float(B * T) * (K * C + C * C)
    res["viterbi_roofline"] = {"bound": "latency (one dependent max-plus step per position; head issue-bound)",
                               "pipe": "fp64", "achieved": cand / (vit_ms / 1e3) / 1e9, "peak": 18100.0,
                               "unit": "G fp64 add/s", "frac": cand / (vit_ms / 1e3) / 1e9 / 18100.0,
                               "peak_source": "profiles/r01_microbench.jsonl (add.f64, measured)",
                               "kernel_ms": vit_ms}
    modes = {}
    for mode in ("full", "sublinear"):
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        ms = _time_device(torch, lambda: S.device_posterior(prob, memory=mode))
        modes[mode] = {"positions_per_s": B * T / (ms / 1e3), "ms": ms,
                       "peak_working_bytes": int(torch.cuda.max_memory_allocated(dev) - base),
                       "input_bytes": int(prob.S.numel() * 8)}
    res["memory_modes"] = modes
    from paper_2604_18780_b200.instances import CONFIGS

    others = {}
    for name in ("c1", "c2", "c3", "c5"):
        c = CONFIGS[name]
        _, p2, cum2 = scrf.equivalence_instance(0, T=c["T"], K=c["K"], C=c["C"], B=c["B"], mode=scrf.CenteringMode.MEAN)
        pr = scrf.DeviceProblem.from_host(cum2, p2, device=dev)
        n = c["B"] * c["T"]
        others[name] = {
            "workload": f"B={c['B']} T={c['T']} K={c['K']} C={c['C']}",
            "fwd_bwd_positions_per_s": n / (_time_device(torch, lambda: S.device_posterior(pr)) / 1e3),
            "viterbi_positions_per_s": n / (_time_device(torch, lambda: S.device_viterbi(pr)) / 1e3),
        }
        del pr
    res["other_configs"] = others
    return res


def main():
    args = parse()
    rank, world, local = dist_env()
    from paper_2604_18780_b200.instances import CONFIGS

    cfg = dict(CONFIGS[args.config])
    if args.impl == "reference":
        if rank != 0:
            return 0
        cb = cpu_baseline(cfg, args.cpu_seconds)
        B_glob = cfg["B"] * (world if args.scaling == "weak" else 1)
        line = {
            "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world, "steps": 1,
            "warmup": 0, "ms_per_step": B_glob * cfg["T"] / cb["value"] * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"BASELINE config {args.config[1:]} fwd+bwd, B={B_glob} T={cfg['T']} "
                                   f"K={cfg['K']} C={cfg['C']}",
                       "note": (f"one steady-state sample (requested --steps {args.steps} --warmup {args.warmup}): "
                                "CPU seconds per position measured on the host cores and scaled to the config")},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0

    out, ctx = run_ours(args, rank, world, local)
    e2e = None if args.no_e2e else e2e_measure(ctx, args)  # all ranks (collective at N > 1)
    if rank == 0:
        if not args.no_e2e:
            out["e2e"] = e2e
        if not args.no_extras and world == 1:
            out["extras"] = extras_measure(ctx, args)
        if not args.no_cpu and world == 1:
            out["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds)
        print(json.dumps(out), flush=True)
    dist = ctx[-2]
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
