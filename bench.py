#!/usr/bin/env python
"""Benchmark of the Kaczmarz++ / CD++ hot path (BASELINE.json metric:
"block-iters/s & HBM GB/s vs 8 TB/s (fp64); time to 1e-8 rel. residual").

One *step* = one cold kpp_solve of `--iters` block iterations on a context whose memo
cache was cleared first, so every step runs every hot-path row (schedule, Phase-1
factorisation of each fresh block, Phase-2 iterations with the adaptive momentum).
Inputs (A, b) are resident in HBM before the timed region; A (512 MiB for c2) is larger
than L2, and each step touches every row of it.

Default workload (N=1): BASELINE configs[1] = c2, Kaczmarz++ m=n=8192, s=128.
N>1 (torchrun): the same problem column-sharded across ranks (NCCL allreduce of the
s-vector per iteration), strong scaling.

`--impl reference` times the CPU oracle (oracle/) on the host cores on a bounded sample
of the same workload (this tier has no reference implementation to install).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "block-iters/s & HBM GB/s vs 8 TB/s (fp64); time to 1e-8 rel. residual"
UNIT = "block-iters/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=list(synth.CONFIGS))
    ap.add_argument("--iters", type=int, default=0, help="block iterations per step (0: config default)")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-1e-8 measurement")
    ap.add_argument("--ttt-cap", type=int, default=0,
                    help="iteration cap of the time-to-tolerance solve (0: 25M, or 1M with --proj 1)")
    ap.add_argument("--cpu-seconds", type=float, default=24.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--engine", type=int, default=-1)
    ap.add_argument("--rht", action="store_true", help="randomized Hadamard preprocessing (SURVEY 8(f) NEXT-1)")
    ap.add_argument("--proj", type=int, default=0, choices=[0, 1],
                    help="K++ projection: 0 exact (memoized factor), 1 sketch + LSQR (Alg 6, SURVEY 8(f) NEXT-2)")
    ap.add_argument("--tmax", type=int, default=8, help="LSQR steps per iteration with --proj 1 (P:1322)")
    ap.add_argument("--secondary", default="c5,c4",
                    help="N=1 only: configs measured after the headline one and reported under 'secondary' "
                         "(the HBM-bound configs, so their roofline is in the driver's line); '' for none")
    return ap.parse_args()


DEFAULT_ITERS = {"c1": 500, "c2": 8192, "c3": 4096, "c4": 1024, "c5": 2048}


def bytes_per_iter(cfg, n_local=None):
    """Algorithmic HBM bytes of one block iteration: A_S once (8 s n),
    the memoized s x s operator, s-vectors and the x / m read+write (32 n)."""
    s = cfg.s
    n = cfg.n if n_local is None else n_local
    return 8 * s * n + 8 * s * s + 12 * s + 32 * n


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.raw = []
        self.t_enter = 0.0

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            # nvidia-smi's start-up (driver initialisation) must not overlap the timed region: it
            # held up the host thread of short steps (c1: 15 ms regions).  Wait for its first sample.
            t_end = time.monotonic() + 5.0
            while not self.raw and time.monotonic() < t_end:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.t_enter = time.monotonic()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.raw.append((time.monotonic(), line.strip()))

    def __exit__(self, *a):
        if self.proc:
            # a region shorter than the 200 ms period: keep the first sample after it
            t_end = time.monotonic() + 0.5
            while not any(t >= self.t_enter for t, _ in self.raw) and time.monotonic() < t_end:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        self.lines = [l for t, l in self.raw if t >= self.t_enter]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(cfg_name, kernel="iterate_kernel"):
    """dram bytes per iteration of the Phase-2 kernel from the committed ncu capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        e = d.get(cfg_name, {}).get(kernel)
        return e.get("dram_bytes_per_iter") if e else None
    except Exception:
        return None


FP64_DGEMM_TFLOPS = 35.47  # measured: torch.matmul fp64 8192^3, best of 10 (profiles/r01/fp64_peak.txt)


def phase1_flops(cfg, n_blocks, n_refined):
    """Algorithmic flops of Phase 1: per fresh block Gram s(s+1)n (K++) plus
    Cholesky, triangular inverse and M = X X^T (s^3/3 each); per refined block (second CholeskyQR
    pass) Q1 = X1^T A_S (s^2 n, X1 triangular), Gram s(s+1)n and the s x s products (~5 s^3/3)."""
    s, n = cfg.s, cfg.n
    small = s ** 3
    if cfg.kind == "cdpp":
        return n_blocks * small
    return n_blocks * (s * (s + 1) * n + small) + n_refined * (s * s * n + s * (s + 1) * n + 5 * small / 3)


def cpu_model():
    try:
        for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if l.startswith("Model name:"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _oracle_timed(cfg, A_host, b_host, T, threads, proj, tmax):
    import oracle
    tm = np.zeros(3)
    run = oracle.cdpp_run if cfg.kind == "cdpp" else oracle.kpp_run
    kw = {} if cfg.kind == "cdpp" else {"proj": proj, "tmax": tmax}
    run(A_host, b_host, cfg.s, lam=cfg.lam, seed=0, max_iters=T, threads=threads, timing=tm, **kw)
    return float(tm[0]), float(tm[1]), int(tm[2])


def cpu_oracle_sample(cfg, A_host, b_host, seconds, iters, proj=0, tmax=8):
    """Time the oracle, as it stands, on the host cores (SURVEY 8(d) protocol): iterations 0..T-1
    of the same cold solve, T grown until a run takes about its share of `seconds`, once with ONE
    thread (primary) and once with every core (OpenMP over independent outputs, secondary).  The
    oracle times its first-visit factorisations apart (instrumentation only), which gives
      - the warm (memoized, Phase-2-only) rate: T / (wall - factor seconds),
      - seconds per fresh-block factorisation (the paper's s^3/3-per-fresh-block split),
      - the cold-prefix rate T / wall (mostly fresh blocks: labelled as such),
    and `value` = the like-for-like rate of ONE bench step: `iters` iterations with the step's own
    number of fresh blocks (the schedule is data independent and bit-identical on both sides):
    iters / (iters / warm + n_fresh * factor seconds)."""
    import oracle
    oracle.build()
    C = oracle.cdpp_C(cfg.n, cfg.s) if cfg.kind == "cdpp" else oracle.kpp_C(cfg.m, cfg.n, cfg.s)
    n_fresh = int(oracle.schedule(0, C, iters)[2])
    allc = os.cpu_count() or 1
    out = {}
    for label, threads, share in (("1_thread", 1, 0.5), ("all_cores", allc, 0.5)):
        T = 4
        while True:
            wall, fac, nf = _oracle_timed(cfg, A_host, b_host, T, threads, proj, tmax)
            if wall >= seconds * share / 2 or T >= 1 << 16:
                break
            T = int(T * min(8.0, max(2.0, seconds * share / 2 / max(wall, 1e-3))))
        warm = T / max(wall - fac, 1e-9)
        per_f = fac / nf if nf else None
        step = iters / (iters / warm + (n_fresh * per_f if per_f else 0.0))
        out[label] = {"threads": threads, "iters_timed": T, "wall_s": wall, "fresh_blocks_timed": nf,
                      "factor_s": fac, "warm_block_iters_per_s": warm, "s_per_fresh_factor": per_f,
                      "cold_prefix_block_iters_per_s": T / wall, "step_block_iters_per_s": step}
    main = out["all_cores"]
    return {"value": main["step_block_iters_per_s"], "unit": UNIT, "cores": allc, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{cfg.name}: iterations 0..T-1 of the cold solve timed on the host "
                      f"({main['iters_timed']} on {allc} threads, {out['1_thread']['iters_timed']} on 1), "
                      f"first-visit {'sketch' if proj else 'Householder'} factors timed apart; value = one bench "
                      f"step of {iters} iterations with its {n_fresh} fresh blocks at the measured warm rate "
                      f"and seconds per factor, all cores",
            "step_fresh_blocks": n_fresh, "single_thread": out["1_thread"], "all_cores": out["all_cores"]}


def workload_config(cfg, iters, world, dist, proj=0, tmax=8):
    """The `config` object of the JSON line (shared by both arms)."""
    algo = "CD++" if cfg.kind == "cdpp" else ("Kaczmarz++(LSQR-%d)" % tmax if proj else "Kaczmarz++")
    return {"workload": f"{cfg.name}: {algo} "
                        f"m={cfg.m} n={cfg.n} s={cfg.s} lam={cfg.lam:g}",
            "iters_per_step": iters, "step": "cold solve (memo cache cleared)",
            "parallelism": f"column-sharded x{world}" if dist else "1 GPU",
            "l2": (f"inputs larger than L2 (A = {cfg.m * cfg.n * 8 / 2**20:.0f} MiB)" if not l2_small(cfg) else
                   f"L2 flushed before every timed step (A = {cfg.m * cfg.n * 8 / 2**20:.1f} MiB fits in L2; "
                   f"{L2_FLUSH_BYTES >> 20} MiB written outside the step's events)")}


L2_BYTES = 126 << 20
L2_FLUSH_BYTES = 512 << 20


def l2_small(cfg):
    """A fits in twice the B200's 126 MB L2: bench steps are timed one by one with a flush between."""
    return cfg.m * cfg.n * 8 < 2 * L2_BYTES


def measure_secondary(name, steps, warmup, dev, hbm_peak):
    """A short N=1 block for an HBM-bound config (c4/c5): cold bench steps of the config's default
    iteration count, one warm solve (pure Phase 2) with its roofline against the measured copy
    bandwidth, and the time to 1e-8.  Device time with CUDA events on the solve's stream."""
    import paper_2501_11673_b200 as kpp
    cfg = synth.CONFIGS[name]
    iters = DEFAULT_ITERS[name]
    A, b, _ = synth.make_problem(cfg, seed=0, device=dev)
    ctx = (kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup)(A, cfg.s, cfg.lam, 0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream)
    x_out = torch.empty(cfg.n, dtype=torch.float64, device=dev)
    for _ in range(warmup):
        ctx.clear_cache()
        ctx.solve(b, max_iters=iters, x_out=x_out)
    torch.cuda.synchronize()
    ctx.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        ctx.clear_cache()
        ctx.solve(b, max_iters=iters, x_out=x_out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    cold = ctx.stats()
    ctx.reset_stats()
    ctx.solve(b, max_iters=iters, x_out=x_out)  # warm: every factor memoized
    warm = ctx.stats()
    bpi = bytes_per_iter(cfg)
    ach = bpi * iters / (warm["phase2_ms"] / 1e3) / 1e9 if warm["phase2_ms"] > 0 else None
    tr = ncu_traffic(name, "iterate_kernel")
    ctx.clear_cache()
    zeta = -(-(cfg.n if cfg.kind == "cdpp" else cfg.m) // cfg.s)
    e0.record(stream)
    r = ctx.solve(b, max_iters=200000, tol=1e-8, x_out=x_out, hist_cap=200000 // (2 * zeta) + 2)
    e1.record(stream)
    torch.cuda.synchronize()
    true_res = float(torch.linalg.vector_norm(A @ x_out - b) / torch.linalg.vector_norm(b))
    out = {"workload": workload_config(cfg, iters, 1, False)["workload"], "iters_per_step": iters,
           "value": steps * iters / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps,
           "phase1_ms_per_step": cold["phase1_ms"] / steps, "phase2_ms_per_step": cold["phase2_ms"] / steps,
           "warm_block_iters_per_s": iters / (warm["phase2_ms"] / 1e3) if warm["phase2_ms"] > 0 else None,
           "roofline": {"bound": "hbm", "kernel": "Phase-2 persistent kernel, warm (iterate_kernel / cdpp_stream_kernel)",
                        "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak if ach else None,
                        "bytes_per_iter": bpi, "traffic": tr * iters if tr else None,
                        "frac_of_nominal_8tbs": ach / 8000.0 if ach else None,
                        "dram_gbs_ncu": tr / (warm["phase2_ms"] / iters / 1e3) / 1e9 if (tr and warm["phase2_ms"] > 0) else None,
                        "traffic_note": "ncu dram read+write bytes per iteration (profiles/ncu_summary.json) x iterations per launch"},
           "time_to_tol": {"seconds": e0.elapsed_time(e1) / 1e3, "iters": r.iters, "converged": r.status == kpp.OK,
                           "est_rel_res": float(r.res_hist[-1]) if len(r.res_hist) else None,
                           "true_rel_res": true_res, "tol": 1e-8}}
    ctx.destroy()
    del A, b, x_out
    torch.cuda.empty_cache()
    return out


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    A, b, _ = synth.make_problem(cfg, seed=0, device="cuda" if torch.cuda.is_available() else "cpu")
    A_host, b_host = A.cpu().numpy(), b.cpu().numpy()
    del A, b
    per_step, step_ms = [], []
    cb = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = cpu_oracle_sample(cfg, A_host, b_host, args.cpu_seconds / max(1, args.steps),
                              args.iters or DEFAULT_ITERS[cfg.name], args.proj, args.tmax)
        if i >= args.warmup:
            per_step.append(r["value"])
            step_ms.append((time.perf_counter() - t0) * 1e3)
            cb = r
    v = float(np.median(per_step))
    cb["value"] = v
    iters = args.iters or DEFAULT_ITERS[cfg.name]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(step_ms)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, iters, 1, False, args.proj, args.tmax),
            "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import paper_2501_11673_b200 as kpp
    from paper_2501_11673_b200 import build as kbuild
    kbuild.build()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = world > 1
    if dist:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=dev)
    iters = args.iters or DEFAULT_ITERS[cfg.name]

    A, b, _ = synth.make_problem(cfg, seed=0, device=dev)
    n = cfg.n
    if dist:
        cb, ce = kpp.column_slabs(n, world)[rank]
        A_loc = A[:, cb:ce].contiguous()
        uid = [kpp.kpp_get_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        if cfg.kind == "cdpp":
            ctx = kpp.cdpp_setup_dist(A_loc, n, cb, ce, cfg.s, cfg.lam, 0, uid[0], rank, world)
        else:
            ctx = kpp.kpp_setup_dist(A_loc, cfg.m, n, cb, ce, cfg.s, cfg.lam, 0, uid[0], rank, world)
        A_keep = A_loc
        del A
        n_local = ce - cb
    else:
        ctx = (kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup)(A, cfg.s, cfg.lam, 0)
        A_keep = A
        n_local = n
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream)
    if args.engine >= 0:
        ctx.set_option(kpp.OPT_ENGINE, args.engine)
    if args.proj:
        if cfg.kind != "kpp" or dist:
            raise SystemExit("--proj 1: single-GPU Kaczmarz++ configs only")
        ctx.set_option(kpp.OPT_PROJ, 1)
        ctx.set_option(kpp.OPT_TMAX, args.tmax)
    rht_ms = None
    if args.rht:
        ctx.enable_rht()  # one-time transform of A (not part of a step: the paper's Alg 5/3 line 2-3)
        rht_ms = ctx.stats()["rht_ms"]
    x_out = torch.empty(n_local, dtype=torch.float64, device=dev)

    def step():
        ctx.clear_cache()
        return ctx.solve(b, max_iters=iters, tol=0.0, x_out=x_out)

    def barrier():
        if dist:
            tdist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    ctx.reset_stats()
    launches = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    small = l2_small(cfg)
    flush = torch.empty(L2_FLUSH_BYTES // 8, dtype=torch.float64, device=dev) if small else None
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        if not small:
            ev0.record(stream)
            for _ in range(args.steps):
                res = step()
                launches += ctx.stats()["kernel_launches"]
            ev1.record(stream)
            torch.cuda.synchronize()
            barrier()
            ms = ev0.elapsed_time(ev1)
        else:  # A fits in L2: flush it before every step, outside the step's events
            ms = 0.0
            for _ in range(args.steps):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                ev0.record(stream)
                res = step()
                ev1.record(stream)
                torch.cuda.synchronize()
                ms += ev0.elapsed_time(ev1)
                launches += ctx.stats()["kernel_launches"]
            barrier()
    st = ctx.stats()
    if dist:
        t = torch.tensor([ms, st["phase2_ms"]], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms, p2max = float(t[0]), float(t[1])
    else:
        p2max = st["phase2_ms"]
    total_iters = args.steps * iters
    value = total_iters / (ms / 1e3)

    # warm Phase-2 rate (memo cache full): one more solve without clearing
    ctx.reset_stats()
    ctx.solve(b, max_iters=iters, tol=0.0, x_out=x_out)
    warm = ctx.stats()
    warm_rate = iters / (warm["phase2_ms"] / 1e3) if warm["phase2_ms"] > 0 else None

    # end to end through the C ABI with HOST buffers: H2D of b, D2H of x inside the timed region
    b_host = b.cpu().pin_memory()
    x_host = torch.empty(n_local, dtype=torch.float64).pin_memory()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.clear_cache()
        ctx.solve(b_host, max_iters=iters, tol=0.0, x_out=x_host)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e = {"value": total_iters / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * cfg.m,
           "d2h_bytes_per_step": 8 * n_local}

    ttt = None
    if not args.no_ttt:
        ctx.clear_cache()
        ctx.reset_stats()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        # c2 needs 19.3M iterations (DESIGN 12); multi-GPU runs keep a bounded 4M cap
        cap = args.ttt_cap or (1_000_000 if args.proj else 25_000_000 if world == 1 else 4_000_000)
        zeta = -(-(cfg.n if cfg.kind == "cdpp" else cfg.m) // cfg.s)
        # history sized for every checkpoint of the capped solve, so res_hist[-1] is the stopping one
        r = ctx.solve(b, max_iters=cap, tol=cfg.tol if cfg.tol > 0 else 1e-8, x_out=x_out,
                      hist_cap=cap // (2 * zeta) + 2)
        e1.record(stream)
        torch.cuda.synchronize()
        tms = e0.elapsed_time(e1)
        true_res = None
        if not dist:
            true_res = float(torch.linalg.vector_norm(A_keep @ x_out - b) / torch.linalg.vector_norm(b))
        ttt = {"seconds": tms / 1e3, "iters": r.iters, "converged": r.status == kpp.OK, "checkpoints": len(r.res_hist),
               "est_rel_res": float(r.res_hist[-1]) if len(r.res_hist) else None,
               "true_rel_res": true_res, "tol": 1e-8}

    if rank != 0:
        if dist:
            tdist.destroy_process_group()
        return

    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    peak_note = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if hbm_peak else "fallback 6650 GB/s"
    hbm_peak = hbm_peak or 6650.0
    bpi = bytes_per_iter(cfg, n_local)
    achieved = bpi * total_iters / (p2max / 1e3) / 1e9 if p2max > 0 else None
    # per launch: one persistent launch per window of min(iters, window) iterations
    iters_per_launch = min(iters, 8192)
    tr = ncu_traffic(cfg.name, "lsqr_persistent_kernel" if args.proj else "iterate_kernel")
    kname = ("lsqr_persistent_kernel (t_max + 1 exchange rounds per iteration)" if args.proj
             else "Phase-2 persistent kernel (iterate_kernel / cdpp_stream_kernel)")
    roof = {"bound": "hbm", "kernel": kname,
            "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": (achieved / hbm_peak) if achieved else None,
            "traffic": tr * iters_per_launch if tr else None,
            "traffic_note": "ncu dram read+write bytes per launch (per-iteration bytes from profiles/ncu_summary.json x iterations per launch)",
            "algorithmic_bytes_per_launch": bpi * iters_per_launch, "iters_per_launch": iters_per_launch,
            "peak_source": peak_note, "bytes_per_iter": bpi,
            "iter_kernel_share": p2max / ms if ms > 0 else None,
            # both HBM numbers, against the nominal 8 TB/s as well as the measured copy
            "frac_of_nominal_8tbs": (achieved / 8000.0) if achieved else None,
            "dram_gbs_ncu": (tr * total_iters / (p2max / 1e3) / 1e9) if (tr and p2max > 0) else None}
    cpu = None
    if not args.no_cpu and not dist:
        cpu = cpu_oracle_sample(cfg, A_keep.cpu().numpy(), b.cpu().numpy(), args.cpu_seconds, iters, args.proj,
                                args.tmax)
    elif not args.no_cpu and dist and rank == 0:
        cpu = None  # N>1: the oracle baseline is reported by the N=1 run only
    secondary = None
    if world == 1 and args.secondary and not args.proj and not args.rht:
        ctx.destroy()
        A = A_keep = None  # free the headline problem before the next one is generated
        torch.cuda.empty_cache()
        secondary = {}
        for nm in [c for c in args.secondary.split(",") if c and c != cfg.name]:
            with ClockSampler(local) as clk2:
                secondary[nm] = measure_secondary(nm, max(2, args.steps // 2), 2, dev, hbm_peak)
            secondary[nm]["clocks"] = clk2.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, iters, world, dist, args.proj, args.tmax),
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "phase1_ms_per_step": st["phase1_ms"] / args.steps,
        "phase2_ms_per_step": st["phase2_ms"] / args.steps,
        "warm_block_iters_per_s": warm_rate,
        "hbm_gbs_alg_warm": (bpi * iters / (warm["phase2_ms"] / 1e3) / 1e9) if warm["phase2_ms"] > 0 else None,
        "time_to_tol": ttt,
        "n_blocks_per_step": warm["n_blocks"],
        "n_refined_per_step": st.get("n_refined", 0) // max(1, args.steps),
        "phase1_fp64": (lambda fl, ms1: {"gflop_per_step": fl / 1e9,
                                          "tflops": fl / (ms1 / 1e3) / 1e12 if ms1 > 0 else None,
                                          "peak_tflops": FP64_DGEMM_TFLOPS,
                                          "frac": fl / (ms1 / 1e3) / 1e12 / FP64_DGEMM_TFLOPS if ms1 > 0 else None,
                                          "peak_source": "measured fp64 DGEMM (cuBLAS, DMMA 8x8x4)"})(
            phase1_flops(cfg, warm["n_blocks"], st.get("n_refined", 0) // max(1, args.steps)),
            st["phase1_ms"] / args.steps),
        "rht_preprocess_ms": rht_ms,
        "phase2_engine": {0: "persistent cluster kernel", 1: "step-kernel graph", 2: "fused-exchange kernel (dist.cu)",
                          3: "sketch + LSQR kernel"}.get(st.get("engine"), st.get("engine")),
        "exchange": ("NVLink peer buffers (fused)" if st.get("xchg") else "NCCL allreduce") if dist else None,
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
