"""Profiling driver: one warm solve of `iters` iterations on a config (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_11673_b200 as kpp  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--cluster", type=int, default=0)
ap.add_argument("--ygl", type=int, default=-1)
ap.add_argument("--reassoc", type=int, default=1)
ap.add_argument("--rht", action="store_true")
ap.add_argument("--proj", type=int, default=0)
ap.add_argument("--tmax", type=int, default=8)
ap.add_argument("--vranks", type=int, default=1, help="emulated column-sharded ranks (engine 2 / CD++ stream)")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
A, b, _ = synth.make_problem(cfg, device="cuda")
ctx = (kpp.cdpp_setup if cfg.kind == "cdpp" else kpp.kpp_setup)(A, cfg.s, cfg.lam, 0)
ctx.set_option(kpp.OPT_ENGINE, a.engine)
ctx.set_option(kpp.OPT_CLUSTER, a.cluster)
ctx.set_option(kpp.OPT_YGL, a.ygl)
if cfg.kind == 'cdpp':
    ctx.set_option(kpp.OPT_REASSOC, a.reassoc)
if a.vranks > 1:
    ctx.set_option(kpp.OPT_VRANKS, a.vranks)
if a.proj:
    ctx.set_option(kpp.OPT_PROJ, a.proj)
    ctx.set_option(kpp.OPT_TMAX, a.tmax)
if a.rht:
    ctx.enable_rht()
    torch.cuda.synchronize()
    st0 = ctx.stats()
    mb = A.numel() * 8 / 1e6
    print(f"{a.config}: RHT preprocessing {st0['rht_ms']:.2f} ms  (matrix {mb:.0f} MB)", flush=True)
ctx.set_option(kpp.OPT_WINDOW, a.iters)
ctx.prepare(a.iters)
st1 = ctx.stats()
print(f"{a.config}: phase1 {st1['phase1_ms']:.2f} ms for {st1['n_blocks']} blocks", flush=True)
for _ in range(a.reps):
    ctx.reset_stats()
    r = ctx.solve(b, max_iters=a.iters)
    st = ctx.stats()
    print(f"{a.config}: {a.iters} iters phase2 {st['phase2_ms']:.3f} ms -> {st['phase2_ms'] * 1e3 / a.iters:.2f} us/iter; "
          f"plan grid={st['grid_ctas']} C={st['cluster']} resident={st['resident']} msm={st['m_in_smem']} tma={st['tma']} ygl={st['ygl']} reassoc={st['reassoc']}")
