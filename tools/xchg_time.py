"""Per-iteration time of the column-sharded graph engine on ONE rank: fused NVLink-peer exchange
(KPP_OPT_XCHG=1, self-mapped) vs the NCCL allreduce between kernels (0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_11673_b200 as kpp  # noqa: E402
import synth  # noqa: E402

for name in sys.argv[1:] or ["c2", "c3"]:
    cfg = synth.CONFIGS[name]
    A, b, _ = synth.make_problem(cfg, device="cuda")
    uid = kpp.kpp_get_unique_id()
    if cfg.kind == "cdpp":
        ctx = kpp.cdpp_setup_dist(A, cfg.n, 0, cfg.n, cfg.s, cfg.lam, 0, uid, 0, 1)
    else:
        ctx = kpp.kpp_setup_dist(A, cfg.m, cfg.n, 0, cfg.n, cfg.s, cfg.lam, 0, uid, 0, 1)
    iters = 4096
    ctx.set_option(kpp.OPT_WINDOW, iters)
    ctx.set_option(kpp.OPT_ENGINE, 1)  # the multi-rank engine (one rank would run the persistent kernel)
    ctx.prepare(iters)
    for xchg in (1, 0, 1):
        ctx.set_option(kpp.OPT_XCHG, xchg)
        ctx.solve(b, max_iters=iters)
        ctx.reset_stats()
        ctx.solve(b, max_iters=iters)
        st = ctx.stats()
        print(f"{name}: xchg={st['xchg']} graph engine {st['phase2_ms'] * 1e3 / iters:.2f} us/iter", flush=True)
    ctx.destroy()
