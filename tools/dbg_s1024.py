import sys, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2501_11673_b200 as kpp, synth
cfg = synth.twin("c3", 2048, 1100, 1024, k=8)
A, b, _ = synth.make_problem(cfg)
for opts in [dict(), dict(OPT_ENGINE=1), dict(OPT_RESIDENT=0), dict(OPT_YGL=1), dict(OPT_YGL=0), dict(OPT_CLUSTER=2), dict(OPT_CLUSTER=8)]:
    ctx = kpp.kpp_setup(A.cuda(), cfg.s, cfg.lam, 0)
    try:
        for k, v in opts.items(): ctx.set_option(getattr(kpp, k), v)
        st = ctx.stats()
        r = ctx.solve(b.cuda(), max_iters=40)
        print(opts, "ok", {k: st[k] for k in ("grid_ctas", "cluster", "resident", "m_in_smem", "tma", "ygl")}, flush=True)
    except Exception as e:
        print(opts, "FAIL", str(e)[:150], {k: st[k] for k in ("grid_ctas", "cluster", "resident", "m_in_smem", "tma", "ygl")}, flush=True)
        break
