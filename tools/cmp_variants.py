import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2501_11673_b200 as kpp, synth
cfg = synth.CONFIGS['c2']
A, b, _ = synth.make_problem(cfg, device='cuda')
for variant in ['plain', 'window2048', 'prepared', 'cluster0']:
    ctx = kpp.kpp_setup(A, cfg.s, cfg.lam, 0)
    if variant == 'window2048': ctx.set_option(kpp.OPT_WINDOW, 2048)
    if variant == 'cluster0': ctx.set_option(kpp.OPT_CLUSTER, 0)
    if variant == 'prepared': ctx.prepare(8192)
    ctx.solve(b, max_iters=8192)
    ctx.reset_stats()
    ctx.solve(b, max_iters=8192)
    st = ctx.stats()
    print(variant, f"{st['phase2_ms']*1e3/8192:.2f} us/iter", {k: st[k] for k in ('grid_ctas','cluster','resident','m_in_smem','tma','iter_launches')})
    ctx.destroy()
