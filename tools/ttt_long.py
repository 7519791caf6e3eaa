import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2501_11673_b200 as kpp, synth
cfg = synth.CONFIGS['c2']
A, b, _ = synth.make_problem(cfg, seed=0, device='cuda')
ctx = kpp.kpp_setup(A, cfg.s, cfg.lam, 0)
t = time.time()
r = ctx.solve(b, max_iters=int(sys.argv[1]), tol=1e-8, hist_cap=1 << 20)
torch.cuda.synchronize()
h = r.res_hist.numpy()
print('status', r.status, 'iters', r.iters, 'time %.1f s' % (time.time() - t))
idx = np.unique(np.geomspace(1, len(h), 25).astype(int)) - 1
zeta = (cfg.m + cfg.s - 1) // cfg.s
for i in idx: print(' it %9d  res %.3e  rho %.4f' % ((i + 1) * 2 * zeta, h[i], ctx.rho_history().numpy()[i] if i < len(ctx.rho_history()) else float('nan')))
x = r.x
print('true', float(torch.linalg.vector_norm(A @ x - b) / torch.linalg.vector_norm(b)))
