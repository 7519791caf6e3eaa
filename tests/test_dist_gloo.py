"""World-size-2 `gloo` tests of the column-sharded (multi-GPU) decomposition on CPU.

The product's N>1 path (include/kpp.h kpp_setup_dist / cdpp_setup_dist, DESIGN.md section 8,
SURVEY 8(e)) shards A by contiguous column slabs, replicates b, the block schedule and rho,
and exchanges exactly one s-vector per iteration (the partial block residual A_p[S,:] x_p)
plus, per fresh block, the s x s Gram partial (K++) or the disjoint-support principal block
(CD++).  NCCL needs GPUs, so here the same exchange runs over gloo between two CPU processes
and the sharded iterates are compared with the unsharded oracle.  This pins the host-side
partition (`column_slabs`) and the decomposition the CUDA path implements, and checks that
the reduced vectors are bit-identical on every rank (the replicated stop / rho decisions
depend on it).
"""
from __future__ import annotations

import os
import socket
import zlib

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as ora_mod
import synth
from paper_2501_11673_b200 import column_slabs


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allreduce(v: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _same_bits_everywhere(v: np.ndarray) -> bool:
    h = torch.tensor([zlib.crc32(v.tobytes())], dtype=torch.int64)  # process-independent
    hs = [torch.zeros_like(h) for _ in range(dist.get_world_size())]
    dist.all_gather(hs, h)
    return all(int(x) == int(hs[0]) for x in hs)


def _sharded_run(kind, A_loc, b, cb, ce, n, s, lam, seed, T, eta, rho):
    """Sharded K++ / CD++ with a fixed rho (Eq (momentum), Alg 5 / Alg 3 with Gram /
    principal-block factors), exchanging only what SURVEY 8(e) lists."""
    m = b.shape[0]
    pop = n if kind == "cdpp" else m
    C = ora_mod.cdpp_C(n, s) if kind == "cdpp" else ora_mod.kpp_C(m, n, s)
    bid, fresh, _ = ora_mod.schedule(seed, C, T)
    factors = {}
    x = np.zeros(ce - cb)
    mom = np.zeros(ce - cb)
    c = (1.0 - rho) / (1.0 + rho)
    ok_bits = True
    nb = 0
    for t in range(T):
        if fresh[t]:
            S = ora_mod.fresh_block(seed, pop, s, nb)
            if kind == "cdpp":
                # each rank fills A[S, S ∩ cols_p], zeros elsewhere: disjoint supports sum exactly
                G = np.zeros((s, s))
                for j, col in enumerate(S):
                    if cb <= col < ce:
                        G[:, j] = A_loc[S, col - cb]
                G = _allreduce(G)
            else:
                G = _allreduce(A_loc[S, :] @ A_loc[S, :].T)
            ok_bits &= _same_bits_everywhere(G)
            R = np.linalg.cholesky(G + lam * np.eye(s)).T
            factors[nb] = (S, R)
            nb += 1
        S, R = factors[int(bid[t])]
        q = _allreduce(A_loc[S, :] @ x)          # the one s-vector exchange of the iteration
        ok_bits &= _same_bits_everywhere(q)
        r = q - b[S]
        y = np.linalg.solve(R, np.linalg.solve(R.T, r))
        if kind == "cdpp":
            w = np.zeros(ce - cb)
            for k, col in enumerate(S):
                if cb <= col < ce:
                    w[col - cb] = y[k]
        else:
            w = A_loc[S, :].T @ y
        mom = c * (mom - w)
        x = x - w + eta * mom
    return x, ok_bits


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if kind == "cdpp":
            cfg = synth.twin("c5", 96, 96, 16, k=6)
        else:
            cfg = synth.twin("c2", 96, 80, 16, k=6)
        A, b, _ = synth.make_problem(cfg)
        A, b = A.numpy(), b.numpy()
        n = A.shape[1]
        cb, ce = column_slabs(n, world)[rank]
        eta = cfg.s / (2.0 * n)
        x_loc, ok_bits = _sharded_run(kind, A[:, cb:ce].copy(), b, cb, ce, n, cfg.s, cfg.lam, 0, 120, eta, 0.3)
        parts = [None] * world
        dist.all_gather_object(parts, (cb, ce, x_loc, ok_bits))
        if rank == 0:
            q.put(parts)
    except Exception:
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _run_world(kind, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    assert not (isinstance(parts, tuple) and parts[0] == "error"), parts
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return parts


def test_column_slabs_partition_world2():
    for n in (1, 7, 80, 131072):
        sl = column_slabs(n, 2)
        assert sl[0][0] == 0 and sl[-1][1] == n and sl[0][1] == sl[1][0]
        assert all(e - b >= 0 for b, e in sl)


@pytest.mark.parametrize("kind", ["kpp", "cdpp"])
def test_sharded_matches_oracle_world2(kind):
    """Two gloo ranks, column-sharded, vs the unsharded oracle (Gram factor route, fixed rho)."""
    parts = _run_world(kind)
    parts.sort(key=lambda p: p[0])
    x = np.concatenate([p[2] for p in parts])
    assert all(p[3] for p in parts), "allreduced vectors differ between ranks"
    if kind == "cdpp":
        cfg = synth.twin("c5", 96, 96, 16, k=6)
    else:
        cfg = synth.twin("c2", 96, 80, 16, k=6)
    A, b, _ = synth.make_problem(cfg)
    run = ora_mod.cdpp_run if kind == "cdpp" else ora_mod.kpp_run
    kw = {} if kind == "cdpp" else {"factor": ora_mod.GRAM}
    ref = run(A.numpy(), b.numpy(), cfg.s, lam=cfg.lam, seed=0, max_iters=120, rho_fixed=0.3, **kw)
    err = np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x)
    assert err <= 1e-10, err
