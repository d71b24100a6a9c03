"""Multi-process host logic on CPU (gloo, world_size 2): batch sharding for the sweep and
synchronous data-parallel MGD.  The per-rank gradient comes from the oracle (test
infrastructure); the device path swaps in toc_glm_grad and NCCL.  DP-MGD with local batch B on G
ranks must equal the reference trainer at batch size B*G."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1702_06943_b200.distributed import DataParallelGLM, dp_step_plan, shard_range


def test_shard_range_covers():
    for n in (0, 1, 7, 1024, 8192):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("n_rows,local,world", [(1000, 250, 2), (1003, 64, 2), (999, 250, 4), (10, 4, 8)])
def test_dp_plan_union_is_global_batch(n_rows, local, world):
    plans = [dp_step_plan(n_rows, local, world, r) for r in range(world)]
    steps = len(plans[0].global_sizes)
    assert steps == (n_rows + local * world - 1) // (local * world)
    for t in range(steps):
        rows = sorted(x for p in plans for x in range(*p.local_rows[t]))
        g0 = t * local * world
        assert rows == list(range(g0, min(n_rows, g0 + local * world)))
        assert plans[0].global_sizes[t] == len(rows)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, payload, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O

        rp, c, v, y, m, local, lr, epochs, loss = payload
        order = O.shuffle_order(len(y), 0)
        plan = dp_step_plan(len(y), local, world, rank)
        trees = {}
        for t, (lo, hi) in enumerate(plan.local_rows):
            if hi > lo:
                idx = order[lo:hi]
                lens = np.diff(rp)[idx]
                brp = np.concatenate([[0], np.cumsum(lens)])
                g = np.concatenate([np.arange(rp[i], rp[i + 1]) for i in idx])
                trees[t] = (O.Tree.from_encoding(O.encode_csr(m, brp, c[g], v[g])), y[idx])

        def grad_fn(t, w):
            if t not in trees:
                return torch.zeros(m, dtype=torch.float64)
            tree, yy = trees[t]
            wn = w.numpy()
            z = tree.matvec(wn)
            s = (-yy / (1.0 + np.exp(yy * z))) if loss == "logistic" else (z - yy)
            return torch.from_numpy(tree.vecmat(s))

        def allreduce(g):
            dist.all_reduce(g, op=dist.ReduceOp.SUM)

        tr = DataParallelGLM(m, plan, lr, grad_fn, allreduce, torch.zeros(m, dtype=torch.float64))
        for _ in range(epochs):
            tr.epoch()
        q.put((rank, tr.w.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("loss", ["logistic", "squared"])
def test_dp_mgd_gloo_world2_matches_global_batch(oracle, loss):
    from paper_1702_06943_b200 import synth

    rp, c, v, y = synth.cfg3_dataset(3000, seed=31)
    if loss == "squared":
        y = y * 0.5 + 0.1
    world, local, lr, epochs = 2, 125, 0.05, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (rp, c, v, y, 68, local, lr, epochs, loss), q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w_ref, _ = oracle.train_glm(rp, c, v, y, 68, loss, local * world, lr, epochs, 0)
    for r in range(world):
        assert np.allclose(got[r], w_ref, rtol=1e-9, atol=1e-12), np.max(np.abs(got[r] - w_ref))
    assert np.array_equal(got[0], got[1])
