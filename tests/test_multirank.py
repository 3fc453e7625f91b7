"""Multi-rank photon-batch sharding on CPU (gloo, world_size 2).

Mirrors bench.py's N-GPU path: each rank accumulates the fixed-point tallies
of its contiguous share of the history range (here with the CPU oracle's
accumulator, which has the device layout), the buffers are sum-reduced, and
rank 0 finalizes with the product's host finalize.  The result must be
bit-identical to a single-rank run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A
import cases


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import oracle_lib
    orc = oracle_lib.oracle()
    ph, g, angle, spec, resp, cfg = cases.poly(1)
    L = A.accum_layout(g.nu, g.nv, spec.n_bins, cfg.track_variance)
    n = X.history_count(spec, cfg.photons_total)
    acc = np.zeros(L["words"], np.uint64)
    orc.accumulate_range(ph, g, angle, spec, resp, cfg, n * rank // ws, n * (rank + 1) // ws, acc)
    t = torch.from_numpy(acc.view(np.int64).copy())
    dist.reduce(t, dst=0, op=dist.ReduceOp.SUM)  # two's-complement sum == u64 sum
    if rank == 0:
        r = X.finalize_host(g, spec, cfg, t.numpy().view(np.uint64), 0, n)
        out_q.put((r.image.copy(), r.variance.copy(), r.total, r.total_std_error,
                   r.histories, t.numpy().view(np.uint64).copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_reduce_is_bit_identical(orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    img, var, total, se, hist, acc2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ph, g, angle, spec, resp, cfg = cases.poly(1)
    L = A.accum_layout(g.nu, g.nv, spec.n_bins, cfg.track_variance)
    n = X.history_count(spec, cfg.photons_total)
    acc1 = np.zeros(L["words"], np.uint64)
    orc.accumulate_range(ph, g, angle, spec, resp, cfg, 0, n, acc1)
    assert np.array_equal(acc1, acc2)
    one = X.finalize_host(g, spec, cfg, acc1, 0, n)
    assert np.array_equal(one.image, img) and np.array_equal(one.variance, var)
    assert one.total == total and one.total_std_error == se and one.histories == hist == n


def _gpu_worker(rank, ws, port, out_q):
    """Two processes on the box's one GPU: each runs the DEVICE transport on its
    photon batch (xs_scatter_accumulate_device), the device-produced limb
    buffers cross the process boundary through a gloo reduce, rank 0 finalizes
    on its device (xs_scatter_finalize_device)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    ph, g, angle, spec, resp, cfg = cases.poly(1)
    proj = X.Projector(ph, resp, ctx=X.Context(0))
    L = A.accum_layout(g.nu, g.nv, spec.n_bins, cfg.track_variance)
    n = X.history_count(spec, cfg.photons_total)
    acc = torch.zeros(L["words"], dtype=torch.int64, device="cuda")
    proj.accumulate(g, angle, spec, cfg, n * rank // ws, n * (rank + 1) // ws, acc.data_ptr())
    t = acc.cpu()
    dist.reduce(t, dst=0, op=dist.ReduceOp.SUM)
    if rank == 0:
        acc.copy_(t)
        torch.cuda.synchronize()
        r = proj.finalize(g, spec, cfg, acc.data_ptr(), 0, n)
        one = proj.scatter_stats(g, angle, spec, cfg)
        out_q.put((np.array_equal(r.image, one.image), np.array_equal(r.variance, one.variance),
                   r.total == one.total, r.ledger == one.ledger))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_process_device_batches_bit_identical():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(res), res
