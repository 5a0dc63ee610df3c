"""The sharded optimizer (paper_2506_10315_b200.dist) on the GPU: two ranks
share the box's single B200 (gloo carries the collectives; on a multi-GPU node
the same code runs NCCL), and the sharded step must equal the single-GPU
step -- bitwise in strict mode, within the fp32 tolerance in fast mode."""

import os
import socket

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SHAPES = [(256, 192), (256,), (96, 256), (96,), (33, 70), (1, 130), (7,), (1, 1, 64)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(seed=0):
    rng = np.random.default_rng(seed)
    init = [np.asarray(rng.standard_normal(s) * 0.05, np.float32) for s in SHAPES]
    grads = [[np.asarray(rng.standard_normal(s) * 1e-2, np.float32) for s in SHAPES]
             for _ in range(3)]
    return init, grads


def _worker(rank, world, port, mode, fs, q, gather="nccl", exchange_off_last=False,
            strategy="range"):
    import sys
    import traceback

    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist

        import paper_2506_10315_b200 as P
        from paper_2506_10315_b200.dist import ShardedLearnedOptimizer

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        init, grads = _init()
        params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
        opt = ShardedLearnedOptimizer(params, feature_set=fs, mode=mode, weight_decay=0.01,
                                      gather=gather, strategy=strategy)
        for k, gs in enumerate(grads):
            for p, g in zip(params, gs):
                p.grad = torch.from_numpy(g).cuda()
            if exchange_off_last and k == len(grads) - 1:
                opt.set_exchange(False)
            opt.step()
        torch.cuda.synchronize()
        out = [p.detach().cpu().numpy().copy() for p in params]
        if exchange_off_last:
            q.put((rank, out, list(opt.ranges)))
        else:
            q.put((rank, out, opt.local_state_bytes()))
        dist.destroy_process_group()
    except Exception:
        q.put((rank, traceback.format_exc(), 0))


@pytest.mark.parametrize("mode,fs,gather,strategy", [
    ("strict", "small_fc_lopt", "nccl", "range"),
    ("fast", "velo_mlp", "nccl", "range"),
    ("fast", "small_fc_lopt", "nccl", "range"),
    ("fast", "small_fc_lopt", "p2p", "range"),
    ("strict", "small_fc_lopt", "nccl", "owner"),
    ("strict", "velo_mlp", "nccl", "owner"),
    ("fast", "small_fc_lopt", "p2p", "owner")])
def test_sharded_equals_single_gpu(mode, fs, gather, strategy):
    """gather="p2p": the parameter arena mapped into the other rank (CUDA
    IPC), the apply kernel storing every updated parameter into it (the
    NVLink path; here both ranks map one device), one barrier instead of the
    all-gather.  strategy="owner": whole tensors per rank (FSDP_A2A), no
    factor/stats merge -- bitwise in strict mode like the range split."""
    import torch
    import torch.multiprocessing as mp

    import paper_2506_10315_b200 as P

    init, grads = _init()
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, feature_set=fs, mode=mode, weight_decay=0.01)
    for gs in grads:
        for p, g in zip(params, gs):
            p.grad = torch.from_numpy(g).cuda()
        opt.step()
    single = [p.detach().cpu().numpy() for p in params]
    full_state = sum(int(opt.state[p]["quad"].numel()) * 4 for p in params)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, fs, q, gather, False, strategy))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, out, state_bytes in res:
        assert not isinstance(out, str), out
        # optimizer state is sharded: each rank holds about half (slices are
        # rounded up to whole 128-element tiles; whole tensors per owner)
        bound = full_state // 2 + 16 * 128 + 4 * 4 * len(SHAPES)
        if strategy == "owner":
            bound = full_state // 2 + 16 * max(int(np.prod(s)) for s in SHAPES) + 16 * len(SHAPES)
        assert state_bytes <= bound
        for a, b in zip(out, single):
            if mode == "strict":
                assert a.tobytes() == b.tobytes()
            else:
                err = np.abs(a.astype(np.float64) - b) / (1 + np.abs(b))
                assert err.max() <= 1e-6, err.max()


@pytest.mark.parametrize("gather", ["nccl", "p2p"])
def test_exchange_off_updates_only_own_slice(gather):
    """set_exchange(False) (bench.py's without-all-gather timing, SURVEY.md
    §8(e)): a rank's own element range advances, the rest of its replica
    keeps the previous step's values."""
    import torch
    import torch.multiprocessing as mp

    import paper_2506_10315_b200 as P

    init, grads = _init()
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, mode="fast", weight_decay=0.01)
    snaps = []
    for gs in grads:
        for p, g in zip(params, gs):
            p.grad = torch.from_numpy(g).cuda()
        opt.step()
        snaps.append([p.detach().cpu().numpy().reshape(-1).copy() for p in params])

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, "fast", "small_fc_lopt", q, gather,
                                               True)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, out, ranges in res:
        assert not isinstance(out, str), out
        for a, new, old, (lo, hi) in zip(out, snaps[-1], snaps[-2], ranges):
            a = a.reshape(-1).astype(np.float64)
            own = np.zeros(a.size, bool)
            own[lo:hi] = True
            err = np.abs(a[own] - new[own]) / (1 + np.abs(new[own]))
            assert own.sum() == 0 or err.max() <= 1e-6
            err = np.abs(a[~own] - old[~own]) / (1 + np.abs(old[~own]))
            assert (~own).sum() == 0 or err.max() <= 1e-6


def _overlap_step_worker(rank, world, port, q):
    import sys
    import traceback

    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist

        from paper_2506_10315_b200.dist import ShardedLearnedOptimizer

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        model = _overlap_model()
        opt = ShardedLearnedOptimizer(model.parameters(), mode="strict", weight_decay=0.01,
                                      bucket_elems=1000)
        opt.overlap_grad_reduce(average=True)
        for step in range(2):
            x, y = _overlap_batch(rank, step)
            opt.zero_grad()
            torch.nn.functional.mse_loss(model(x), y).backward()
            opt.step()
        torch.cuda.synchronize()
        q.put((rank, [p.detach().cpu().numpy().copy() for p in model.parameters()],
               len(opt.buckets)))
        dist.destroy_process_group()
    except Exception:
        q.put((rank, traceback.format_exc(), 0))


def _overlap_model():
    import torch

    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(64, 96), torch.nn.ReLU(),
                               torch.nn.Linear(96, 33), torch.nn.ReLU(),
                               torch.nn.Linear(33, 10)).cuda()


def _overlap_batch(rank, step):
    import torch

    g = torch.Generator().manual_seed(1000 * step + rank)
    return (torch.randn(8, 64, generator=g).cuda(), torch.randn(8, 10, generator=g).cuda())


def test_backward_overlapped_reduce_scatter_step_bitwise():
    """Data-parallel training step fed straight from backward (SURVEY.md
    §8(f) rank 2): two ranks with different batches, bucketed gradient
    reduce-scatter launched from post-accumulate-grad hooks, sharded strict
    step -- bitwise equal to one process stepping with the mean gradient."""
    import torch
    import torch.multiprocessing as mp

    import paper_2506_10315_b200 as P

    model = _overlap_model()
    opt = P.LearnedOptimizer(model.parameters(), mode="strict", weight_decay=0.01)
    for step in range(2):
        gs = []
        for r in range(2):
            model.zero_grad()
            x, y = _overlap_batch(r, step)
            torch.nn.functional.mse_loss(model(x), y).backward()
            gs.append([p.grad.clone() for p in model.parameters()])
        for p, a, b in zip(model.parameters(), *gs):
            p.grad = (a + b) / 2
        opt.step()
    single = [p.detach().cpu().numpy() for p in model.parameters()]

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_step_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, out, nb in res:
        assert not isinstance(out, str), out
        assert nb > 1
        for a, b in zip(out, single):
            assert a.tobytes() == b.tobytes()


def _velo_worker(rank, world, port, mode, strategy, q):
    import sys
    import traceback

    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist

        from paper_2506_10315_b200.dist import ShardedVeLO

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        init, grads = _init()
        params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
        opt = ShardedVeLO(params, mode=mode, weight_decay=0.01, strategy=strategy)
        for k, gs in enumerate(grads):
            for p, g in zip(params, gs):
                p.grad = torch.from_numpy(g).cuda()
            # rank-local losses differ (each rank sees its own batch); the
            # hypernetwork must see their mean on every rank
            opt.step(loss=2.5 - 0.1 * k + (0.4 if rank == 0 else -0.4))
        torch.cuda.synchronize()
        q.put((rank, [p.detach().cpu().numpy().copy() for p in params]))
        dist.destroy_process_group()
    except Exception:
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("mode,strategy", [("strict", "range"), ("strict", "owner"),
                                           ("fast", "range")])
def test_sharded_velo_equals_single_gpu(mode, strategy):
    """The full VeLO optimizer sharded over two ranks with DIFFERENT local
    losses: every rank runs the per-tensor LSTM on the merged statistics and
    the mean loss, so all ranks mix the same MLPs and the result equals
    VeLO_CUDA on one GPU stepped with the mean loss (bitwise in strict mode)."""
    import torch
    import torch.multiprocessing as mp

    import paper_2506_10315_b200 as P

    init, grads = _init()
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.VeLO_CUDA(params, mode=mode, weight_decay=0.01)
    for k, gs in enumerate(grads):
        for p, g in zip(params, gs):
            p.grad = torch.from_numpy(g).cuda()
        opt.step(loss=2.5 - 0.1 * k)
    single = [p.detach().cpu().numpy() for p in params]

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_velo_worker, args=(r, 2, port, mode, strategy, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, out in res:
        assert not isinstance(out, str), out
        for a, b in zip(out, single):
            if mode == "strict":
                assert a.tobytes() == b.tobytes()
            else:
                err = np.abs(a.astype(np.float64) - b) / (1 + np.abs(b))
                assert err.max() <= 1e-6, err.max()


def _nccl_worker(port, q):
    """World size 1 over NCCL: every collective branch of dist.py runs on the
    real backend (all_reduce of the factor / stats / flag blocks,
    all_gather_into_tensor of the parameter arena, reduce_scatter_tensor of
    the gradient buckets from the backward hooks, the VeLO loss mean)."""
    import sys
    import traceback

    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist

        import paper_2506_10315_b200 as P
        from paper_2506_10315_b200.dist import ShardedLearnedOptimizer, ShardedVeLO

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
        assert dist.get_backend() == "nccl"
        init, grads = _init()
        results = {}
        for name in ("range", "owner", "bucketed", "velo", "single", "single_velo"):
            ps = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
            if name == "single":
                opt = P.LearnedOptimizer(ps, mode="fast", weight_decay=0.01)
            elif name == "single_velo":
                opt = P.VeLO_CUDA(ps, mode="fast", weight_decay=0.01)
            elif name == "velo":
                opt = ShardedVeLO(ps, mode="fast", weight_decay=0.01)
            elif name == "bucketed":
                opt = ShardedLearnedOptimizer(ps, mode="fast", weight_decay=0.01,
                                              bucket_elems=20000)
                opt.overlap_grad_reduce(average=True)
            else:
                opt = ShardedLearnedOptimizer(ps, mode="fast", weight_decay=0.01,
                                              strategy=name)
            for k, gs in enumerate(grads):
                if name == "bucketed":
                    # gradients produced by a backward pass: the hooks launch
                    # each bucket's NCCL reduce-scatter as it completes
                    opt.zero_grad()
                    loss = sum((p * torch.from_numpy(g).cuda()).sum() for p, g in zip(ps, gs))
                    loss.backward()
                else:
                    for p, g in zip(ps, gs):
                        p.grad = torch.from_numpy(g).cuda()
                if name in ("velo", "single_velo"):
                    opt.step(loss=2.0 - 0.1 * k)
                else:
                    opt.step()
            torch.cuda.synchronize()
            results[name] = [p.detach().cpu().numpy().copy() for p in ps]
        # explicit reduce-scatter entry point on the NCCL backend as well
        ps = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
        opt = ShardedLearnedOptimizer(ps, mode="fast")
        fg = opt.flat_grads()
        fg.fill_(2.0)
        sl = opt.reduce_scatter_grads(average=True)
        results["rs_ok"] = bool(torch.all(sl == 2.0).item())
        q.put(results)
        dist.destroy_process_group()
    except Exception:
        q.put(traceback.format_exc())


def test_nccl_world_size_one_runs_every_collective():
    """The NCCL code paths of dist.py (never executed by the gloo tests) on
    the box's GPU with a one-rank NCCL group: every sharded variant equals the
    single-GPU optimizer bitwise (one rank owns everything; the collectives
    are identities that must not corrupt anything)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    pr.start()
    res = q.get(timeout=600)
    pr.join(timeout=60)
    assert not isinstance(res, str), res
    assert res["rs_ok"]
    for name in ("range", "owner", "bucketed"):
        for a, b in zip(res[name], res["single"]):
            assert a.tobytes() == b.tobytes(), name
    for a, b in zip(res["velo"], res["single_velo"]):
        assert a.tobytes() == b.tobytes()
