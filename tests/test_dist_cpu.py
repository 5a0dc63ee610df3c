"""World-size-2 gloo tests of the sharded step's partition and merge algebra
(paper_2506_10315_b200/dist.py), on CPU with the oracle as the per-shard
compute -- the same checks the reference runs on its simulated strategies
(pkg/tests/test_distsim.py:126-167), here over real torch.distributed
collectives: flat-arena element ranges, f64 factor-sum all-reduce, f64
feature-sum all-reduce, parameter all-gather, result == single device."""

import os
import socket

import numpy as np
import pytest

from conftest import F32, ROOT

SHAPES = [(16, 98), (16,), (10, 16), (10,), (33, 70), (1, 130), (7,)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind_name, out_q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2506_10315_b200.dist import flat_shard_ranges
    from paper_2506_10315_b200.optim import view_2d

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kind = O.KIND_BY_NAME[kind_name]
        rng = np.random.default_rng(0)
        shapes2 = [view_2d(s) for s in SHAPES]
        params = [(rng.standard_normal(s) * 0.05).astype(F32) for s in shapes2]
        states = [O.OState.zeros(*s) for s in shapes2]
        for _ in range(2):   # warm the accumulators identically on every rank
            for j, s in enumerate(shapes2):
                states[j] = O.state_step(states[j], (rng.standard_normal(s) * 1e-2).astype(F32))
        grads = [(rng.standard_normal(s) * 1e-2).astype(F32) for s in shapes2]
        w = O.random_weights(39 if kind == O.SMALL_FC_LOPT else 29, seed=0)
        sizes = [m * n for m, n in shapes2]
        ranges, S, padded = flat_shard_ranges(sizes, world, rank)
        flat_out = np.zeros(padded, F32)
        mism = 0
        factor_mism = 0
        off = 0
        for j, ((m, n), (lo, hi)) in enumerate(zip(shapes2, ranges)):
            g = grads[j]
            s = states[j]
            # single-device reference for this tensor
            s_ref = O.state_step(s, g)
            ref_out, _, ref_sumsq = O.step_fused(params[j], g, s_ref, w, kind)
            # phase 0: f64 partial row/column sums over the local range
            idx = np.arange(lo, hi, dtype=np.int64)
            g2 = np.square(g.ravel()[lo:hi], dtype=np.float64)
            fs = np.concatenate([np.bincount(idx // n, weights=g2, minlength=m),
                                 np.bincount(idx % n, weights=g2, minlength=n)]).astype(np.float64)
            t = torch.from_numpy(fs)
            dist.all_reduce(t)
            fs = t.numpy()
            s2 = s.copy()
            row_mean, col_mean = (fs[:m] / n).astype(F32), (fs[m:] / m).astype(F32)
            for i in range(3):
                b = F32(O.DEFAULT_BETAS[4 + i])
                s2.r[i] = b * s.r[i] + (F32(1.0) - b) * row_mean
                s2.c[i] = b * s.c[i] + (F32(1.0) - b) * col_mean
                factor_mism += int(np.count_nonzero(s2.r[i] != s_ref.r[i]))
                factor_mism += int(np.count_nonzero(s2.c[i] != s_ref.c[i]))
                if factor_mism:
                    print("factor mismatch", rank, j, i, s2.r[i][:4], s_ref.r[i][:4], fs[:4], flush=True)
            s2.M = [a.copy() for a in s_ref.M]   # element-wise, identical by construction
            s2.V = s_ref.V.copy()
            s2.t = s_ref.t
            # phase 1: f64 feature sums over the local range, merged
            if hi > lo:
                part, _ = O.fused_stats(params[j], g, s2, kind, lo=lo, hi=hi)
            else:
                part = np.zeros(39 if kind == O.SMALL_FC_LOPT else 29)
            t = torch.from_numpy(np.ascontiguousarray(part))
            dist.all_reduce(t)
            sumsq = t.numpy()
            np.testing.assert_allclose(sumsq, ref_sumsq, rtol=1e-12)
            # phase 2 on the local range, into the flat arena
            out = params[j].copy()
            if hi > lo:
                O.fused_apply(params[j], g, s2, w, kind, sumsq, m * n, lo=lo, hi=hi, out=out)
            flat_out[off + lo:off + hi] = out.ravel()[lo:hi]
            off += m * n
        # parameter gather: every rank contributes its slice of the arena
        local = torch.from_numpy(flat_out[rank * S:(rank + 1) * S].copy())
        chunks = [torch.empty(S) for _ in range(world)]
        dist.all_gather(chunks, local)
        full = torch.cat(chunks).numpy()
        off = 0
        for j, (m, n) in enumerate(shapes2):
            s_ref = O.state_step(states[j], grads[j])
            ref_out, _, _ = O.step_fused(params[j], grads[j], s_ref, w, kind)
            mism += int(np.count_nonzero(full[off:off + m * n] != ref_out.ravel()))
            off += m * n
        out_q.put((rank, mism + factor_mism, [(lo, hi) for lo, hi in ranges]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind_name", ["small_fc_lopt", "velo_mlp"])
def test_sharded_step_equals_single_device_gloo_world2(oracle, kind_name):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind_name, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mism, ranges in results:
        assert mism == 0, (rank, mism)
    # the two ranks' ranges tile every tensor exactly once
    by_rank = {r: rg for r, _, rg in results}
    from paper_2506_10315_b200.optim import view_2d

    for j, s in enumerate(SHAPES):
        m, n = view_2d(s)
        covered = sum(hi - lo for lo, hi in (by_rank[0][j], by_rank[1][j]))
        assert covered == m * n


def test_flat_shard_ranges_partition():
    from paper_2506_10315_b200.dist import flat_shard_ranges, owner_plan, worker_ranges

    sizes = [590592, 768, 151296, 7, 1, 2359296, 3]
    for world in (1, 2, 3, 8):
        total = 0
        for r in range(world):
            ranges, S, padded = flat_shard_ranges(sizes, world, r)
            assert padded % world == 0 and S * world == padded
            total += sum(hi - lo for lo, hi in ranges)
            for (lo, hi), n in zip(ranges, sizes):
                assert 0 <= lo <= hi <= n
        assert total == sum(sizes)
    r = worker_ranges(10, 27, 4)
    assert r[0][0] == 10 and r[-1][1] == 27
    assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1
    owners = owner_plan([5, 100, 7, 60, 60], 2)
    assert owners[1] == 0 and sorted(set(owners)) == [0, 1]


def _rs_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_10315_b200.dist import ShardedLearnedOptimizer

        rng = np.random.default_rng(0)
        params = [torch.nn.Parameter(torch.from_numpy((rng.standard_normal(s) * 0.05).astype(F32)))
                  for s in SHAPES]
        opt = ShardedLearnedOptimizer(params)
        # rank-dependent local gradients, accumulated into the gradient arena
        lrng = np.random.default_rng(100 + rank)
        fg = opt.flat_grads()
        local_g = [(lrng.standard_normal(s) * 1e-2).astype(F32) for s in SHAPES]
        for p, g in zip(params, local_g):
            p.grad.copy_(torch.from_numpy(g))
        sl = opt.reduce_scatter_grads(average=True).clone()
        q.put((rank, opt.slice_len, [g.reshape(-1) for g in local_g], sl.numpy()))
    except Exception:
        import traceback
        q.put((rank, -1, traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


def test_reduce_scatter_grads_gloo_world2():
    """Each rank ends up with the mean of all ranks' gradients on exactly its
    own slice of the flat arena (what the sharded step reads)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rs_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] > 0, r[2]
    S = res[0][1]
    flat = [np.concatenate(r[2]) for r in res]
    mean = (flat[0] + flat[1]) / np.float32(2)
    mean = np.concatenate([mean, np.zeros(2 * S - mean.size, np.float32)])
    for rank, _, _, sl in res:
        np.testing.assert_allclose(sl, mean[rank * S:(rank + 1) * S], rtol=0, atol=1e-9)


def test_owner_layout_partitions_the_arena():
    """FSDP_A2A ownership (distsim.py:109-118): greedy largest-first owners;
    the arena puts each owner's tensors in its own slice, disjoint, and every
    tensor is stepped by exactly one rank."""
    from paper_2506_10315_b200.dist import owner_layout, owner_plan

    sizes = [2359296, 768, 589824, 3, 1, 2304, 50257 * 1024, 7]
    for world in (1, 2, 3, 8):
        owner = owner_plan(sizes, world)
        loads = [sum(n for n, w in zip(sizes, owner) if w == r) for r in range(world)]
        assert max(loads) - min(loads) <= max(sizes)
        seen = np.zeros(world * max(128, (max(loads) + 127) // 128 * 128), np.int32)
        for rank in range(world):
            ranges, offsets, S, padded = owner_layout(sizes, owner, world, rank)
            assert S % 128 == 0 and padded == world * S
            for n, w, (lo, hi), off in zip(sizes, owner, ranges, offsets):
                assert (lo, hi) == ((0, n) if w == rank else (0, 0))
                assert w * S <= off and off + n <= (w + 1) * S
                if w == rank:
                    seen[off:off + n] += 1
        assert seen.max() == 1 and seen.sum() == sum(sizes)


def test_bucketed_layout_single_bucket_is_flat_layout():
    from paper_2506_10315_b200.dist import bucketed_layout, flat_shard_ranges

    sizes = [int(np.prod(s)) for s in SHAPES]
    for world in (1, 2, 3, 4):
        for rank in range(world):
            r0, S, padded = flat_shard_ranges(sizes, world, rank)
            r1, offsets, buckets, padded1 = bucketed_layout(sizes, world, rank)
            assert r0 == r1 and padded == padded1 and buckets[0][1] == S
            assert offsets == list(np.cumsum([0] + sizes[:-1]))


def test_bucketed_layout_partitions_every_bucket():
    from paper_2506_10315_b200.dist import bucketed_layout

    sizes = [int(np.prod(s)) for s in SHAPES] + [1, 5000, 129]
    order = list(reversed(range(len(sizes))))
    for world in (1, 2, 4):
        cover = {}
        for rank in range(world):
            ranges, offsets, buckets, padded = bucketed_layout(sizes, world, rank, 300, order)
            assert sum(len(b[2]) for b in buckets) == len(sizes)
            for base, S, tl in buckets:
                assert S % 128 == 0
                for j in tl:   # a tensor lies inside its bucket's segment
                    assert base <= offsets[j] and offsets[j] + sizes[j] <= base + world * S
            for j, (lo, hi) in enumerate(ranges):
                for e in range(lo, hi):
                    cover[(j, e)] = cover.get((j, e), 0) + 1
        assert len(cover) == sum(sizes) and max(cover.values()) == 1


def _overlap_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_10315_b200.dist import ShardedLearnedOptimizer

        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.ReLU(),
                                    torch.nn.Linear(32, 8))
        opt = ShardedLearnedOptimizer(model.parameters(), bucket_elems=200)
        opt.overlap_grad_reduce(average=True)
        g = torch.Generator().manual_seed(10 + rank)
        x, y = torch.randn(4, 16, generator=g), torch.randn(4, 8, generator=g)
        model.zero_grad()   # Module.zero_grad sets grads to None: the hooks re-home them
        torch.nn.functional.mse_loss(model(x), y).backward()
        launched = len(opt._rs_hooks["works"])   # buckets reduced during backward
        opt._finish_grad_reduce()
        ps = list(model.parameters())
        out = [(opt.offsets[j], opt.state[p]["range"], p.grad.detach().reshape(-1).clone().numpy())
               for j, p in enumerate(ps)]
        q.put((rank, launched, len(opt.buckets), out))
    except Exception:
        import traceback
        q.put((rank, -1, -1, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_reduce_scatter_overlapped_with_backward_gloo_world2():
    """§8(f) rank 2: gradient buckets are reduce-scattered from inside
    backward (post-accumulate-grad hooks); afterwards each rank holds the
    mean gradient on its own element range of every tensor."""
    import torch
    import torch.multiprocessing as mp

    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.ReLU(), torch.nn.Linear(32, 8))
    grads = []
    for r in range(2):
        model.zero_grad()
        g = torch.Generator().manual_seed(10 + r)
        x, y = torch.randn(4, 16, generator=g), torch.randn(4, 8, generator=g)
        torch.nn.functional.mse_loss(model(x), y).backward()
        grads.append([p.grad.reshape(-1).clone().numpy() for p in model.parameters()])
    mean = [(a + b) / np.float32(2) for a, b in zip(*grads)]

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    for rank, launched, nb, out in res:
        assert launched >= 0, out
        assert nb > 1 and launched == nb
        for (off, (lo, hi), g), m in zip(out, mean):
            np.testing.assert_allclose(g[lo:hi], m[lo:hi], rtol=1e-6, atol=1e-9)


def _guard_worker(rank, world, port, q):
    """Accumulating a second backward into buckets whose reduce-scatter was
    already launched must raise (it would race with the collective and
    double-count); a state_dict saved by the other rank must not load."""
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        from paper_2506_10315_b200.dist import ShardedLearnedOptimizer
        from paper_2506_10315_b200.optim import OptimError

        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.ReLU(),
                                    torch.nn.Linear(32, 8))
        opt = ShardedLearnedOptimizer(model.parameters(), bucket_elems=200)
        opt.overlap_grad_reduce(average=True)
        x, y = torch.randn(4, 16), torch.randn(4, 8)
        torch.nn.functional.mse_loss(model(x), y).backward()
        try:
            torch.nn.functional.mse_loss(model(x), y).backward()
            out["accum"] = "no error"
        except RuntimeError as e:
            out["accum"] = "raised" if "accumulation" in str(e) else str(e)
        # zero_grad waits for / clears the outstanding bucket reductions
        opt.zero_grad()
        torch.nn.functional.mse_loss(model(x), y).backward()
        out["after_zero"] = len(opt._rs_hooks["works"]) == len(opt.buckets)
        # checkpoint layout check
        mine = opt.state_dict()
        objs = [None] * world
        dist.all_gather_object(objs, mine)
        other = objs[1 - rank]
        try:
            opt.load_state_dict(other)
            out["foreign"] = "loaded"
        except OptimError:
            out["foreign"] = "raised"
        opt.load_state_dict(objs[rank])
        out["own"] = "loaded"
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_overlap_guard_and_sharded_state_layout_check_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_guard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    for rank, out in res:
        assert isinstance(out, dict), out
        assert out == {"accum": "raised", "after_zero": True, "foreign": "raised",
                       "own": "loaded"}, out
