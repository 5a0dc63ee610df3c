"""Data-parallel sharded optimizer step over torch.distributed (NCCL on GPUs).

The reference simulates three strategies in distsim.py; this module runs two
of them for real.  strategy="range" is REDUCE_SCATTER (distsim.py:403-534):

  * parameters are flattened into one arena (like ZeRO / FSDP flat params) and
    rank r owns the contiguous slice [r*S, (r+1)*S) of it; for every tensor
    this yields an element range [lo, hi) (possibly empty), so optimizer state
    is held for 1/N of the elements only;
  * phase 0 computes f64 partial row/column sums of g^2 over the local
    elements; one all-reduce (sum, float64) of the contiguous factor block
    merges them -- the "factor merge" of distsim.py:427-476;
  * phase 1 computes f64 feature sums over the local elements; one all-reduce
    of the [tensors x d_feat] block merges them -- the "stats merge",
    normalization_across_shards (distsim.py:598-610);
  * phase 2 updates the local slice in place; one all-gather of the flat
    parameter arena (in place, NCCL over NVLink) replaces the "parameter
    gather" (distsim.py:523-530).

Merging f64 partials reproduces the single-device f32 factors and scales
(SURVEY.md Appendix A), so the sharded step matches the 1-GPU step.

strategy="owner" is FSDP_A2A (distsim.py:536-595): every tensor is stepped
whole by one owner (greedy largest-first, distsim.py:109-118), so there is no
factor or stats merge -- only the one-word non-finite-gradient flag is
all-reduced, keeping the step all-or-nothing across ranks.  The arena is laid
out owner by owner (rank r's tensors in [r*S, (r+1)*S)), so the same in-place
all-gather (or the fused peer stores) redistributes the parameters.  Balance
is limited by the largest tensor.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .engine import Slot, StepPlan
from .optim import LearnedOptimizer, view_2d


def worker_ranges(lo: int, hi: int, workers: int):
    """engine.py:597-605: split [lo, hi) into `workers` ranges, sizes within 1."""
    if workers < 1:
        raise ValueError("worker count must be >= 1")
    span = hi - lo
    b = [lo + span * w // workers for w in range(workers + 1)]
    return [(b[w], b[w + 1]) for w in range(workers)]


def flat_shard_ranges(sizes, world: int, rank: int):
    """Per-tensor local ranges of rank `rank` when the concatenation of the
    tensors (in order) is cut into `world` equal contiguous slices (the arena
    is padded to a multiple of 128 * `world`).  Returns (ranges, slice_len, padded)."""
    total = int(sum(sizes))
    # slices are whole multiples of 128 elements, so shard boundaries fall on
    # tile boundaries of the fast path (16-byte aligned bulk copies)
    unit = world * 128
    padded = (total + unit - 1) // unit * unit
    S = padded // world
    s0, s1 = rank * S, (rank + 1) * S
    out, off = [], 0
    for n in sizes:
        lo, hi = max(off, s0) - off, min(off + n, s1) - off
        out.append((lo, hi) if hi > lo else (0, 0))
        off += n
    return out, S, padded


def bucketed_layout(sizes, world: int, rank: int, bucket_elems=None, order=None):
    """Element-range layout with gradient buckets: tensors (in `order`, by
    default parameter order) are grouped into buckets of at least
    `bucket_elems` elements (None: one bucket), each bucket is padded to a
    multiple of 128 * world and cut into `world` equal portions, rank r
    stepping portion r of every bucket.  A tensor lies in one bucket, so it
    still gets a single (possibly empty) element range per rank, and each
    bucket's gradient reduce-scatter / parameter all-gather is one in-place
    collective on a contiguous arena segment.  With one bucket this is
    flat_shard_ranges' layout.  Returns (ranges, offsets, buckets, padded),
    buckets = [(base, portion_len, tensor indices)]."""
    n = len(sizes)
    order = list(range(n)) if order is None else [int(j) for j in order]
    groups = [order]
    if bucket_elems is not None:
        groups, cur, acc = [], [], 0
        for j in order:
            cur.append(j)
            acc += sizes[j]
            if acc >= bucket_elems:
                groups.append(cur)
                cur, acc = [], 0
        if cur:
            groups.append(cur)
    unit = world * 128
    offsets, ranges, buckets = [0] * n, [(0, 0)] * n, []
    base = 0
    for tl in groups:
        tot = sum(sizes[j] for j in tl)
        seg = max(unit, (tot + unit - 1) // unit * unit)
        S = seg // world
        s0, s1 = base + rank * S, base + (rank + 1) * S
        off = base
        for j in tl:
            offsets[j] = off
            lo, hi = max(off, s0) - off, min(off + sizes[j], s1) - off
            ranges[j] = (lo, hi) if hi > lo else (0, 0)
            off += sizes[j]
        buckets.append((base, S, list(tl)))
        base += seg
    return ranges, offsets, buckets, base


def owner_layout(sizes, owner, world: int, rank: int):
    """Arena layout of the ownership strategy: rank r's tensors (in tensor
    order) packed from r*S, S = the largest owner total rounded up to 128.
    Returns (ranges, offsets, S, padded): this rank steps (0, n) of the
    tensors it owns and the empty range of the others."""
    load = [0] * world
    for n, w in zip(sizes, owner):
        load[w] += n
    S = max(128, (max(load) + 127) // 128 * 128)
    cursor = [r * S for r in range(world)]
    offsets, ranges = [], []
    for n, w in zip(sizes, owner):
        offsets.append(cursor[w])
        cursor[w] += n
        ranges.append((0, n) if w == rank else (0, 0))
    return ranges, offsets, S, world * S


def owner_plan(sizes, workers: int):
    """distsim.py:109-118 FSDP_A2A ownership: greedy largest-first."""
    order = sorted(range(len(sizes)), key=lambda j: -sizes[j])
    load = [0] * workers
    owner = [0] * len(sizes)
    for j in order:
        w = min(range(workers), key=lambda i: (load[i], i))
        owner[j] = w
        load[w] += sizes[j]
    return owner


class ShardedLearnedOptimizer(LearnedOptimizer):
    """LearnedOptimizer whose step is sharded by element ranges across the
    ranks of the default process group.  Parameters must be identical on all
    ranks at construction; gradients are expected to be already reduced
    (e.g. DDP), of which each rank reads only its own slice."""

    def __init__(self, params, *args, process_group=None, gather: str = "nccl",
                 strategy: str = "range", bucket_elems=None, **kw):
        super().__init__(params, *args, **kw)
        self.pg = process_group
        self.world = dist.get_world_size(self.pg)
        self.rank = dist.get_rank(self.pg)
        if len(self.param_groups) != 1:
            raise ValueError("the sharded step supports one parameter group")
        if gather not in ("nccl", "p2p"):
            raise ValueError(f"unknown gather {gather!r}")
        if strategy not in ("range", "owner"):
            raise ValueError(f"unknown strategy {strategy!r}")
        self.gather = gather
        self.strategy = strategy
        self.exchange = True
        ps = self.param_groups[0]["params"]
        sizes = [p.numel() for p in ps]
        if strategy == "range":
            # buckets in reverse parameter order: roughly the order backward
            # produces the gradients (what DDP's bucketing assumes)
            order = None if bucket_elems is None else list(reversed(range(len(sizes))))
            ranges, offsets, buckets, padded = bucketed_layout(sizes, self.world, self.rank,
                                                               bucket_elems, order)
        else:
            if bucket_elems is not None:
                raise ValueError("gradient buckets need strategy='range'")
            self.owner = owner_plan(sizes, self.world)
            ranges, offsets, S, padded = owner_layout(sizes, self.owner, self.world, self.rank)
            buckets = [(0, S, list(range(len(sizes))))]
        self.buckets = buckets
        self.offsets = [int(o) for o in offsets]
        dev = ps[0].device
        self._peers = None
        if gather == "p2p":
            # every rank maps every other rank's parameter arena (CUDA IPC;
            # NVLink peer access between GPUs) and the apply kernel stores each
            # updated parameter into all of them, so no all-gather is launched
            from torch.multiprocessing.reductions import reduce_tensor

            if self.mode != "fast":
                raise ValueError("gather='p2p' needs mode='fast'")
            self.flat = torch.zeros(padded, dtype=torch.float32, device=dev)
            handles = [None] * self.world
            dist.all_gather_object(handles, reduce_tensor(self.flat), group=self.pg)
            self._peers = [fn(*args) for r, (fn, args) in enumerate(handles) if r != self.rank]
            # the apply kernel on this device stores into the peers' memory:
            # peer access from this device to each peer's device, explicitly
            # (IPC's lazy enable is tied to the context the handle was opened in)
            from . import _lib

            L = _lib.require_cuda()
            with torch.cuda.device(dev):
                for q in self._peers:
                    if q.device != dev:
                        _lib.check(L.lopt_enable_peer_access(q.device.index), "enable_peer_access")
            base = self.flat.data_ptr()
            self._peer_offsets = [q.data_ptr() - base for q in self._peers]
            self.set_peer_copies(self._peer_offsets)
        else:
            self.flat = torch.zeros(padded, dtype=torch.float32, device=dev)
        for p, n, off in zip(ps, sizes, self.offsets):
            self.flat[off:off + n].copy_(p.data.view(-1))
            p.data = self.flat[off:off + n].view(p.shape)
        # single bucket: rank r's slice is [r*S, (r+1)*S) of the whole arena
        self.slice_len = buckets[0][1] if len(buckets) == 1 else None
        self._rs_hooks = None
        self.ranges = ranges
        for p, (lo, hi) in zip(ps, ranges):
            st = self.state[p]
            m, n = view_2d(p.shape)
            st["quad"] = torch.zeros(max(hi - lo, 1), 4, device=dev, dtype=torch.float32)
            st["row_factors"] = torch.zeros(3, m, device=dev, dtype=torch.float32)
            st["col_factors"] = torch.zeros(3, n, device=dev, dtype=torch.float32)
            st["step"] = self.T
            st["range"] = (lo, hi)

    # -- gradient reduce-scatter (all-reduce = reduce-scatter +
    # all-gather; the step only needs this rank's slice of the summed
    # gradient, and the all-gather is the parameter gather that follows) -----
    def flat_grads(self) -> torch.Tensor:
        """The gradient arena: p.grad of every parameter becomes a view of it,
        laid out like the parameter arena (rank r's slice is its element
        range).  Backward accumulates local (unreduced) gradients into it."""
        ps = self.param_groups[0]["params"]
        if getattr(self, "_flat_grad", None) is None:
            self._flat_grad = torch.zeros_like(self.flat)
        for p, off in zip(ps, self.offsets):
            # (re-)home gradients that are not arena views -- e.g. after
            # Module.zero_grad() set them to None and backward made new ones
            n = p.numel()
            view = self._flat_grad[off:off + n]
            if p.grad is None:
                view.zero_()
            elif p.grad.data_ptr() == view.data_ptr():
                continue
            else:
                view.copy_(p.grad.reshape(-1))
            p.grad = view.view(p.shape)
        return self._flat_grad

    def _bucket_rs(self, b: int, average: bool, async_op: bool):
        """Reduce-scatter of bucket b's gradient segment into this rank's
        portion of it (in place).  Returns the NCCL work handle (async_op)."""
        base, S, _ = self.buckets[b]
        fg = self._flat_grad
        seg = fg[base:base + self.world * S]
        local = seg[self.rank * S:(self.rank + 1) * S]
        if self._nccl():
            op = dist.ReduceOp.AVG if average else dist.ReduceOp.SUM
            return dist.reduce_scatter_tensor(local, seg, op=op, group=self.pg, async_op=async_op)
        # gloo has no reduce-scatter: all-reduce through the host, keep the portion
        h = seg.cpu()
        dist.all_reduce(h, group=self.pg)
        local.copy_(h[self.rank * S:(self.rank + 1) * S].to(fg.device))
        if average:
            local.div_(self.world)
        return None

    def reduce_scatter_grads(self, average: bool = True):
        """Sum (or average) the ranks' local gradients so that each rank holds
        the reduced values of its own slice -- all the sharded step reads
        (distsim.py:323-334 mean_grads, restricted to the owned range).  One
        in-place NCCL reduce-scatter per bucket: half the bytes of the
        all-reduce DDP would otherwise run.  Returns this rank's portion
        (one bucket) or the list of portions."""
        fg = self.flat_grads()
        out = []
        for b, (base, S, _) in enumerate(self.buckets):
            self._bucket_rs(b, average, async_op=False)
            out.append(fg[base + self.rank * S:base + (self.rank + 1) * S])
        return out[0] if len(out) == 1 else out

    # -- reduce-scatter overlapped with backward -----
    def overlap_grad_reduce(self, average: bool = True):
        """Feed the step straight from backward: gradients accumulate into the
        bucketed gradient arena and, as soon as every gradient of a bucket
        has been accumulated (post-accumulate-grad hooks), that bucket's
        reduce-scatter is launched asynchronously, overlapping the rest of
        backward -- DDP's bucketed all-reduce replaced by half its bytes
        (PAPER.md:344).  step() waits for the outstanding buckets first.  Use
        zero_grad() (which zeroes the arena in place) between steps."""
        self.flat_grads()
        ps = self.param_groups[0]["params"]
        bucket_of = {}
        for b, (_, _, tl) in enumerate(self.buckets):
            for j in tl:
                bucket_of[j] = b
        self._rs_hooks = {"average": average, "bucket_of": bucket_of,
                          "ready": [0] * len(self.buckets), "works": {},
                          "handles": []}
        for j, p in enumerate(ps):
            self._rs_hooks["handles"].append(
                p.register_post_accumulate_grad_hook(lambda q, j=j: self._grad_ready(j, q)))

    def _grad_ready(self, j: int, p=None):
        h = self._rs_hooks
        if p is not None:
            # a gradient that is not the arena view (e.g. after Module.zero_grad(),
            # which sets grads to None) is moved into the arena before its
            # bucket is reduced
            off, n = self.offsets[j], p.numel()
            view = self._flat_grad[off:off + n]
            if p.grad is not None and p.grad.data_ptr() != view.data_ptr():
                view.copy_(p.grad.reshape(-1))
                p.grad = view.view(p.shape)
        b = h["bucket_of"][j]
        if b in h["works"]:
            # a second backward into a bucket whose reduce-scatter is already
            # in flight: it would race with the collective writing the same
            # arena segment and add into an already-reduced portion
            raise RuntimeError(
                "gradient accumulation across backward passes is not supported with "
                "overlap_grad_reduce(): call step() (or zero_grad()) after every backward, "
                "or accumulate with overlapped reduction turned off")
        h["ready"][b] += 1
        if h["ready"][b] == len(self.buckets[b][2]):
            h["works"][b] = self._bucket_rs(b, h["average"], async_op=True)

    def _finish_grad_reduce(self):
        h = self._rs_hooks
        for b in range(len(self.buckets)):
            if b not in h["works"]:   # a bucket with unused parameters: reduce it now
                h["works"][b] = self._bucket_rs(b, h["average"], async_op=True)
        for w in h["works"].values():
            if w is not None:
                w.wait()
        h["works"] = {}
        h["ready"] = [0] * len(self.buckets)

    def zero_grad(self, set_to_none: bool = True):
        """With a gradient arena the views are kept and the arena is zeroed in
        place (backward must accumulate into the arena)."""
        if getattr(self, "_flat_grad", None) is not None:
            h = self._rs_hooks
            if h is not None and h["works"]:
                # reductions of a backward that is being discarded: let them
                # finish before the arena they write is cleared
                for w in h["works"].values():
                    if w is not None:
                        w.wait()
                h["works"] = {}
                h["ready"] = [0] * len(self.buckets)
            self._flat_grad.zero_()
            return
        super().zero_grad(set_to_none=set_to_none)

    def _rehome_params(self):
        """The exchange writes into the arena: parameters moved out of it (for
        example by `p.data = ...`) are copied back and re-pointed."""
        for p, off in zip(self.param_groups[0]["params"], self.offsets):
            n = p.numel()
            view = self.flat[off:off + n]
            if p.data.data_ptr() != view.data_ptr():
                view.copy_(p.data.reshape(-1))
                p.data = view.view(p.shape)

    def step(self, closure=None, loss=None):
        self._rehome_params()
        if self._rs_hooks is not None:
            if closure is not None:
                with torch.enable_grad():
                    loss = closure()
                closure = None
            self._finish_grad_reduce()
        return super().step(closure=closure, loss=loss)

    def step_host(self, *args, **kw):
        """Not for the sharded optimizer: its parameters live in the shared
        arena the exchange writes into.  Copy each rank's slice in and out
        around step() instead (what bench.py's sharded e2e does)."""
        raise NotImplementedError("step_host is single-GPU; copy flat_grads()/flat slices "
                                  "around step() on each rank")

    def _slot(self, p, weight_slot=0) -> Slot:
        s = super()._slot(p, weight_slot)
        s.lo, s.hi = self.state[p]["range"]
        return s

    def _run_plan(self, plan: StepPlan, lr, weight_decay, t, gi, params):
        timed = self._timed
        plan.set_step(lr, weight_decay, t)
        timed("factors", plan.factor_partials)
        if self.strategy == "range":
            timed("factor_merge", lambda: self._all_reduce(plan.factor_sums()))
        else:   # whole tensors: only the abort flag is shared (all-or-nothing step)
            timed("factor_merge", lambda: self._all_reduce(plan.factor_sums()[-1:]))
        timed("finalize", plan.factor_finalize)
        timed("stats", plan.feature_stats)
        if self.strategy == "range" or self._after_stats is not None:
            # (owner + VeLO: the per-tensor LSTM runs on every rank and needs
            # every tensor's statistics; 47 KB for ViT-B/16)
            timed("stats_merge", lambda: self._all_reduce(plan.stat_sums()))
        if self._after_stats is not None:
            timed("hypernet", lambda: self._after_stats(gi, plan, params))
        timed("apply", plan.apply)
        if not self.exchange:
            return
        if self._peers is not None:
            # the peers' stores into this arena happened inside their apply
            # kernels; one cross-rank barrier orders them before any read
            timed("param_gather", self._peer_barrier)
        else:
            timed("param_gather", self._gather)

    def set_exchange(self, on: bool):
        """Diagnostics (step time with and without the
        all-gather): off, each rank updates only its own slice and the
        replicas go stale.  Turn it back on before relying on the parameters."""
        self.exchange = bool(on)
        if self._peers is not None:
            self.set_peer_copies(self._peer_offsets if on else [])

    def _nccl(self) -> bool:
        return dist.get_backend(self.pg) == "nccl"

    def _all_reduce(self, t):
        if self._nccl():
            dist.all_reduce(t, group=self.pg)
        else:   # gloo (tests, several ranks on one device): stage through the host
            h = t.cpu()
            dist.all_reduce(h, group=self.pg)
            t.copy_(h)

    def _peer_barrier(self):
        if self._nccl():
            # stream-ordered: completes after every rank's apply kernel (whose
            # peer stores end with a system-scope fence)
            t = getattr(self, "_barrier_buf", None)
            if t is None:
                t = self._barrier_buf = torch.zeros(1, device=self.flat.device)
            dist.all_reduce(t, group=self.pg)
        else:
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.pg)

    def _gather(self):
        for base, S, _ in self.buckets:
            seg = self.flat[base:base + self.world * S]
            local = seg[self.rank * S:(self.rank + 1) * S]
            if self._nccl():
                # in place: input is this rank's portion of the output segment
                dist.all_gather_into_tensor(seg, local, group=self.pg)
            else:
                chunks = [torch.empty(S, dtype=torch.float32) for _ in range(self.world)]
                dist.all_gather(chunks, local.cpu(), group=self.pg)
                seg.copy_(torch.cat(chunks).to(seg.device))

    def load_state_dict(self, state_dict):
        """LearnedOptimizer.load_state_dict, then a layout check: every tensor's
        saved element range must be the one this rank steps under the current
        world size (a state saved by another rank, or under another world
        size, would otherwise update the wrong slice)."""
        from .optim import OptimError

        super().load_state_dict(state_dict)
        for j, p in enumerate(self.param_groups[0]["params"]):
            st = self.state[p]
            got = tuple(int(x) for x in st.get("range", (-1, -1)))
            if got != tuple(self.ranges[j]):
                raise OptimError(f"tensor {j}: saved element range {got} is not this rank's "
                                 f"range {tuple(self.ranges[j])} (rank {self.rank} of "
                                 f"{self.world}); load the state saved by this rank")
            n = self.ranges[j][1] - self.ranges[j][0]
            if "quad" in st and st["quad"].shape[0] != max(n, 1):
                raise OptimError(f"tensor {j}: state holds {st['quad'].shape[0]} elements, "
                                 f"the range has {n}")
            st["range"] = tuple(self.ranges[j])

    def local_state_bytes(self) -> int:
        return sum(int(st["quad"].numel()) * 4 for st in self.state.values() if "quad" in st)


def _sharded_velo_cls():
    from .velo import VeLOHyperNet, _VeLOMixin

    class ShardedVeLO(_VeLOMixin, ShardedLearnedOptimizer):
        """VeLO_CUDA sharded by element ranges: every rank runs the (tiny)
        hypernetwork on the merged statistics, so all ranks mix identical
        per-tensor MLPs."""

        def __init__(self, params, lr=1.0, weight_decay=0.0, *, hypernet=None, **kw):
            kw.pop("feature_set", None)
            hn = hypernet or VeLOHyperNet()
            super().__init__(params, lr=lr, weight_decay=weight_decay, feature_set="velo_mlp",
                             weights=hn.bank[0], **kw)
            self._velo_init(hn)
            # the loss is a host scalar: averaged over a gloo group on the
            # host, so a step never waits for the device queue to drain (an
            # NCCL all-reduce + .item() would block on the previous step)
            ranks = dist.get_process_group_ranks(self.pg or dist.group.WORLD)
            self._host_pg = dist.new_group(ranks=ranks, backend="gloo") if self._nccl() else self.pg

        def step(self, closure=None, loss=None):
            if closure is not None:
                with torch.enable_grad():
                    loss = closure()
            if loss is None:
                self._set_loss(None)   # raises: VeLO needs the loss
            # the hypernetwork's loss features must be the same on every rank
            # (each rank mixes the MLP for its slices of the same tensors):
            # the data-parallel batch loss, i.e. the mean of the ranks' losses
            self._set_loss(self.global_loss(loss))
            return super().step(loss=loss)

        def global_loss(self, loss) -> float:
            """Mean of `loss` over the ranks of the process group (host
            all-reduce over gloo)."""
            t = torch.tensor([float(loss)], dtype=torch.float64)
            dist.all_reduce(t, group=self._host_pg)
            return float(t.item()) / self.world

    return ShardedVeLO


def ShardedVeLO(*args, **kw):
    return _sharded_velo_cls()(*args, **kw)
