"""Data-parallel replicas over the GPUs of one node.

Images are independent, so batched inference shards the batch into
contiguous slices, one per process/GPU, each running its own compiled
network (own arena, own CUDA graph).  There is no collective on the data
path; ``torch.distributed`` is only used around it -- a barrier before the
timed region, a MAX reduction of the per-rank device time, and an optional
gather of the outputs for the caller (outside any timed region).
"""

import os

import numpy as np


def shard(global_batch, world, rank):
    """Contiguous slice of ``global_batch`` for ``rank``: (start, count);
    the first ``global_batch % world`` ranks take one extra image."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(global_batch, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


class ReplicaGroup:
    """One replica of a compiled network per rank.

    ``engine_factory(count)`` builds the per-rank engine; by default it is
    ``CompiledNetwork(manifest, weights, options, batch=count,
    device=LOCAL_RANK)``.  The engine must offer ``run(inputs) -> outputs``.
    """

    def __init__(self, global_batch, engine_factory, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.global_batch = global_batch
        self.start, self.count = shard(global_batch, self.world, self.rank)
        self.engine = engine_factory(self.count)

    @classmethod
    def compiled(cls, manifest, weights, global_batch, options=None, group=None, **kw):
        from .runtime import compile_model
        local = int(os.environ.get("LOCAL_RANK", "0"))
        return cls(global_batch, lambda c: compile_model(manifest, weights, options, batch=c,
                                                         device=local, **kw), group)

    def local_inputs(self, global_inputs):
        return [x[self.start:self.start + self.count] for x in global_inputs]

    def run(self, global_inputs):
        """Run this rank's shard; returns the local outputs."""
        return self.engine.run(self.local_inputs(global_inputs))

    def gather(self, local_outputs):
        """All shards' outputs concatenated in rank order (every rank gets
        them; host-side, outside the hot path)."""
        if self.world == 1:
            return [np.asarray(o) for o in local_outputs]
        arrs = [np.asarray(o.cpu() if hasattr(o, "cpu") else o) for o in local_outputs]
        got = [None] * self.world
        self.dist.all_gather_object(got, arrs, group=self.group)
        return [np.concatenate([g[i] for g in got]) for i in range(len(arrs))]

    def max_time(self, seconds):
        """MAX over ranks of a per-rank duration (the job's time)."""
        if self.world == 1:
            return seconds
        import torch
        t = torch.tensor([float(seconds)], dtype=torch.float64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


class MultiDeviceNetwork:
    """One host process driving one replica per device (SURVEY.md 8(e)'s
    single-thread alternative to one process per GPU): the global batch is
    sharded into contiguous slices (``shard``), replica ``r`` is a
    ``CompiledNetwork`` on ``devices[r]`` with its own arena, weights and
    CUDA graph, and ``apply()`` enqueues every replica's graph on its
    device's current stream before anything waits -- the devices run
    concurrently, with no collective and no peer traffic on the data path.

    ``devices`` may repeat an id (several replicas on one GPU), which is how
    the single-GPU tests exercise this class.
    """

    def __init__(self, manifest, weights, options=None, *, batch, devices, **kw):
        from .runtime import CompiledNetwork
        if not devices:
            raise ValueError("devices must name at least one GPU")
        self.devices = list(devices)
        self.batch = int(batch)
        self.slices = [shard(self.batch, len(self.devices), r) for r in range(len(self.devices))]
        if any(c == 0 for _, c in self.slices):
            raise ValueError(f"batch {batch} is smaller than the {len(devices)} replicas")
        self.replicas = [CompiledNetwork(manifest, weights, options, batch=c, device=d, **kw)
                         for (_, c), d in zip(self.slices, self.devices)]

    @property
    def input_views(self):
        """Per replica: its input views (torch tensors on its device)."""
        return [r.input_views for r in self.replicas]

    @property
    def output_views(self):
        return [r.output_views for r in self.replicas]

    def apply(self):
        """Enqueue every replica's replay (asynchronous across devices)."""
        for r in self.replicas:
            r.apply()

    def synchronize(self):
        for r in self.replicas:
            r.synchronize()

    def run(self, inputs, gather_device=None):
        """Scatter ``inputs`` (arrays with the global batch leading), replay
        all replicas, and return the outputs concatenated in batch order: torch
        tensors on ``gather_device`` (default: the first device) -- the copies
        are the only cross-device traffic and happen after the replays."""
        import torch
        xs = [x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, np.float32))
              for x in inputs]
        for (start, count), rep in zip(self.slices, self.replicas):
            for view, x in zip(rep.input_views, xs):
                if tuple(x.shape[1:]) != tuple(view.shape[1:]) or x.shape[0] != self.batch:
                    from .errors import InputShapeMismatch
                    raise InputShapeMismatch(f"input shape {tuple(x.shape)} does not match "
                                             f"({self.batch},) + {tuple(view.shape[1:])}")
                view.copy_(x[start:start + count], non_blocking=True)
        self.apply()
        dev = torch.device("cuda", self.devices[0] if gather_device is None else gather_device)
        outs = []
        for i in range(len(self.replicas[0].output_views)):
            parts = [rep.output_views[i].to(dev, non_blocking=True) for rep in self.replicas]
            outs.append(torch.cat(parts))
        for d in sorted(set(self.devices) | {dev.index}):
            torch.cuda.synchronize(d)       # every replica's device, not only the gather's
        return outs
