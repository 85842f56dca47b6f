"""Arena planner soundness (pinned inputs, aliasing, shadow simulation) and
the multi-process replica logic (world_size 2 over gloo, on CPU)."""
import os
import socket

import numpy as np
import pytest

from builders import random_network
from paper_1906_05737_b200 import build_graph, build_plan, plan_buffers, zoo
from paper_1906_05737_b200.buffers import (BufferAssignment, compute_lifetimes,
                                           verify_assignment, round16)
from paper_1906_05737_b200.errors import PlannerError
from paper_1906_05737_b200.replicas import shard

F32 = np.float32


def plans():
    for cfg in range(5):
        yield build_plan(build_graph(*zoo.build(cfg)))


def test_round16_and_alignment():
    assert [round16(n) for n in (0, 1, 16, 17)] == [0, 16, 16, 32]
    for p in plans():
        a = plan_buffers(p)
        assert all(off % 16 == 0 for off, _ in a.offsets.values())
        assert set(a.offsets) == set(p.tensors)


def test_inputs_pinned_outputs_live_to_end():
    p = build_plan(build_graph(*zoo.build(2)))
    iv = {i.tensor: i for i in compute_lifetimes(p)}
    end = len(p.units)
    for t in p.input_ids:
        assert iv[t].first_def == -1 and iv[t].last_use == end
    for t in p.output_ids:
        assert iv[t].last_use == end
    unpinned = {i.tensor: i for i in compute_lifetimes(p, pin_inputs=False)}
    assert unpinned[p.input_ids[0]].last_use < end


def test_live_tensors_never_overlap():
    for p in plans():
        a = plan_buffers(p)
        alias = {frozenset(x) for x in a.aliases}
        ivs = list(a.intervals.values())
        for i, x in enumerate(ivs):
            for y in ivs[i + 1:]:
                if not x.overlaps(y) or frozenset((x.tensor, y.tensor)) in alias:
                    continue
                ox, sx = a.offsets[x.tensor]
                oy, sy = a.offsets[y.tensor]
                assert ox + sx <= oy or oy + sy <= ox, (x, y)


def test_in_place_alias_for_standalone_softmax():
    p = build_plan(build_graph(*zoo.build(3)))          # Dense 1000 -> Softmax stays standalone
    a = plan_buffers(p)
    sm = p.units[-1]
    assert sm.kind == "Softmax"
    # its input is the Dense output which dies at the softmax, but the softmax
    # output is the network output -> the alias must be refused
    assert (sm.output_id, sm.input_ids[0]) not in a.aliases


def test_shadow_sim_catches_forced_overlap():
    p = build_plan(build_graph(*zoo.build(0)))
    a = plan_buffers(p)
    assert verify_assignment(p, a) == []
    bad = BufferAssignment(a.arena_size, {t: (0, s) for t, (_, s) in a.offsets.items()},
                           [], a.intervals)
    assert verify_assignment(p, bad)


def test_planner_deterministic_and_random_sweep():
    rng = np.random.default_rng(7)
    for _ in range(300):
        m, w, _ = random_network(rng)
        p = build_plan(build_graph(m, w))
        a1, a2 = plan_buffers(p), plan_buffers(p)
        assert a1.offsets == a2.offsets and verify_assignment(p, a1) == []


def test_corrupt_plan_rejected():
    p = build_plan(build_graph(*zoo.build(1)))
    p.tensors[999] = p.tensors[p.output_ids[0]]
    with pytest.raises(PlannerError):
        plan_buffers(p)


@pytest.mark.parametrize("b,w", [(7, 2), (8, 4), (3, 8), (65536, 8), (1, 1)])
def test_shard_partition(b, w):
    parts = [shard(b, w, r) for r in range(w)]
    assert sum(c for _, c in parts) == b
    pos = 0
    for s, c in parts:
        assert s == pos
        pos += c
    assert max(c for _, c in parts) - min(c for _, c in parts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _replica_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    from oracle import oracle
    from paper_1906_05737_b200.replicas import ReplicaGroup
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, w = zoo.build(0)
        g = build_graph(m, w)

        class CpuEngine:                     # stands in for the per-GPU network
            def __init__(self, count):
                self.count = count

            def run(self, xs):
                assert xs[0].shape[0] == self.count
                return oracle.run_graph(g, xs, threads=1)

        grp = ReplicaGroup(9, CpuEngine)
        x = zoo.inputs(0, 9)
        out = grp.gather(grp.run([x]))[0]
        t = grp.max_time(0.5 + rank)
        q.put((rank, grp.start, grp.count, out, t))
    finally:
        dist.destroy_process_group()


def test_replicas_world2_gloo():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import oracle
    m, w = zoo.build(0)
    want = oracle.run(m, w, [zoo.inputs(0, 9)])[0]
    assert [(r[1], r[2]) for r in res] == [(0, 5), (5, 4)]
    for r in res:
        np.testing.assert_array_equal(r[3], want)
        assert r[4] == 1.5                    # max over ranks
