"""Device-arena planning: lifetimes, in-place aliases, offsets, hazard check.

Counterpart of pkg/src/nnjit/memory_planner.py with three deliberate
differences for the B200 runtime:

* **Inputs are pinned.**  The reference lets an input's range be recycled
  after its last read (memory_planner.py:57-79), so a second ``apply()``
  computes on clobbered data (finding 3).  Here network
  inputs live for the whole schedule: ``apply()`` is idempotent and a CUDA
  graph can be replayed on the same input views.
* **Placement is greedy-by-size** (largest tensor first, lowest offset that
  does not collide with any already placed tensor whose lifetime overlaps) --
  a different heuristic from the reference's alternating first-fit; the
  soundness check below is what both must pass.
* **Batch scaling.**  Offsets are planned per image and 16-byte aligned; the
  runtime multiplies every offset by the batch capacity (a multiple of 16), so
  each tensor becomes one contiguous ``[capacity, *dims]`` block aligned to
  256 bytes.

``verify_assignment`` shadow-simulates the schedule like the reference's
(memory_planner.py:199-237), vectorised over 16-byte slots.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import PlannerError

ALIGN = 16


def round16(nbytes):
    return (nbytes + ALIGN - 1) // ALIGN * ALIGN


@dataclass(frozen=True)
class LifetimeInterval:
    tensor: int
    first_def: int      # -1 for network inputs
    last_use: int       # len(units) for network inputs and outputs
    size: int           # bytes per image, 16-byte multiple

    def overlaps(self, other):
        return self.first_def <= other.last_use and other.first_def <= self.last_use


@dataclass
class BufferAssignment:
    arena_size: int                       # bytes per image
    offsets: dict                         # tensor -> (offset, size) per image
    aliases: list = field(default_factory=list)   # (output, input) shared ranges
    intervals: dict = field(default_factory=dict)

    def describe(self):
        lines = []
        for t in sorted(self.offsets):
            off, size = self.offsets[t]
            iv = self.intervals.get(t)
            life = f"[{iv.first_def},{iv.last_use}]" if iv else "?"
            lines.append(f"  t{t:<3d} offset {off:8d}  size {size:8d}  live {life}")
        al = ", ".join(f"t{o}=t{i}" for o, i in self.aliases) or "none"
        lines.append(f"  arena {self.arena_size} bytes/image, aliases: {al}")
        return "\n".join(lines)


def _reads(u):
    return tuple(u.input_ids) + ((u.residual_id,) if getattr(u, "residual_id", None)
                                 is not None else ())


def _writes(u):
    dp = getattr(u, "dual_pool", None)
    da = getattr(u, "dw_after", None)
    return ((u.output_id,) + ((dp.output_id,) if dp is not None else ())
            + ((da.output_id,) if da is not None else ()))


def head_pairs(plan):
    """Positions of Dense units whose output feeds only the next unit, a
    Dense head with <= 16 outputs: the tcgen05 GEMM may compute that head in
    its epilogue (kernels.py HEAD), i.e. write the head's output while still
    reading its own input."""
    out = []
    for pos in range(len(plan.units) - 1):
        u, v = plan.units[pos], plan.units[pos + 1]
        if (u.kind == "Dense" and v.kind == "Dense" and v.input_ids == (u.output_id,)
                and v.kernel.shape[1] <= 16 and u.output_id not in plan.output_ids
                and plan.consumer_count(u.output_id) == 1):
            out.append(pos)
    return out


def compute_lifetimes(plan, pin_inputs=True, reserve_heads=False):
    """``reserve_heads`` (the B200 runtime) keeps the inputs of a head-fusable
    Dense (``head_pairs``) live through its head, so the head's output never
    takes their space."""
    end = len(plan.units)
    first, last = {}, {}
    for t in plan.input_ids:
        first[t] = -1
        last[t] = end if pin_inputs else -1
    heads = set(head_pairs(plan)) if reserve_heads else set()
    for pos, u in enumerate(plan.units):
        for w in _writes(u):
            first.setdefault(w, pos)
            last[w] = max(last.get(w, pos), pos)
        for t in _reads(u):
            last[t] = max(last.get(t, pos), pos + 1 if pos in heads else pos)
    for t in plan.output_ids:
        last[t] = end
    out = []
    for t, shape in plan.tensors.items():
        if t not in first:
            raise PlannerError(f"tensor t{t} has no producer and is not an input")
        out.append(LifetimeInterval(t, first[t], last[t], round16(4 * shape.elements)))
    return out


def assign_buffers(intervals, plan):
    by_id = {iv.tensor: iv for iv in intervals}
    external = set(plan.input_ids) | set(plan.output_ids)

    # in-place requests: union output with the input it overwrites
    root = {}

    def find(t):
        while root.get(t, t) != t:
            t = root[t]
        return t

    aliases = []
    for pos, u in enumerate(plan.units):
        k = u.in_place_preference
        if k is None or k >= len(u.input_ids):
            continue
        src, dst = u.input_ids[k], u.output_id
        if src in external or dst in external or src not in by_id or dst not in by_id:
            continue
        if by_id[src].last_use != pos or by_id[src].size != by_id[dst].size:
            continue
        root[dst] = find(src)
        aliases.append((dst, src))

    groups = {}
    for iv in intervals:
        g = find(iv.tensor)
        lo, hi, sz = groups.get(g, (iv.first_def, iv.last_use, iv.size))
        if sz != iv.size:
            raise PlannerError("aliased tensors with different sizes")
        groups[g] = (min(lo, iv.first_def), max(hi, iv.last_use), sz)

    # largest first; ties by first definition then id (deterministic)
    order = sorted(groups, key=lambda g: (-groups[g][2], groups[g][0], g))
    placed = []            # (lo, hi, off, size)
    offset_of = {}
    for g in order:
        lo, hi, sz = groups[g]
        busy = sorted((o, o + s) for (l2, h2, o, s) in placed if l2 <= hi and lo <= h2)
        cand = 0
        for a, b in busy:
            if cand + sz <= a:
                break
            cand = max(cand, round16(b))
        offset_of[g] = cand
        placed.append((lo, hi, cand, sz))
    arena = max((o + s for (_, _, o, s) in placed), default=0)

    asg = BufferAssignment(
        arena_size=arena,
        offsets={iv.tensor: (offset_of[find(iv.tensor)], iv.size) for iv in intervals},
        aliases=aliases, intervals={iv.tensor: iv for iv in intervals})
    bad = verify_assignment(plan, asg)
    if bad:
        raise PlannerError("unsound assignment: " + "; ".join(bad[:4]))
    return asg


def plan_buffers(plan, pin_inputs=True, reserve_heads=False):
    return assign_buffers(compute_lifetimes(plan, pin_inputs, reserve_heads), plan)


def verify_assignment(plan, assignment):
    """Replay the schedule over 16-byte slots; report every read of a slot
    that no longer holds the tensor being read."""
    owner = np.full(max(assignment.arena_size // ALIGN, 1), -1, dtype=np.int64)
    parent = dict(assignment.aliases)

    def canon(t):
        while t in parent:
            t = parent[t]
        return t

    def span(t):
        off, size = assignment.offsets[t]
        return slice(off // ALIGN, (off + size) // ALIGN)

    def write(t):
        owner[span(t)] = canon(t)

    def check(t, where):
        sl = span(t)
        wrong = owner[sl] != canon(t)
        if wrong.any():
            s = sl.start + int(np.argmax(wrong))
            held = owner[s]
            return [f"{where}: t{t} slot {s} holds "
                    + (f"t{held}" if held >= 0 else "nothing")]
        return []

    bad = []
    for t in plan.input_ids:
        write(t)
    for pos, u in enumerate(plan.units):
        for t in _reads(u):
            bad += check(t, f"unit {pos} ({u.kind}) read")
        for t in _writes(u):
            write(t)
    for t in plan.output_ids:
        bad += check(t, "network output")
    end = len(plan.units)
    for t in plan.input_ids:
        iv = assignment.intervals.get(t)
        if iv is not None and iv.last_use == end:
            bad += check(t, "pinned input")
    return bad
