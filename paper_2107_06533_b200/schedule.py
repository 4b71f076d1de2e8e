"""Communication schedule of the SPD-KFAC step (host logic, no device code).

Pure functions shared by `SPDKFAC` (GPU, NCCL) and the CPU/gloo tests that check the
multi-rank logic without a GPU:

  packed_layout   offsets of each layer's packed factor in the two fusion buffers
                  (A in forward order, G in backward order: a fusion group, planner.py:94-121,
                  is then one contiguous slice = one all-reduce)
  fusion_slices   {layer index that completes the group: (start, end)} per pass
  bcast_layout    per owner rank, the CT tensors it broadcasts (placement order) and the
                  packed offsets inside that owner's staging buffer (planner.py:141-207 and
                  the owner-compute-then-share walk of emulator.py:256-262)
"""

from __future__ import annotations

from typing import Sequence

from .planner import FactorKind, FusionPlan, PlacementPlan


def packed_size(d: int) -> int:
    return d * (d + 1) // 2


def packed_layout(a_dims: Sequence[int], g_dims: Sequence[int]):
    """Returns (a_off, g_off, size_a, size_g): a_off[l] in forward order, g_off[l] in backward order."""
    a_off, off = [], 0
    for d in a_dims:
        a_off.append(off)
        off += packed_size(d)
    size_a = off
    g_off = [0] * len(g_dims)
    off = 0
    for l in reversed(range(len(g_dims))):
        g_off[l] = off
        off += packed_size(g_dims[l])
    return a_off, g_off, size_a, off


def fusion_slices(plan: FusionPlan, offsets: Sequence[int], dims: Sequence[int]) -> dict:
    """{0-based layer index of the group's last member: (start, end)} for one pass."""
    out = {}
    for group in plan.groups:
        idx = [t.layer_index - 1 for t in group]
        first, last = idx[0], idx[-1]
        out[last] = (offsets[first], offsets[last] + packed_size(dims[last]))
    return out


def fusion_members(plan: FusionPlan) -> tuple:
    """(group id of every 0-based layer, member count of every group) for one pass: a group's
    all-reduce is issued once all its members are written, whatever order the hooks fire in."""
    gid, sizes = {}, []
    for k, group in enumerate(plan.groups):
        for t in group:
            gid[t.layer_index - 1] = k
        sizes.append(len(group))
    return gid, sizes


def reduce_segments(plan: FusionPlan, offsets: Sequence[int], dims: Sequence[int], placement: PlacementPlan,
                    parity: int) -> list:
    """Per fusion group (plan order): [(start, end, root)] covering the group's slice, where root is
    the owner rank of a CT factor's inverse (its aggregate is read only there: reduce) or None
    for an NCT factor (every rank inverts it: all-reduce).  Adjacent factors with the same root
    share one segment.  parity 0 = A (tensor 2l), 1 = G (tensor 2l+1)."""
    out = []
    for group in plan.groups:
        idx = sorted((t.layer_index - 1 for t in group), key=lambda li: offsets[li])
        segs = []
        for li in idx:
            t = 2 * li + parity
            root = None if t in placement.nct else placement.owner(t)
            s, e = offsets[li], offsets[li] + packed_size(dims[li])
            if segs and segs[-1][2] == root and segs[-1][1] == s:
                segs[-1] = (segs[-1][0], e, root)
            else:
                segs.append((s, e, root))
        out.append(segs)
    return out


def check_fusion_cover(slices: dict, total: int) -> None:
    """The groups of one pass tile its fusion buffer exactly once (no gap, no overlap)."""
    spans = sorted(slices.values())
    pos = 0
    for s, e in spans:
        if s != pos or e <= s:
            raise ValueError(f"fusion slices do not tile the buffer at {pos}: {spans}")
        pos = e
    if pos != total:
        raise ValueError(f"fusion slices cover {pos} of {total} elements")


def bcast_layout(placement: PlacementPlan, dims: Sequence[int], parity: int | None = None,
                 members=None) -> list:
    """Per owner rank p: (ct tensor indices in p's placement order, their dims, offsets, total).
    `parity` 0/1 restricts to A/G tensors (tensor_index = 2l / 2l+1, simulator.py:276-282);
    `members` (a set) restricts to one inversion group."""
    out = []
    for lst in placement.workers:
        ct = [t for t in lst if t not in placement.nct and (parity is None or t % 2 == parity)
              and (members is None or t in members)]
        offs, o = [], 0
        for t in ct:
            offs.append(o)
            o += packed_size(dims[t])
        out.append((ct, [dims[t] for t in ct], offs, o))
    return out


def inversion_groups(a_dims: Sequence[int], g_dims: Sequence[int], early_fraction=0.85) -> dict:
    """Tensor sets inverted as soon as their factors exist:
      "A"       every input-side factor (complete after the forward pass)
      "G1".."Gk" output-side factors of the layers the backward pass reaches first, cut where
                the cumulative output-side inversion work (sum d^3, from the last layer) first
                reaches each of the increasing fractions in `early_fraction` (a float or a
                sequence); each is inverted mid-backward as soon as its factors are complete
      "G{k+1}"  the remaining output-side factors (the tail, inverted in step()).
    Returns the sets plus "early" (names G1..Gk), "tail" (G{k+1}) and "n_g" (layers per G set,
    in backward order)."""
    fracs = [float(early_fraction)] if isinstance(early_fraction, (int, float)) else [float(f) for f in early_fraction]
    if any(not 0.0 < f <= 1.0 for f in fracs) or any(b <= a for a, b in zip(fracs, fracs[1:])):
        raise ValueError(f"early fractions must increase within (0, 1], got {fracs}")
    nl = len(g_dims)
    total = sum(float(d) ** 3 for d in g_dims)
    out = {"A": {2 * l for l in range(nl)}}
    acc, l, names, counts = 0.0, nl - 1, [], []
    for f in fracs:
        members = set()
        while l >= 1 and not (total and members and acc >= f * total):  # the tail keeps layer 0
            acc += float(g_dims[l]) ** 3
            members.add(2 * l + 1)
            l -= 1
        if members:
            names.append(f"G{len(names) + 1}")
            out[names[-1]] = members
            counts.append(len(members))
    tail = f"G{len(names) + 1}"
    out[tail] = {2 * i + 1 for i in range(l + 1)}
    counts.append(l + 1)
    out.update(early=names, tail=tail, n_g=counts)
    return out


def kind_of(tensor_index: int) -> FactorKind:
    return FactorKind.A if tensor_index % 2 == 0 else FactorKind.G
