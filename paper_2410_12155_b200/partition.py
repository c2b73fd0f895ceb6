"""Phase-space partition plans and their communication accounting.

The planning half of the reference's multi-rank layer
(/root/reference/pkg/src/vpfv/partition.py): every species' phase-space box
is tiled by a uniform grid of partitions (boxes), boxes are mapped to ranks
(``r`` co-located species per rank), and the ghost-exchange traffic is
enumerated as segments -- 3-deep faces along every dimension plus 1-deep
diagonal edges for the dimension pairs the chosen strategy keeps:

* ``"vp"``  -- only the pairs the transverse flux corrections couple
  (correction_edge_pairs, partition.py:65-83);
* ``"fvm"`` -- every dimension pair of the general fourth-order stencil;
* ``"all"`` -- the whole 3-deep ghost shell (accounting studies).

The same plan drives the B200 execution of general box decompositions
(``cluster.ClusterSimulation``): the segment windows become device gather /
scatter maps, the ``reduce`` combine order is the reference fold tree, and
the TrafficLog rows it writes are the ones the reference's simulated
exchange records.  Everything here is host-side bookkeeping (no device
work); the names, arguments, errors and numbers follow the reference so a
caller of ``vpfv.partition`` can switch over unchanged.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field as dfield

import numpy as np

from .grid import NGHOST, DistField, PhaseSpaceGrid, make_grid

STRATEGIES = ("vp", "fvm", "all")


def _payload(x):
    return x.data if isinstance(x, DistField) else np.asarray(x)


def _check_dv(d, v):
    if d < 1 or v < d:
        raise ValueError(f"need d >= 1 and v >= d, got d={d}, v={v}")


# ---------------------------------------------------------------------------
# neighbour / pair counting (partition.py:47-115)


def neighbor_pairs(d, v):
    """Neighbour counts of a partition inside a 3^(d+v) block: the whole
    hypercube shell (N_all), faces plus every width-1 diagonal edge of the
    general stencil (N_FVM), and the reduced set the electrostatic
    corrections need (N_VP) -- partition.py:47-62."""
    _check_dv(d, v)
    D = d + v
    return {"N_all": 3 ** D - 1, "N_FVM": 2 * D * D,
            "N_VP": 2 * D * D - 4 * math.comb(d, 2) - 4 * (v - d) * d}


def correction_edge_pairs(d, v):
    """Dimension pairs (i < j) whose diagonal ghosts the corrections read
    (partition.py:65-83): x_i with its own and every field-carrying velocity
    component, and -- through the magnetic rotation -- the two in-plane
    velocity dims when v == 2."""
    _check_dv(d, v)
    out = {(i, d + k) for i in range(d) for k in range(v) if k == i or k < d}
    if v == 2:
        out.add((d, d + 1))
    return frozenset(out)


def _edge_pairs(strategy, d, v):
    if strategy == "vp":
        return sorted(correction_edge_pairs(d, v))
    if strategy == "fvm":
        return list(itertools.combinations(range(d + v), 2))
    raise ValueError(f"unknown ghost strategy {strategy!r}")


def ghost_fraction(N_local, d, v, strategy="fvm"):
    """Share of the full 3-deep ghost shell of a cubic N_local^(d+v) box a
    strategy moves (partition.py:95-115)."""
    if N_local < 8:
        raise ValueError(f"N_local={N_local} below the stencil minimum of 8")
    D = d + v
    shell = (N_local + 2 * NGHOST) ** D - N_local ** D
    if strategy == "all":
        return 1.0
    moved = 2 * D * NGHOST * N_local ** (D - 1) + 4 * len(_edge_pairs(strategy, d, v)) * N_local ** (D - 2)
    return moved / shell


# ---------------------------------------------------------------------------
# plan objects (partition.py:118-252)


@dataclass(frozen=True)
class Box:
    """One partition: species, lexicographic number, multi-index, cell range
    [lo, hi) per dim and owning rank."""

    species: int
    lex: int
    index: tuple
    lo: tuple
    hi: tuple
    rank: int

    @property
    def shape(self):
        return tuple(b - a for a, b in zip(self.lo, self.hi))


@dataclass(frozen=True)
class GhostSegment:
    """A rectangular ghost slab copied from one box into another; windows are
    (start, stop) per dim in each box's padded local coordinates, ``dims``
    the dims it is offset along (one for a face, two for an edge)."""

    src_box: tuple
    dst_box: tuple
    src_rank: int
    dst_rank: int
    kind: str
    dims: tuple
    src_window: tuple
    dst_window: tuple
    count: int


@dataclass(frozen=True)
class PartitionPlan:
    """Boxes per species, the rank map and the ghost segments."""

    d: int
    v: int
    S: int
    r: int
    ranks: int
    strategy: str
    grids: tuple
    n: tuple
    boxes: tuple
    rank_members: tuple
    segments: tuple

    def box(self, species, lex):
        return self.boxes[species][lex]

    def boxes_flat(self):
        return itertools.chain.from_iterable(self.boxes)

    def box_grid(self, species, lex):
        """Local grid of one box; a dim stays periodic only when one box spans
        it (partition.py:177-196), split dims are fed by the exchange."""
        g, b = self.grids[species], self.box(species, lex)
        lo = tuple(g.lo[k] + b.lo[k] * g.h[k] for k in range(g.ndim))
        hi = tuple(g.lo[k] + b.hi[k] * g.h[k] for k in range(g.ndim))
        per = tuple(bool(g.periodic[k] and self.n[species][k] == 1) for k in range(g.ndim))
        return make_grid(g.d, g.v, b.shape, lo, hi, periodic=per, spacing=g.h)

    def segments_to(self, species, lex):
        return [x for x in self.segments if x.dst_box == (species, lex)]

    def segments_from(self, species, lex):
        return [x for x in self.segments if x.src_box == (species, lex)]

    def directed_pairs(self):
        """Segments grouped by (src_box, dst_box), first-appearance order:
        one packed message per pair (partition.py:204-215)."""
        groups = {}
        for seg in self.segments:
            groups.setdefault((seg.src_box, seg.dst_box), []).append(seg)
        return [(k, tuple(v)) for k, v in groups.items()]

    def to_report(self):
        """The ``plan`` report (partition.py:217-252)."""
        rank_map = []
        for rank, members in enumerate(self.rank_members):
            rows = []
            for s, lex in members:
                b = self.box(s, lex)
                rows.append({"species": s, "box": list(b.index), "cells_lo": list(b.lo), "cells_hi": list(b.hi)})
            rank_map.append({"rank": rank, "members": rows})
        return {"d": self.d, "v": self.v, "species": self.S, "species_per_rank": self.r, "ranks": self.ranks,
                "strategy": self.strategy, "partition_grid": [list(x) for x in self.n], "rank_map": rank_map,
                "neighbor_pairs": neighbor_pairs(self.d, self.v), "comm_volumes": comm_volumes(self),
                "ghost_accounting": ghost_accounting(self),
                "ghost_fraction_small_N": {k: ghost_fraction(8, self.d, self.v, k) for k in ("fvm", "vp")}}


def _per_species(value, S, what):
    seq = list(value)
    if seq and not hasattr(seq[0], "__len__"):
        seq = [seq] * S
    if len(seq) != S:
        raise ValueError(f"{what}: expected one entry per species ({S}), got {len(seq)}")
    return [tuple(int(x) for x in e) for e in seq]


def _validate(grids, ns, r):
    d, v = grids[0].d, grids[0].v
    D = d + v
    for g in grids:
        if (g.d, g.v) != (d, v):
            raise ValueError("all species must share (d, v)")
        if g.N[:d] != grids[0].N[:d] or g.periodic != grids[0].periodic:
            raise ValueError("physical grids must be identical across species")
    for s, (g, ns_) in enumerate(zip(grids, ns)):
        if len(ns_) != D:
            raise ValueError(f"species {s}: need {D} partition counts, got {len(ns_)}")
        if ns_[:d] != ns[0][:d]:
            raise ValueError("physical partition counts must be identical across species")
        for k, (N, c) in enumerate(zip(g.N, ns_)):
            if c < 1:
                raise ValueError(f"species {s}: partition count must be >= 1 in dim {k}")
            if N % c:
                raise ValueError(f"species {s}: partition count {c} does not divide N[{k}]={N}")
            if N // c < 8:
                raise ValueError(f"species {s}: partition span {N // c} in dim {k} "
                                 "is below the stencil + correction footprint minimum of 8")
    S = len(grids)
    if S % r:
        raise ValueError(f"species_per_rank r={r} must divide species count S={S}")
    if r > 1 and any(x != ns[0] for x in ns):
        raise ValueError("r > 1 requires identical partition grids across species")


def plan_partitions(grids, n, ranks=None, r=1, strategy="vp"):
    """Tile each species' box by ``n`` partitions per dim and map the boxes to
    ranks (partition.py:264-365).  ``n`` is one count per dim (shared) or one
    tuple per species; ``r`` co-locates boxes of r species with the same
    index on one rank; ``ranks`` (optional) must equal the resulting rank
    count; ``strategy`` selects the diagonal ghost segments."""
    if isinstance(grids, PhaseSpaceGrid):
        grids = (grids,)
    grids = tuple(grids)
    if not grids:
        raise ValueError("need at least one species grid")
    S = len(grids)
    ns = _per_species(n, S, "partition counts")
    _validate(grids, ns, r)
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown ghost strategy {strategy!r}")
    counts = [int(np.prod(x)) for x in ns]
    nranks = sum(counts) // r
    if ranks is not None and ranks != nranks:
        raise ValueError(f"rank-count mismatch: plan yields {nranks} ranks, caller expects {ranks}")
    first = np.cumsum([0] + counts)
    members = [[] for _ in range(nranks)]
    boxes = []
    for s, (g, ns_) in enumerate(zip(grids, ns)):
        span = [N // c for N, c in zip(g.N, ns_)]
        mine = []
        for lex, idx in enumerate(itertools.product(*(range(c) for c in ns_))):
            # co-located species share the rank of the same box index
            rank = (s // r) * counts[0] + lex if r > 1 else int(first[s]) + lex
            lo = tuple(i * w for i, w in zip(idx, span))
            mine.append(Box(s, lex, tuple(idx), lo, tuple(a + w for a, w in zip(lo, span)), rank))
            members[rank].append((s, lex))
        boxes.append(tuple(mine))
    plan = PartitionPlan(grids[0].d, grids[0].v, S, r, nranks, strategy, grids, tuple(ns), tuple(boxes),
                         tuple(tuple(m) for m in members), ())
    object.__setattr__(plan, "segments", tuple(_segments(plan)))
    return plan


# ---------------------------------------------------------------------------
# ghost segments (partition.py:368-486)


def _box_at(plan, s, index):
    lex = 0
    for c, i in zip(plan.n[s], index):
        lex = lex * c + i
    return plan.boxes[s][lex]


def _offsets(plan):
    """Neighbour offsets of one box, in the reference's generation order."""
    D = plan.d + plan.v
    if plan.strategy == "all":
        return [(tuple(o - 1 for o in idx), "full") for idx in itertools.product(range(3), repeat=D)
                if any(o != 1 for o in idx)]
    out = [(tuple(side if k == dim else 0 for k in range(D)), "face") for dim in range(D) for side in (-1, 1)]
    for i, j in _edge_pairs(plan.strategy, plan.d, plan.v):
        for si, sj in itertools.product((-1, 1), repeat=2):
            out.append((tuple(si if k == i else sj if k == j else 0 for k in range(D)), "edge"))
    return out


def _segment(plan, s, b, off, width):
    """Segment filling box ``b``'s ghost region at neighbour offset ``off``,
    or None where the offset leaves a non-periodic domain (frozen slabs,
    never transferred) or wraps onto the box itself along no dim."""
    g = plan.grids[s]
    depth = 1 if width == "edge" else NGHOST
    region, src_index, shift = [], list(b.index), []
    for k, o in enumerate(off):
        if o == 0:
            region.append((b.lo[k], b.hi[k]))
            shift.append(0)
            continue
        region.append((b.hi[k], b.hi[k] + depth) if o > 0 else (b.lo[k] - depth, b.lo[k]))
        nb = b.index[k] + o
        if 0 <= nb < plan.n[s][k]:
            src_index[k], sh = nb, 0
        elif g.periodic[k]:
            src_index[k], sh = nb % plan.n[s][k], -o * g.N[k]
        else:
            return None
        shift.append(sh)
    src = _box_at(plan, s, src_index)
    if src.lex == b.lex and not any(shift):
        return None
    count = int(np.prod([z - a for a, z in region]))
    return GhostSegment(
        src_box=(s, src.lex), dst_box=(s, b.lex), src_rank=src.rank, dst_rank=b.rank,
        kind={"face": "face", "edge": "edge", "full": "shell"}[width],
        dims=tuple(k for k, o in enumerate(off) if o),
        src_window=tuple((a + sh - src.lo[k] + NGHOST, z + sh - src.lo[k] + NGHOST)
                         for k, ((a, z), sh) in enumerate(zip(region, shift))),
        dst_window=tuple((a - b.lo[k] + NGHOST, z - b.lo[k] + NGHOST) for k, (a, z) in enumerate(region)),
        count=count)


def _segments(plan):
    offs = _offsets(plan)
    out = []
    for s in range(plan.S):
        for b in plan.boxes[s]:
            for off, width in offs:
                seg = _segment(plan, s, b, off, width)
                if seg is not None:
                    out.append(seg)
    return out


# ---------------------------------------------------------------------------
# transfer-volume formulas and the counted comparison (partition.py:489-600)


def _prod(xs):
    out = 1
    for x in xs:
        out *= int(x)
    return out


def reduce_volume_formula(N, n, d, S, r=1):
    """ceil(log2((S/r) x velocity partitions)) combine rounds, one value per
    physical cell each (partition.py:489-504)."""
    m = (S // r) * _prod(n[d:len(N)])
    return ((m - 1).bit_length() if m > 0 else 0) * _prod(N[:d])


def phi_volume_formula(N, n, p, d, S, r=1):
    """The reduction term plus 3 ghost layers per side of every physical
    interface, (n_i - p_i) interfaces per physical dim (partition.py:507-524)."""
    faces = sum((n[i] - p[i]) * _prod(N[j] for j in range(d) if j != i) for i in range(d))
    return reduce_volume_formula(N, n, d, S, r) + 6 * S * _prod(n[d:len(N)]) * faces


def ghost_volume_formula(N, n, p, S):
    """6 ghost layers per interface plus two width-1 strips per interface
    pair, as printed (p_i = 1 on periodic dims; partition.py:527-552)."""
    D = len(N)
    faces = edges = 0
    for i in range(D):
        faces += (n[i] - p[i]) * _prod(N[j] for j in range(D) if j != i)
        for j in range(D):
            if j != i:
                edges += (n[i] - p[i]) * (n[j] - p[j]) * _prod(N[k] for k in range(D) if k not in (i, j))
    return S * (6 * faces + 2 * edges)


def comm_volumes(plan):
    """B_reduce, B_phi, B_ghost from species 0's counts (partition.py:555-572)."""
    g, n = plan.grids[0], plan.n[0]
    p = [1 if g.periodic[k] else 0 for k in range(g.ndim)]
    return {"B_reduce": reduce_volume_formula(g.N, n, plan.d, plan.S, plan.r),
            "B_phi": phi_volume_formula(g.N, n, p, plan.d, plan.S, plan.r),
            "B_ghost": ghost_volume_formula(g.N, n, p, plan.S)}


def ghost_accounting(plan):
    """Printed B_ghost next to the counted segment volume, all segments and
    only those crossing ranks (partition.py:575-600)."""
    formula = comm_volumes(plan)["B_ghost"]
    counted = sum(x.count for x in plan.segments)
    return {"formula": formula, "counted": counted,
            "counted_off_rank": sum(x.count for x in plan.segments if x.src_rank != x.dst_rank),
            "strategy": plan.strategy, "agrees": formula == counted}


# ---------------------------------------------------------------------------
# gather / scatter maps and host pack/unpack (partition.py:603-650)


def window_flat_indices(window, shape):
    """C-order flat indices of a rectangular window of an array of ``shape``."""
    axes = [np.arange(a, z, dtype=np.int64) for a, z in window]
    strides = np.cumprod((list(shape[1:]) + [1])[::-1])[::-1].astype(np.int64)
    flat = np.zeros((1,) * len(shape), dtype=np.int64)
    for k, (ax, st) in enumerate(zip(axes, strides)):
        flat = flat + (ax * st).reshape([-1 if j == k else 1 for j in range(len(shape))])
    return flat.reshape(-1)


def segment_flat_maps(segments, src_shape, dst_shape):
    """Flat source and destination indices of a pair's segments, concatenated
    in segment order (one buffer per pair)."""
    if not segments:
        e = np.empty(0, dtype=np.intp)
        return e, e.copy()
    return (np.concatenate([window_flat_indices(x.src_window, src_shape) for x in segments]),
            np.concatenate([window_flat_indices(x.dst_window, dst_shape) for x in segments]))


def pack_ghosts(field, segments):
    data = _payload(field)
    src, _ = segment_flat_maps(segments, data.shape, data.shape)
    return data.reshape(-1)[src]


def unpack_ghosts(buffer, field, segments):
    data = _payload(field)
    _, dst = segment_flat_maps(segments, data.shape, data.shape)
    if buffer.shape != dst.shape:
        raise ValueError(f"buffer length {buffer.shape} does not match segment cells {dst.shape}")
    data.reshape(-1)[dst] = buffer
    return field


# ---------------------------------------------------------------------------
# traffic log (partition.py:653-676), host exchanger, scatter / gather


@dataclass
class TrafficRow:
    stage: int
    kind: str
    src: int
    dst: int
    count: int


@dataclass
class TrafficLog:
    """Per-message records (kind: ghost / reduce / field), counts in cells."""

    rows: list = dfield(default_factory=list)

    def log(self, stage, kind, src, dst, count):
        self.rows.append(TrafficRow(stage, kind, src, dst, int(count)))

    def total(self, kind=None):
        return sum(x.count for x in self.rows if kind in (None, x.kind))

    def to_csv_rows(self):
        yield ("stage", "kind", "src", "dst", "count")
        for x in self.rows:
            yield (x.stage, x.kind, x.src, x.dst, x.count)


def padded_box_shape(box):
    return tuple(w + 2 * NGHOST for w in box.shape)


class Exchanger:
    """Host (numpy) exchange of a plan's ghost segments: every pair packed
    first, then every pair unpacked (partition.py:679-724)."""

    def __init__(self, plan):
        self.plan = plan
        self.pairs = []
        for (src, dst), segs in plan.directed_pairs():
            si, di = segment_flat_maps(segs, padded_box_shape(plan.box(*src)), padded_box_shape(plan.box(*dst)))
            self.pairs.append({"src": src, "dst": dst, "src_rank": segs[0].src_rank,
                               "dst_rank": segs[0].dst_rank, "src_idx": si, "dst_idx": di, "count": int(si.size)})

    def exchange(self, fields, log=None, stage=0):
        bufs = [_payload(fields[p["src"]]).reshape(-1)[p["src_idx"]] for p in self.pairs]
        for p, buf in zip(self.pairs, bufs):
            _payload(fields[p["dst"]]).reshape(-1)[p["dst_idx"]] = buf
            if log is not None:
                log.log(stage, "ghost", p["src_rank"], p["dst_rank"], p["count"])
        return log


def simulate_exchange(plan, fields, log=None, stage=0):
    log = TrafficLog() if log is None else log
    Exchanger(plan).exchange(fields, log=log, stage=stage)
    return log


def scatter_field(plan, species, dist):
    """Per-box padded copies of a ghost-filled global padded array."""
    data = _payload(dist)
    return {(species, b.lex): data[tuple(slice(a, z + 2 * NGHOST) for a, z in zip(b.lo, b.hi))].copy()
            for b in plan.boxes[species]}


def gather_field(plan, species, fields):
    """Global interior array assembled from the boxes' interiors."""
    out = np.empty(plan.grids[species].N)
    for b in plan.boxes[species]:
        local = _payload(fields[(species, b.lex)])
        out[tuple(slice(a, z) for a, z in zip(b.lo, b.hi))] = local[tuple(slice(NGHOST, NGHOST + w)
                                                                         for w in b.shape)]
    return out


# ---------------------------------------------------------------------------
# cross-partition combine (partition.py:778-814)


def combine_partials(partials, ranks=None, log=None, stage=0, cell_count=None):
    """Adjacent pairs level by level, lower index on the left, odd tail
    carried: the reference fold tree above the per-box subtrees, so power-of-
    two spans give sums bitwise equal to one rank's fold.  One ``reduce``
    row per pairwise message (sender = the upper box) when logging."""
    level = list(partials)
    who = list(ranks) if ranks is not None else [None] * len(level)
    while len(level) > 1:
        nxt, nwho = [], []
        for i in range(0, len(level) - 1, 2):
            if log is not None and who[i] is not None:
                up = level[i + 1]
                n = cell_count if cell_count is not None else (up.numel() if hasattr(up, "numel") else np.size(up))
                log.log(stage, "reduce", who[i + 1], who[i], n)
            nxt.append(level[i] + level[i + 1])
            nwho.append(who[i])
        if len(level) % 2:
            nxt.append(level[-1])
            nwho.append(who[-1])
        level, who = nxt, nwho
    return level[0]


def reduction_rounds(m):
    """ceil(log2 m) combine rounds for m partials."""
    return (int(m) - 1).bit_length()


def _main(argv=None):
    """``python -m paper_2410_12155_b200.partition plan ...``: the plan report
    of the reference's ``vpfv plan`` (cli.py:207-222) for a uniform grid given
    on the command line instead of an INI file (the config layer is out of
    scope)."""
    import argparse
    import json

    ap = argparse.ArgumentParser(prog="python -m paper_2410_12155_b200.partition")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("plan", help="partition plan report (JSON)")
    p.add_argument("--d", type=int, required=True)
    p.add_argument("--v", type=int, required=True)
    p.add_argument("--N", type=int, nargs="+", required=True, help="cells per dim (one species)")
    p.add_argument("--n", type=int, nargs="+", required=True, help="partitions per dim")
    p.add_argument("--species", type=int, default=1)
    p.add_argument("--r", type=int, default=1, help="species per rank")
    p.add_argument("--strategy", default="vp", choices=STRATEGIES)
    p.add_argument("--vmax", type=float, default=6.0)
    a = ap.parse_args(argv)
    g = make_grid(a.d, a.v, a.N, [0.0] * a.d + [-a.vmax] * a.v, [2 * math.pi] * a.d + [a.vmax] * a.v,
                  periodic=tuple([True] * a.d + [False] * a.v))
    plan = plan_partitions([g] * a.species, a.n, r=a.r, strategy=a.strategy)
    print(json.dumps(plan.to_report(), indent=2))


if __name__ == "__main__":
    _main()
