"""N3 front-ends: the paper's two ways of writing a schedule, lowered to one xtc_schedule.

PAPER.md §IV-A: "when a Graph is created, its associated Scheduler records the scheduling
API calls and builds an internal representation of the schedule.  It then applies this schedule ...".
Two front-ends build that internal representation here:

  * the imperative API of Fig.4 -- ``Scheduler.split / strip_mine / unroll / vectorize /
    interchange / parallelize / pack / bufferize`` -- every call appended to ``Scheduler.log`` (the
    primitive log) and applied to the loop-nest state at once, so the log replayed into a fresh
    Scheduler (``Scheduler.replay``) rebuilds the same state;
  * the declarative ``descript`` language of §V-A, Fig.8: a dict whose keys declare loops in
    nest order -- ``D`` (outermost loop of D), ``D#N`` (a tile of size N along D), ``D[A:B]`` (a split
    region of D with its own inner dict) -- and whose values are annotations (``unroll``, ``vectorize``,
    ``parallelize``; here also ``pack`` / ``pack=S`` and ``buffer``).

Both give the same canonical loop nest (``Scheduler.nest()``): a tuple of entries, each either a loop
``(dim, size, annotations)`` or a split ``("split", dim, ((lo, hi, sub-nest), ...))``, where ``size`` is
the extent the loop covers (the dim's extent, a split region, or a tile size) and loop names are dropped
(``K1`` in Fig.4 is ``K#4`` in Fig.8).  Vectorization "implicitly unrolls the concerned dimensions"
(P:538-539), so ``vectorize`` carries ``unroll = size`` in the canonical form.

``Scheduler.schedule()`` lowers the canonical nest to the GPU knobs of include/xtc.h (DESIGN.md §4 and
reading 23).  The planner (``xtc_schedule_check`` / ``xtc_schedule_apply``) stays the only judge of
legality.  Lowering rules, for a matmul ``C[I][J] = sum_K A[I][K] B[K][J]`` (GEMM view M = I, N = J):

  * the I and J loops placed above the outermost K loop are the parallel tile loops; the block of each
    dim that the K loop sees (the step of the innermost such loop) is the register / MMA tile
    (SIMT: ``inner_m`` x ``inner_n``; tcgen05: the UMMA atom = the CTA tile); their order gives
    ``order`` (I first = MN);
  * ``parallelize`` on an I / J loop distributes it over the grid: the CTA tile is the step of the
    innermost parallelized loop of that dim (SIMT: threads = CTA tile / register tile); with no
    parallelized loop of a dim, the CTA tile of that dim is the register tile (one thread);
  * the step of the outermost K loop is ``tile_k`` (the k-block staged in shared memory); ``unroll`` on
    the innermost K tile is ``unroll_k``; ``vectorize`` on the innermost J loop is ``vector_n = 4``
    (float4, the SIMT engine's vector width); ``pack=S`` on a K loop is the ring depth ``stages``;
    ``buffer`` on the innermost parallel loop is ``buffer_c = 1``;
  * a split of J into [0, s) and [s, N) whose second region is a plain K loop is the remainder root
    ``split_n_at = s`` (Fig.3/4); a split of K into equal contiguous regions with identical
    sub-nests is ``split_k``;
  * knobs with no loop-nest counterpart (engine, CTA pair, clusters, raster group, persistence, TMEM
    buffers, ...) come from ``target``.
"""
from __future__ import annotations

import copy
import re
from typing import Dict, List, Optional, Tuple

from . import (XTC_ENGINE_SIMT, XTC_ENGINE_TCGEN05, XTC_F32, XTC_OK, XTC_OP_MATMUL, schedule, xtc_op_desc,
               xtc_schedule, xtc_schedule_apply, xtc_schedule_check)

ANNOTATIONS = ("unroll", "vectorize", "parallelize", "pack", "buffer")


class ScheduleError(ValueError):
    """A primitive call or descript entry that is malformed for the current loop nest."""


# ------------------------------------------------------------------ state ---
class _Loop:
    __slots__ = ("name", "dim", "size", "ann")

    def __init__(self, name, dim, size, ann=None):
        self.name, self.dim, self.size = name, dim, size
        self.ann: Dict[str, int] = dict(ann or {})


class _Root:
    """A root: the operator, or one region of a split.  ``region`` = (dim, lo, hi) for a
    split region (the region's own loop over dim), None for the operator root.  ``items`` = the loops
    below it, in nest order, and references (names) to child roots after a split."""

    def __init__(self, name, region=None):
        self.name = name
        self.region: Optional[Tuple[str, int, int]] = region
        self.items: List[object] = []


def _norm_ann(ann: Dict[str, int], size: int) -> Tuple:
    a = dict(ann)
    if "vectorize" in a:
        a.setdefault("unroll", size)          # vectorization implicitly unrolls
    return tuple(sorted(a.items()))


class Scheduler:
    """The scheduling state of one matmul operator (``desc``), driven by the Fig.4 primitives or by
    ``descript`` (Fig.8).  ``root`` is the operator id (the paper's ``mm0``)."""

    def __init__(self, desc: xtc_op_desc, root: str = "mm0"):
        if desc.kind != XTC_OP_MATMUL:
            raise ScheduleError("the loop-nest front-ends lower matmul (I, J, K); conv2d schedules use the knobs")
        self.desc = desc
        self.root_name = root
        self.extent = {"I": int(desc.m), "J": int(desc.n), "K": int(desc.k)}
        self.log: List[Tuple[str, dict]] = []
        self._reset()

    def _reset(self):
        self.roots: Dict[str, _Root] = {}
        r = _Root(self.root_name)
        for d in ("I", "J", "K"):
            r.items.append(_Loop(d, d, self.extent[d]))
        self.roots[self.root_name] = r
        self._dims = ["I", "J", "K"]

    # ------------------------------------------------------- primitives --
    @property
    def dims(self):
        return list(self._dims)

    @dims.setter
    def dims(self, names):
        names = list(names)
        if names != ["I", "J", "K"]:
            raise ScheduleError("matmul dims are ['I', 'J', 'K'] (P:349-352)")
        self._record("dims", names=names)

    def _record(self, prim, **kw):
        self.log.append((prim, copy.deepcopy(kw)))

    def _root(self, name) -> _Root:
        if name not in self.roots:
            raise ScheduleError(f"unknown root {name!r} (roots: {list(self.roots)})")
        return self.roots[name]

    def _find(self, root: _Root, name: str) -> int:
        for i, it in enumerate(root.items):
            if isinstance(it, _Loop) and it.name == name:
                return i
        raise ScheduleError(f"no loop {name!r} in root {root.name!r}")

    def _loop(self, root: _Root, name: str) -> _Loop:
        return root.items[self._find(root, name)]

    def split(self, root: str, dim: str, segments: Dict[str, int]):
        """Split loop ``dim`` of ``root`` into contiguous regions starting at the given offsets
        (P:516-527); each region becomes a new root holding a copy of the loops inside ``dim``."""
        r = self._root(root)
        i = self._find(r, dim)
        loop = r.items[i]
        lo0 = r.region[1] if (r.region and r.region[0] == dim) else 0
        starts = sorted(segments.items(), key=lambda kv: kv[1])
        if starts[0][1] != 0:
            raise ScheduleError("the first segment must start at 0")
        inner = r.items[i + 1:]
        if any(not isinstance(it, _Loop) for it in inner):
            raise ScheduleError("split below an existing split is not supported")
        names = []
        for k, (nm, lo) in enumerate(starts):
            hi = starts[k + 1][1] if k + 1 < len(starts) else loop.size
            if not 0 <= lo < hi <= loop.size:
                raise ScheduleError(f"segment {nm!r} = [{lo}, {hi}) is empty or outside [0, {loop.size})")
            if nm in self.roots:
                raise ScheduleError(f"root {nm!r} exists")
            child = _Root(nm, (dim, lo0 + lo, lo0 + hi))
            child.items = [_Loop(it.name, it.dim, it.size, it.ann) for it in inner]
            self.roots[nm] = child
            names.append(nm)
        r.items = r.items[:i] + names
        self._record("split", root=root, dim=dim, segments=dict(segments))

    def strip_mine(self, root: str, dim: str, tiles: Dict[str, int]):
        """Tile loop ``dim``: each (name, size) adds a loop of that size immediately inside
        the previous one (the first right inside ``dim``'s innermost loop, or at the top of a split
        region whose own loop is ``dim``)."""
        r = self._root(root)
        pos = None
        for k, it in enumerate(r.items):
            if isinstance(it, _Loop) and it.dim == dim:
                pos = k
        at = 0 if pos is None else pos + 1
        if pos is None and not (r.region and r.region[0] == dim):
            raise ScheduleError(f"root {root!r} has no loop along {dim!r}")
        for nm, size in tiles.items():
            if int(size) < 1:
                raise ScheduleError("tile sizes must be >= 1")
            r.items.insert(at, _Loop(nm, dim, int(size)))
            at += 1
        self._record("strip_mine", root=root, dim=dim, tiles=dict(tiles))

    def interchange(self, root: str, permutation: List[str]):
        """Reorder the loops (and child roots) of ``root``."""
        r = self._root(root)
        key = lambda it: it.name if isinstance(it, _Loop) else it
        cur = {key(it): it for it in r.items}
        if sorted(cur) != sorted(permutation):
            raise ScheduleError(f"interchange of {root!r}: {permutation} is not a permutation of {sorted(cur)}")
        r.items = [cur[n] for n in permutation]
        self._record("interchange", root=root, permutation=list(permutation))

    def _annotate(self, root, names, what, value=1):
        r = self._root(root)
        for n in names:
            self._loop(r, n).ann[what] = value

    def unroll(self, root: str, unrolls: Dict[str, int]):
        r = self._root(root)
        for n, f in unrolls.items():
            lp = self._loop(r, n)
            if f < 1 or lp.size % int(f):
                raise ScheduleError(f"unroll factor {f} must divide the trip count {lp.size} of {n!r} (S:271)")
            lp.ann["unroll"] = int(f)
        self._record("unroll", root=root, unrolls=dict(unrolls))

    def vectorize(self, root: str, axes: List[str]):
        self._annotate(root, axes, "vectorize")
        self._record("vectorize", root=root, axes=list(axes))

    def parallelize(self, root: str, axes: List[str]):
        self._annotate(root, axes, "parallelize")
        self._record("parallelize", root=root, axes=list(axes))

    def pack(self, root: str, at: str, stages: int = 2):
        """Pack the operands below loop ``at`` into a ``stages``-deep shared-memory ring."""
        self._annotate(root, [at], "pack", int(stages))
        self._record("pack", root=root, at=at, stages=int(stages))

    def bufferize(self, root: str, at: str):
        """A local output buffer below loop ``at``: staged in shared memory, TMA-stored."""
        self._annotate(root, [at], "buffer")
        self._record("bufferize", root=root, at=at)

    # --------------------------------------------------------- descript --
    _KEY = re.compile(r"^([A-Za-z]\w*?)(?:#(\d+)|\[(\d+):(\d+)\])?$")

    def descript(self, spec: dict):
        """The declarative form (Fig.8): the whole loop nest at once (replaces the current state)."""
        self._reset()
        self.log = [("descript", {"spec": copy.deepcopy(spec)})]
        root = self.roots[self.root_name]
        root.items = []
        self._fill(root, spec, {"I": (0, self.extent["I"]), "J": (0, self.extent["J"]),
                                "K": (0, self.extent["K"])}, path=self.root_name)

    def _fill(self, root: _Root, spec: dict, rng: Dict[str, Tuple[int, int]], path: str):
        seen_outer = set()
        splits: Dict[str, List[Tuple[int, int, dict]]] = {}
        order: List[Tuple[str, object]] = []
        for key, val in spec.items():
            m = self._KEY.match(str(key))
            if not m or m.group(1) not in self.extent:
                raise ScheduleError(f"descript key {key!r}: expected D, D#N or D[A:B] with D in I, J, K")
            d = m.group(1)
            if m.group(3) is not None:                       # split region
                if not isinstance(val, dict):
                    raise ScheduleError(f"{key!r}: a split region carries a dict (its inner schedule)")
                lo, hi = int(m.group(3)), int(m.group(4))
                if d in splits:
                    splits[d].append((lo, hi, val))
                else:
                    splits[d] = [(lo, hi, val)]
                    order.append(("split", d))
                continue
            if isinstance(val, dict):
                raise ScheduleError(f"{key!r}: only split regions carry an inner dict")
            ann = {}
            for a in (val or []):
                nm, _, v = str(a).partition("=")
                if nm not in ANNOTATIONS:
                    raise ScheduleError(f"{key!r}: unknown annotation {a!r} (one of {ANNOTATIONS})")
                ann[nm] = int(v) if v else (0 if nm == "unroll" else 1)
            if m.group(2) is None:
                if d in seen_outer:
                    raise ScheduleError(f"{key!r} declared twice")
                seen_outer.add(d)
                size = rng[d][1] - rng[d][0]
            else:
                size = int(m.group(2))
            if ann.get("unroll") == 0:
                ann["unroll"] = size                           # 'unroll' = the whole tile
            order.append(("loop", _Loop(str(key), d, size, ann)))
        n_split = 0
        for kind, obj in order:
            if kind == "loop":
                root.items.append(obj)
                continue
            d = obj
            regs = sorted(splits[d], key=lambda t: t[0])
            lo0, hi0 = rng[d]
            if regs[0][0] != lo0 - lo0 or regs[-1][1] != hi0 - lo0 or any(
                    regs[i][1] != regs[i + 1][0] for i in range(len(regs) - 1)):
                raise ScheduleError(f"split regions of {d} must tile [0, {hi0 - lo0}) contiguously")
            for lo, hi, sub in regs:
                nm = f"{d}[{lo}:{hi}]" if path == self.root_name else f"{path}/{d}[{lo}:{hi}]"
                child = _Root(nm, (d, lo0 + lo, lo0 + hi))
                r2 = dict(rng)
                r2[d] = (lo0 + lo, lo0 + hi)
                self.roots[nm] = child
                self._fill(child, sub, r2, nm)
                root.items.append(nm)
            n_split += 1
            if n_split > 1:
                raise ScheduleError("one split per root")

    # ------------------------------------------------------- canonical --
    def _canon(self, root: _Root) -> Tuple:
        out = []
        pending = None
        for it in root.items:
            if isinstance(it, _Loop):
                if pending:
                    out.append(pending)
                    pending = None
                out.append((it.dim, int(it.size), _norm_ann(it.ann, it.size)))
            else:
                ch = self.roots[it]
                d, lo, hi = ch.region
                if pending and pending[1] == d:
                    pending = ("split", d, pending[2] + ((lo, hi, self._canon(ch)),))
                else:
                    if pending:
                        out.append(pending)
                    pending = ("split", d, ((lo, hi, self._canon(ch)),))
        if pending:
            out.append(pending)
        return tuple(out)

    def nest(self) -> Tuple:
        """The canonical loop nest (names dropped; see the module docstring)."""
        return self._canon(self.roots[self.root_name])

    @classmethod
    def replay(cls, desc: xtc_op_desc, log, root: str = "mm0") -> "Scheduler":
        """Rebuild a Scheduler from a primitive log."""
        s = cls(desc, root)
        for prim, kw in log:
            if prim == "dims":
                s.dims = kw["names"]
            else:
                getattr(s, prim)(**copy.deepcopy(kw))
        return s

    # ----------------------------------------------------------- lower --
    def knobs(self, target: Optional[dict] = None) -> dict:
        """The xtc_schedule fields for this loop nest (module docstring; reading 23)."""
        target = dict(target or {})
        engine = target.pop("engine", XTC_ENGINE_SIMT if self.desc.in_dtype == XTC_F32 else XTC_ENGINE_TCGEN05)
        nest = self.nest()
        kn: Dict[str, int] = {"engine": engine}
        # flatten: the loops above a split + the main region's loops (the region's own loop first)
        flat: List[Tuple[str, int, Tuple]] = []
        entries = list(nest)
        while entries:
            e = entries.pop(0)
            if e[0] != "split":
                flat.append(e)
                continue
            if entries:
                raise ScheduleError("loops after a split region are not supported")
            _, d, regs = e
            if d == "J":
                if len(regs) != 2:
                    raise ScheduleError("a split of J lowers to [0, s) + the remainder root [s, N): two regions")
                (lo, s, main), (_, hi, tail) = regs
                if any(x[0] != "K" or x[2] for x in tail) or len(tail) != 1:
                    raise ScheduleError("the J remainder region must be a plain K loop (the SIMT remainder root)")
                kn["split_n_at"] = s
                flat.append(("J", s - lo, ()))
                entries = list(main)
            elif d == "K":
                sizes = {hi - lo for lo, hi, _ in regs}
                subs = {sub for _, _, sub in regs}
                if len(sizes) != 1 or len(subs) != 1:
                    raise ScheduleError("a split of K lowers to split_k: equal regions, identical sub-nests")
                kn["split_k"] = len(regs)
                flat.append(("K", sizes.pop(), ()))
                entries = list(regs[0][2])
            else:
                raise ScheduleError("a split of I has no GPU lowering (split J or K)")
        dims = [e[0] for e in flat]
        if "K" not in dims:
            raise ScheduleError("no K loop")
        kpos = dims.index("K")

        def step(i):
            for e in flat[i + 1:]:
                if e[0] == flat[i][0]:
                    return e[1]
            return 1

        outer = {d: [i for i in range(kpos) if flat[i][0] == d] for d in ("I", "J")}
        for d in ("I", "J"):
            if not outer[d]:
                raise ScheduleError(f"loop {d} must be placed above the reduction loop K (reading 15)")
        reg = {d: step(outer[d][-1]) for d in ("I", "J")}
        cta = {}
        for d in ("I", "J"):
            par = [i for i in outer[d] if dict(flat[i][2]).get("parallelize")]
            cta[d] = step(par[-1]) if par else reg[d]
        kn["order"] = 0 if dims.index("I") < dims.index("J") else 1
        kn["tile_m"], kn["tile_n"] = cta["I"], cta["J"]
        kloops = [i for i, e in enumerate(flat) if e[0] == "K"]
        kn["tile_k"] = step(kloops[0])
        inner_k = kloops[-1]
        un = dict(flat[inner_k][2]).get("unroll")
        if un and len(kloops) > 1:
            kn["unroll_k"] = un
        packs = [dict(flat[i][2]).get("pack") for i in kloops if dict(flat[i][2]).get("pack")]
        kn["stages"] = packs[0] if packs else (1 if engine == XTC_ENGINE_SIMT else 2)
        jloops = [i for i, e in enumerate(flat) if e[0] == "J"]
        if dict(flat[jloops[-1]][2]).get("vectorize"):
            kn["vector_n"] = 4
        if any(dict(e[2]).get("buffer") for e in flat):
            kn["buffer_c"] = 1
        if engine == XTC_ENGINE_SIMT:
            kn["inner_m"], kn["inner_n"] = reg["I"], reg["J"]
        else:
            if (reg["I"], reg["J"]) != (cta["I"], cta["J"]):
                raise ScheduleError("tcgen05: the tile the K loop sees is the UMMA atom = the CTA tile "
                                    "(parallelize the loops that step by it)")
            kn.pop("vector_n", None)
            kn["swizzle"] = 128
        kn.update(target)
        return kn

    def schedule(self, target: Optional[dict] = None) -> xtc_schedule:
        return schedule(**self.knobs(target))

    def check(self, target: Optional[dict] = None, num_sms: int = 148):
        """(status, plan_info, reason) of the lowered schedule from the C planner."""
        return xtc_schedule_check(self.desc, self.schedule(target), num_sms)

    def apply(self, op_handle, target: Optional[dict] = None) -> None:
        """xtc_schedule_apply of the lowered schedule (the Compiler step)."""
        xtc_schedule_apply(op_handle, self.schedule(target))
