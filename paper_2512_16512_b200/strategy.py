"""a10 -- design spaces, seeded sampling and generation (§V-B).

The paper's ``Strategy`` interface:
  * ``sample(num) -> list[Sample]``         seeded draws from the design space
  * ``generate(sch, sample)``               puts the scheduler in the sample's state
  * ``default_schedule(opt_level)``         heuristic default

Here a Sample is a flat vector of knob values and
``generate`` returns the ``xtc_schedule`` the C planner applies.  Samples
are drawn uniformly *with replacement* from the enumerated legal set, so
legality holds by construction; legality itself is the
C planner's verdict (``xtc_schedule_check``), never re-implemented here.

Also here, as host-side helpers with their paper pins:
  * ``divisor_tiles`` / ``goto_space_size``: the §VI-A enumeration rule
    ("register tile 4x32, outer tile sizes free under divisibility",
    1024x1024 -> 594 instances).
  * ``prt_tiles``: the StrategyPRT sample -> tile-size semantics of Fig.9
    (reading 18).
"""
from __future__ import annotations

import itertools
import random
from typing import Dict, List, Sequence

from . import (XTC_ENGINE_SIMT, XTC_ENGINE_TCGEN05, XTC_OK, schedule, xtc_op_desc, xtc_schedule,
               xtc_schedule_check, xtc_schedule_default, gemm_view)


# ----------------------------------------------------------- paper pins ----
def divisors(n: int) -> List[int]:
    return [d for d in range(1, n + 1) if n % d == 0]


def divisor_tiles(extent: int, multiple_of: int = 1) -> List[int]:
    """Tile sizes 'free under divisibility': divisors of the extent that are
    multiples of the inner (register) tile."""
    return [d for d in divisors(extent) if d % multiple_of == 0]


def goto_space_size(m: int, n: int, k: int, reg_m: int, reg_n: int) -> int:
    """Size of the §VI-A Goto design space: one outer tile per dim, each a
    divisor of the extent and a multiple of the register tile (K free)."""
    return len(divisor_tiles(m, reg_m)) * len(divisor_tiles(n, reg_n)) * len(divisor_tiles(k, 1))


def prt_tiles(sample: Sequence[int], n_pdims: int = 2, p_levels: int = 3, r_levels: int = 1,
              pdim_names=("i", "j"), rdim_names=("k",)) -> Dict[str, object]:
    """StrategyPRT sample semantics (reading 18): for each parallel
    dim, ``p_levels`` inner trip counts (outer -> inner); then for each
    reduction dim ``r_levels`` trip counts; then the W flag.  The tile size at
    level l is the product of the trip counts of levels >= l.
    Fig.9: [1,16,4, 4,1,16, 16, 1] -> i1=64 i2=64 i3=4, j1=64 j2=16 j3=16, k1=16, W."""
    s = list(sample)
    need = n_pdims * p_levels + len(rdim_names) * r_levels + 1
    if len(s) != need:
        raise ValueError(f"sample has {len(s)} entries, expected {need}")
    out: Dict[str, object] = {}
    pos = 0
    for name in pdim_names[:n_pdims]:
        trips = s[pos:pos + p_levels]
        pos += p_levels
        for lvl in range(p_levels):
            t = 1
            for v in trips[lvl:]:
                t *= v
            out[f"{name}{lvl + 1}"] = t
    for name in rdim_names:
        trips = s[pos:pos + r_levels]
        pos += r_levels
        for lvl in range(r_levels):
            t = 1
            for v in trips[lvl:]:
                t *= v
            out[f"{name}{lvl + 1}"] = t
    out["W"] = bool(s[pos])
    return out


# ------------------------------------------------------ GPU design space ---
# The B200 loop-nest hierarchy is a P P W R P R P sketch:
# P grid-tile raster | P CTA tile | W TMEM accumulator | R k-stage ring |
# P UMMA atom | R UMMA k-steps | P instruction tile.  Slots below are the
# free choices of that sketch.
TC_SLOTS = {
    "cluster_m": [1, 2],          # parallelize: 1 CTA or a CTA pair (cta_group::2)
    "m_subtiles": [1, 2],         # strip_mine: 128-row UMMA subtiles per CTA (tile_m = 128 x cluster_m x this)
    "cluster_n": [1, 2],          # parallelize: CTAs on adjacent N tiles sharing A stages by multicast
    "tile_n": [64, 128, 192, 256],
    "tile_k": [64, 128],
    "stages": [2, 3, 4, 5, 6, 7, 8],
    "order": [0, 1],
    "raster_group": [1, 2, 4, 8],
    "split_k": [1, 2, 4, 8],
    "split_k_mode": [0, 2, 3],    # split: reduction by a second kernel, in-kernel across a cluster, stream-K
    "buffer_c": [0, 1],
    "acc_buffers": [1, 2],
    "persistent": [0, 1],
}

SIMT_SLOTS = {
    "tile_m": [16, 32, 64, 128],
    "tile_n": [16, 32, 64, 128],
    "tile_k": [8, 16, 32],
    "inner_m": [1, 2, 4, 8],
    "inner_n": [1, 2, 4, 8],
    "unroll_k": [1, 4],
    "vector_n": [1, 4],
    "stages": [1, 2],
    "order": [0, 1],
    "split_k": [1, 2],
}


class GpuStrategy:
    """Seeded sampler over the legal schedules of one operator."""

    def __init__(self, desc: xtc_op_desc, engine: int = XTC_ENGINE_TCGEN05, slots: Dict[str, list] = None,
                 exact_divisors: bool = True, num_sms: int = 148):
        self.desc = desc
        self.engine = engine
        self.slots = dict(slots or (TC_SLOTS if engine == XTC_ENGINE_TCGEN05 else SIMT_SLOTS))
        self.exact_divisors = exact_divisors
        self.num_sms = num_sms
        self._legal = None

    def _base(self) -> Dict[str, int]:
        if self.engine == XTC_ENGINE_TCGEN05:
            return dict(engine=XTC_ENGINE_TCGEN05, tile_m=128, swizzle=128)
        return dict(engine=XTC_ENGINE_SIMT)

    def _kw(self, names, values) -> Dict[str, int]:
        kw = self._base()
        kw.update({n: int(v) for n, v in zip(names, values)})
        if self.engine == XTC_ENGINE_TCGEN05:
            # UMMA M = 128 per CTA; m_subtiles (a slot, not a schedule field) stacks 1 or 2 per CTA
            kw["tile_m"] = 128 * max(1, kw.get("cluster_m", 1)) * max(1, kw.pop("m_subtiles", 1))
        return kw

    def generate(self, sample: Sequence[int]) -> xtc_schedule:
        """Sample (flat vector in slot order) -> schedule (the planner input)."""
        return schedule(**self._kw(list(self.slots), sample))

    def _divisible(self, kw) -> bool:
        if not self.exact_divisors:
            return True
        M, N, K = gemm_view(self.desc)
        tm = kw.get("tile_m", 128)
        if M % tm or N % kw["tile_n"]:
            return False
        return K % (kw.get("tile_k", 1) * kw.get("split_k", 1)) == 0

    def legal_samples(self) -> List[tuple]:
        """All legal samples, in slot-product order (the enumerated design space)."""
        if self._legal is None:
            names = list(self.slots)
            legal = []
            for combo in itertools.product(*(self.slots[n] for n in names)):
                kw = self._kw(names, combo)
                if not self._divisible(kw):
                    continue
                if kw.get("split_k", 1) <= 1 and kw.get("split_k_mode", 0) == 2:
                    continue                      # no split: the cluster reduction is moot (one schedule, not two)
                st, _, _ = xtc_schedule_check(self.desc, schedule(**kw), self.num_sms)
                if st == XTC_OK:
                    legal.append(tuple(combo))
            self._legal = legal
        return self._legal

    def sample(self, num: int, seed: int = 0) -> List[tuple]:
        """`num` draws, uniform with replacement over the legal set (duplicates
        allowed); deterministic for a given seed."""
        legal = self.legal_samples()
        if not legal:
            return []
        rng = random.Random(seed)
        return [legal[rng.randrange(len(legal))] for _ in range(num)]

    def default_schedule(self, opt_level: int = 2) -> xtc_schedule:
        return xtc_schedule_default(self.desc, opt_level)
