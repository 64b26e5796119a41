"""Multi-GPU partitioning of the hot path.

Only the two shardings the path has are implemented:
  1. candidate data-parallelism: a sweep's schedule candidates are dealt to
     ranks by id (id mod world == rank); every rank regenerates identical inputs
     and the identical candidate list from the seed; fixed-size records are
     collected with one all-gather (NCCL over NVLink on the GPU box).
  2. M-sharding of a large GEMM (conv: batch sharding): rank r computes the
     contiguous output rows [r0, r1); B is replicated by regenerating it from
     the seed (no broadcast); C is assembled by all_gather_into_tensor.
     With the gather FUSED into the GEMM (xtc_run_gather), C is a
     symmetric-memory buffer on every rank and each rank's epilogue TMA-stores its
     tiles straight into every peer's copy over NVLink (no NCCL call on the data path).
There is no tensor/pipeline/sequence parallelism: the operator has none.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch

# record layout of one measured candidate (float64 slots)
REC_FIELDS = ["id", "status", "valid", "max_norm_err", "n_mismatch", "n_nan", "t_min_ns", "t_med_ns",
              "tflops_med", "sm_clock_mhz"]
REC = len(REC_FIELDS)


def shard_rows(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced row range of `rank` (the first m % world ranks get one more row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(m, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def rank_candidates(n: int, world: int, rank: int) -> List[int]:
    """Candidate ids of `rank`: interleaved (id mod world) to balance random per-candidate cost."""
    return list(range(rank, n, world))


def pack_records(ids: Sequence[int], metrics: Sequence, rows: int) -> torch.Tensor:
    """Fixed-size [rows, REC] float64 block; unused rows have id = -1.  One numpy pass over the
    records (no per-row tensor construction: this runs inside the sweep's timed region)."""
    import numpy as np
    t = np.full((rows, REC), -1.0, dtype=np.float64)
    n = min(len(ids), rows)
    if n:
        fields = REC_FIELDS[1:]
        if isinstance(metrics[0], dict):
            vals = [[m.get(f, 0.0) for f in fields] for m in metrics[:n]]
        else:
            vals = [[getattr(m, f) for f in fields] for m in metrics[:n]]
        t[:n, 0] = np.asarray(ids[:n], dtype=np.float64)
        t[:n, 1:] = np.asarray(vals, dtype=np.float64)
    return torch.from_numpy(t)


def unpack_gathered(gathered: torch.Tensor, n: int) -> List[dict]:
    """[world*rows, REC] -> list of n records ordered by candidate id."""
    out = [None] * n
    for row in gathered.tolist():
        cid = int(row[0])
        if 0 <= cid < n:
            out[cid] = dict(zip(REC_FIELDS, row))
            out[cid]["id"] = cid
    missing = [i for i, r in enumerate(out) if r is None]
    if missing:
        raise RuntimeError(f"records missing for candidates {missing[:8]}...")
    return out


def _all_gather(out: torch.Tensor, local: torch.Tensor, group=None) -> None:
    """all_gather_into_tensor; NCCL gathers device tensors in place over NVLink.  The
    gloo backend (CPU tests, or the single-GPU rehearsal of the multi-rank bench)
    gathers through host copies."""
    import torch.distributed as dist
    if dist.get_backend(group) == "gloo" and local.is_cuda:
        host = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(host, local.cpu(), group=group)
        out.copy_(host)
    else:
        dist.all_gather_into_tensor(out, local, group=group)


def gather_records(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather the per-rank record blocks (NCCL on GPU tensors, gloo on CPU)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty((world * local.shape[0], local.shape[1]), dtype=local.dtype, device=local.device)
    _all_gather(out, local, group)
    return out


def gather_rows(c_shard: torch.Tensor, m_total: int, group=None, out: torch.Tensor = None) -> torch.Tensor:
    """Assemble C from equal row shards (M-sharded GEMM, config 5)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if m_total % world:
        raise ValueError("all_gather_into_tensor needs equal shards: M % world must be 0")
    if out is None:
        out = torch.empty((m_total,) + tuple(c_shard.shape[1:]), dtype=c_shard.dtype, device=c_shard.device)
    _all_gather(out, c_shard.contiguous(), group)
    return out


def rotated_destinations(ptrs: Sequence[int], rank: int) -> List[int]:
    """Destination order of the fused all-gather for `rank`: its own buffer first, then the
    peers r+1, r+2, ... (mod W), so at any moment the W ranks' stores target W different
    GPUs instead of all starting on rank 0's buffer."""
    w = len(ptrs)
    if not 0 <= rank < w:
        raise ValueError("rank out of range")
    return [int(ptrs[(rank + i) % w]) for i in range(w)]


class SymmetricOutput:
    """C as a symmetric-memory tensor (torch.distributed._symmetric_memory: every rank's buffer
    mapped into every peer's address space over NVLink).  ``dests`` are the device pointers
    xtc_run_gather stores to (this rank's first); ``barrier()`` (on the current stream) orders
    every rank's stores before any later read."""

    def __init__(self, shape, dtype, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        group = group or dist.group.WORLD
        self.tensor = symm.empty(*shape, dtype=dtype, device=device)
        self.handle = symm.rendezvous(self.tensor, group)
        self.dests = rotated_destinations(list(self.handle.buffer_ptrs), dist.get_rank(group))
        # NVLS multicast address of the same buffer on every rank (0 when the allocator could not
        # set one up): with it the epilogue stores each tile once and the switch replicates it
        try:
            self.multicast_ptr = int(self.handle.multicast_ptr)
        except Exception:  # noqa: BLE001 -- older allocators have no multicast
            self.multicast_ptr = 0

    def barrier(self):
        self.handle.barrier(channel=0)


def checksum_rows(c: torch.Tensor) -> torch.Tensor:
    """Order-sensitive integer checksum of a 2-D tensor's bits (sum, and sum weighted by the
    row index), computed in row blocks; equal on every rank iff the gathered copies agree
    (up to checksum collisions)."""
    bits = c.view(torch.int16 if c.element_size() == 2 else torch.int32)
    out = torch.zeros(2, dtype=torch.int64, device=c.device)
    step = max(1, (1 << 24) // max(1, c.shape[1]))
    for r0 in range(0, c.shape[0], step):
        x = bits[r0:r0 + step].to(torch.int64)
        rows = torch.arange(r0 + 1, r0 + 1 + x.shape[0], device=c.device, dtype=torch.int64)[:, None]
        out[0] += x.sum()
        out[1] += (x * rows).sum()
    return out
