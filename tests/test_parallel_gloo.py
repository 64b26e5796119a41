"""world_size-2 gloo tests (CPU) of the multi-GPU host logic (§8(e)):
candidate dealing + record all-gather, and M-sharded GEMM row assembly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_16512_b200.parallel import (REC_FIELDS, gather_records, gather_rows, pack_records,
                                            rank_candidates, rotated_destinations, shard_rows, unpack_gathered,
                                            checksum_rows)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1) sweep records: ids dealt by id % world, fixed-size blocks, one all-gather
        n = 13
        mine = rank_candidates(n, world, rank)
        recs = [{f: float(cid * 10 + j) for j, f in enumerate(REC_FIELDS[1:])} for cid in mine]
        rows = (n + world - 1) // world
        g = gather_records(pack_records(mine, recs, rows))
        allr = unpack_gathered(g, n)
        assert [r["id"] for r in allr] == list(range(n))
        assert all(r["status"] == r["id"] * 10 for r in allr)
        # 2) M-sharded GEMM: every rank regenerates B and its rows of A from the seed
        from seeded_inputs import MODE_INT, gen_f32
        M, N, K = 64, 24, 40
        r0, r1 = shard_rows(M, world, rank)
        A = gen_f32(1, M * K, MODE_INT).reshape(M, K)
        B = gen_f32(2, K * N, MODE_INT).reshape(K, N)
        import oracle
        C_r, _ = oracle.matmul(A[r0:r1].astype(np.float64), B.astype(np.float64))
        full = gather_rows(torch.from_numpy(C_r), M)
        want, _ = oracle.matmul(A.astype(np.float64), B.astype(np.float64))
        assert np.array_equal(full.numpy(), want)
        # 3) the overlapped form (bench.py N>1): CH block-cyclic chunks of Mc rows per rank, chunk j
        #    of rank r = global rows (j*W + r)*Mc ...; gathering chunk by chunk assembles C in order
        CH = 4
        Mc = M // (world * CH)
        rows_mine = np.concatenate([np.arange((j * world + rank) * Mc, (j * world + rank + 1) * Mc)
                                    for j in range(CH)])
        C_bc, _ = oracle.matmul(A[rows_mine].astype(np.float64), B.astype(np.float64))
        C_bc = torch.from_numpy(C_bc)
        full_bc = torch.empty((M, N), dtype=C_bc.dtype)
        for j in range(CH):
            gather_rows(C_bc[j * Mc:(j + 1) * Mc].contiguous(), world * Mc,
                        out=full_bc[j * world * Mc:(j + 1) * world * Mc])
        assert np.array_equal(full_bc.numpy(), want)
        # 4) fused gather (xtc_run_gather, bench.py --gather fused): each rank stores to its own
        #    buffer first, then to the peers in rotation; the consistency check compares
        #    whole-buffer checksums across ranks
        order = rotated_destinations([100 + r for r in range(world)], rank)
        assert order[0] == 100 + rank and sorted(order) == [100 + r for r in range(world)]
        c32 = torch.from_numpy(want.astype(np.float32))
        cs = checksum_rows(c32)
        cs_all = [torch.empty_like(cs) for _ in range(world)]
        dist.all_gather(cs_all, cs)
        assert all(torch.equal(x, cs_all[0]) for x in cs_all)
        swapped = c32.clone()
        swapped[[0, 1]] = swapped[[1, 0]]
        assert not torch.equal(checksum_rows(swapped), cs)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_shard_rows_cover_exactly():
    for m in (1, 7, 8192):
        for w in (1, 2, 3, 8):
            spans = [shard_rows(m, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    assert rank_candidates(10, 4, 1) == [1, 5, 9]
