"""World-size-2 gloo run of the multi-GPU dataflow on CPU.

Each rank takes its contiguous shard [floor(gN/G), floor((g+1)N/G)), runs the
per-shard probe with its global row offset, and the two ranks merge with one
all-reduce(sum) over [n_sampled, counts, joints] and one all-reduce(max) over
the HLL registers -- the exchange the product does with NCCL.  The merged
result must equal the single-process whole-table probe bit for bit.  The
shard arithmetic and the unique-id broadcast are the product's host helpers
(paper_2512_19750_b200.dist), exercised here without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, nrows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import reference as R
        from paper_2512_19750_b200 import dist as gdist
        w = synth.get(name, nrows)
        r0, r1 = gdist.shard_range(rank, world, w.nrows)
        cols = [x.numpy() for x in w.table(r0, r1)]
        n, c, j, regs = R.probe(cols, w.preds, w.pairs, rate=0.7, seed=31,
                                hll_cols=w.hll_cols, row_offset=r0)
        sums = torch.tensor(np.concatenate([[n], c, j]).astype(np.int64))
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        mx = torch.tensor(regs.astype(np.int32))
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        uid = gdist.broadcast_unique_id(bytes(range(128)) if rank == 0 else None)
        if rank == 0:
            q.put((sums.numpy(), mx.numpy(), uid))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,nrows", [("C1", 10007), ("C5", 6001)])
def test_two_rank_merge_equals_whole(oracle, name, nrows):
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, nrows, q)) for r in range(2)]
    for p in procs:
        p.start()
    sums, mx, uid = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = synth.get(name, nrows)
    n, c, j, regs = oracle.probe([x.numpy() for x in w.table()], w.preds, w.pairs, rate=0.7,
                                 seed=31, hll_cols=w.hll_cols)
    assert sums[0] == n
    assert np.array_equal(sums[1:1 + len(c)], c.astype(np.int64))
    assert np.array_equal(sums[1 + len(c):], j.astype(np.int64))
    assert np.array_equal(mx, regs.astype(np.int32))
    assert uid == bytes(range(128))


def test_shard_ranges_cover():
    from paper_2512_19750_b200 import dist as gdist
    for N in (0, 1, 7, 600_037_902):
        for G in (1, 2, 3, 4, 8):
            rs = [gdist.shard_range(g, G, N) for g in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(e - s for s, e in rs) - min(e - s for s, e in rs) <= 1


def _plan_worker(rank, world, port, q):
    """Each rank plans the same batch for its own shard of C5 through the product's planner
    (host-only hook gace_debug_jit_source: the specialised kernel's layout-keyed source, i.e.
    every table offset, shift and constant of the plan), once over its shard's own value
    domains and once over the domains all-reduced (min / max) across the ranks -- what
    gace_table_attach does over NCCL for a multi-rank table -- and gets the NCCL unique id
    through the product's dist_info (rank 0 creates it, the process group broadcasts it)."""
    import ctypes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2512_19750_b200 import dist as gdist
        from paper_2512_19750_b200 import gace
        L = gace.lib()
        vp, u32, u64, i32, dbl = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        L.gace_debug_jit_source.argtypes = [u32, vp, vp, vp, i32, vp, u32, vp, u32, u64, dbl, i32, vp, u64,
                                            ctypes.POINTER(u64)]
        w = synth.get("C5", 40_000)
        r0, r1 = gdist.shard_range(rank, world, w.nrows)
        t = [x.numpy() for x in w.table(r0, r1)]
        lo = torch.tensor([int(x.min()) for x in t], dtype=torch.int64)
        hi = torch.tensor([int(x.max()) for x in t], dtype=torch.int64)

        def src(dlo, dhi):
            dt = np.zeros(len(t), dtype=np.int32)
            dl = np.ascontiguousarray(dlo.numpy(), dtype=np.int64)
            dh = np.ascontiguousarray(dhi.numpy(), dtype=np.int64)
            P = gace.as_preds(w.preds)
            Q = gace.as_pairs(w.pairs)
            buf = ctypes.create_string_buffer(1 << 17)
            n = ctypes.c_uint64()
            rc = L.gace_debug_jit_source(len(t), dt.ctypes.data, dl.ctypes.data, dh.ctypes.data, 0, P.ctypes.data,
                                         len(P), Q.ctypes.data, len(Q), w.hll_mask, 1.0, 1, buf, 1 << 17,
                                         ctypes.byref(n))
            assert rc == 0
            return buf.value.decode()

        own = src(lo, hi)
        glo, ghi = lo.clone(), hi.clone()
        dist.all_reduce(glo, op=dist.ReduceOp.MIN)
        dist.all_reduce(ghi, op=dist.ReduceOp.MAX)
        agreed = src(glo, ghi)
        info = gdist.dist_info(w.nrows)
        out = [None] * world
        dist.all_gather_object(out, (own, agreed, info.unique_id, info.row_offset, info.nranks))
        if rank == 0:
            whole = [x.numpy() for x in w.table()]
            q.put((out, src(torch.tensor([int(x.min()) for x in whole]), torch.tensor([int(x.max()) for x in whole]))))
    finally:
        dist.destroy_process_group()


def test_two_rank_plans_agree():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, whole = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (own0, agreed0, uid0, off0, n0), (own1, agreed1, uid1, off1, n1) = out
    assert own0 != own1                    # shard-local domains: the ranks would plan differently
    assert agreed0 == agreed1 == whole     # agreed domains: identical plans, the whole table's plan
    assert uid0 == uid1 and len(uid0) == 128 and n0 == n1 == 2
    assert (off0, off1) == (0, 20_000)
