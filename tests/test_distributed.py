"""N>1 host logic on CPU: world-size-2 gloo groups run the row partition, the
B all-gather and the offset exchange; each rank computes its C rows with the
CPU oracle (the checker) and the gathered result must equal the single-rank
product.  The device kernels are the same as on one GPU."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from paper_1804_00695_b200 import distributed as D
    from paper_1804_00695_b200 import generators as gen
    from paper_1804_00695_b200.csr import CsrMatrix, slice_rows
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = gen.stencil(gen.BRICK3D, (6, 6, 4 * world))
        p, r = gen.aggregation((6, 6, 4 * world))
        # B = A, row-sharded by rank; replicate with one all-gather
        lo, hi = rank * a.num_rows // world, (rank + 1) * a.num_rows // world
        shard = slice_rows(a, lo, hi)
        rp, cols, vals = D.allgather_csr(torch.from_numpy(np.diff(shard.row_ptr)),
                                         torch.from_numpy(shard.col_idx),
                                         torch.from_numpy(shard.values), dist, "cpu")
        b_full = CsrMatrix(a.num_rows, a.num_cols, rp.numpy(), cols.numpy(), vals.numpy())
        assert np.array_equal(b_full.col_idx, a.col_idx) and np.array_equal(b_full.values, a.values)
        # flops-balanced row partition of R, local product, offset exchange
        flops = np.diff(a.row_ptr)[r.col_idx]
        row_flops = np.add.reduceat(flops, r.row_ptr[:-1]) if r.nnz else np.zeros(r.num_rows)
        bounds = D.flops_partition(row_flops, world)
        r_loc = slice_rows(r, int(bounds[rank]), int(bounds[rank + 1]))
        ptr, col, val = O.multiply(r_loc, b_full)
        off, total = D.exchange_offsets(len(col), dist, "cpu")
        q.put((rank, int(bounds[rank]), int(bounds[rank + 1]), off, total, ptr, col, val,
               bounds.tolist(), [int(row_flops[int(bounds[k]):int(bounds[k + 1])].sum())
                                 for k in range(world)]))
    finally:
        dist.destroy_process_group()


def test_two_rank_row_partition_matches_single_rank():
    from paper_1804_00695_b200 import generators as gen
    from oracle import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=180) for _ in range(world)])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    a = gen.stencil(gen.BRICK3D, (6, 6, 4 * world))
    _, r = gen.aggregation((6, 6, 4 * world))
    ptr, col, val = O.multiply(r, a)
    total = len(col)
    for rank, lo, hi, off, tot, lp, lc, lv, bounds, per in res:
        assert tot == total
        assert off == int(ptr[lo])
        assert np.array_equal(lc, col[ptr[lo]:ptr[hi]])
        assert np.array_equal(lv, val[ptr[lo]:ptr[hi]])
    assert res[0][8][0] == 0 and res[0][8][-1] == r.num_rows
    per = res[0][9]
    assert max(per) <= 1.2 * min(per)        # flops-balanced


def test_flops_partition_properties():
    from paper_1804_00695_b200.distributed import flops_partition
    rng = np.random.default_rng(3)
    for world in (1, 2, 4, 8):
        f = rng.integers(0, 1000, size=500) ** 2
        b = flops_partition(f, world)
        assert b[0] == 0 and b[-1] == 500 and np.all(np.diff(b) >= 0)
        parts = [int(f[b[k]:b[k + 1]].sum()) for k in range(world)]
        assert max(parts) - min(parts) <= 2 * int(f.max())


def _shard_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    import torch.multiprocessing as tmp
    from paper_1804_00695_b200 import distributed as D
    from paper_1804_00695_b200 import generators as gen
    tmp.set_sharing_strategy("file_system")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = gen.stencil(gen.LAPLACE3D, (5, 5, 3 * world))
        bounds = D.shard_bounds(np.diff(b.row_ptr), world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        local = D.local_shard_tensors(b, lo, hi, "cpu")
        shards = D.share_shards(local, lo, hi, dist)
        # every rank sees every shard, in row order, with the owner's contents
        got = []
        for lo_r, hi_r, rp, col, val in shards:
            e0 = int(b.row_ptr[lo_r])
            got.append((lo_r, hi_r, bool(np.array_equal(rp.numpy() + e0, b.row_ptr[lo_r:hi_r + 1])),
                        bool(np.array_equal(col.numpy(), b.col_idx[e0:int(b.row_ptr[hi_r])])),
                        bool(np.array_equal(val.numpy(), b.values[e0:int(b.row_ptr[hi_r])]))))
        dist.barrier()
        q.put((rank, got, bounds.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_b_shards_shared():
    """B sharded (§8e): each rank publishes its row shard as tensor handles;
    every rank can read all shards in row order (CPU tensors here, CUDA IPC
    handles into peer HBM on GPUs)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, got, bounds in res:
        assert bounds[0] == 0 and len(got) == world
        assert [g[0] for g in got] == bounds[:-1] and [g[1] for g in got] == bounds[1:]
        assert all(g[2] and g[3] and g[4] for g in got)
