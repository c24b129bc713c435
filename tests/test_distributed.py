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


def test_element_shards_fill_whole_granules():
    from paper_1804_00695_b200 import distributed as D
    g = 2 << 20
    for nnz in (1, 1000, 524288, 524289, 10**9 + 7):
        for world in (1, 2, 3, 8):
            e = D.element_shards(nnz, world, g)
            assert (4 * e) % g == 0 and (8 * e) % g == 0
            assert e * world >= nnz and (e - g // 4) * world < max(nnz, 1) + world * (g // 4)


def _fd_worker(rank, world, port, q):
    """exchange_fds on CPU: each rank shares a memfd holding its rank; every
    rank reads every peer's file through the received descriptor."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    from paper_1804_00695_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fd = os.memfd_create("shard%d" % rank)
        os.write(fd, ("rank-%d" % rank).encode())
        got = D.exchange_fds([fd], dist)
        seen = [os.pread(f[0], 16, 0).decode() for f in got]
        q.put((rank, seen))
    finally:
        dist.destroy_process_group()


def test_two_rank_fd_exchange():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fd_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, seen in res:
        assert seen == ["rank-%d" % r for r in range(world)]


def _mg_worker(rank, world, port, q, mode, scale):
    """One rank of the config-5 path on the product kernels: R-MAT built on
    the device, K0-flops row partition, B replicated (gloo all-gather) or
    sharded (VMM shards mapped into one VA, descriptors over Unix sockets),
    block multiply materialised and streamed, offset exchange."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from paper_1804_00695_b200 import _lib, distributed as D, generators as gen
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ctx = _lib.Context.get(0)
        da = gen.rmat_graph_device(scale).set_values(1.0)
        n = da.num_rows
        row_flops, total = _lib.d_row_flops(da, da)
        bounds = D.flops_partition(row_flops, world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        a_blk = da.slice_rows(lo, hi)
        if mode == "sharded":
            db, info = D.shard_b(ctx, da, dist)
        else:
            rp = np.empty(n + 1, dtype=np.int64)
            _lib.memcpy(ctx, rp.ctypes.data, da.device_ptrs()[0], rp.nbytes)
            sb = D.shard_bounds(np.diff(rp), world)
            db = D.replicate_b(ctx, da.slice_rows(int(sb[rank]), int(sb[rank + 1])), n, n, dist)
        c, st = D.mg_multiply(a_blk, db, 0, keep_c=True)
        _, st2 = D.mg_multiply(a_blk, db, 1 << 20, keep_c=False)   # streamed in small blocks
        off, tot = D.exchange_offsets(st["nnz"], dist)
        h = c.download()
        q.put((rank, lo, hi, off, tot, h.row_ptr.copy(), h.col_idx.copy(), h.values.copy(), st, st2,
               int(row_flops[lo:hi].sum()), bounds.tolist()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["replicated", "sharded"])
def test_two_process_config5_on_product_kernels(mode):
    """Two processes (gloo; both on GPU 0 -- their kernels never wait on each
    other) run the multi-GPU path end to end; the gathered blocks equal the
    oracle's A*A, the streamed-C statistics equal the materialised ones, and
    every block's value sum equals its multiplications."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_1804_00695_b200 import generators as gen
    from paper_1804_00695_b200.csr import CsrMatrix
    from oracle import oracle as O
    from conftest import assert_same_product
    world, scale = 2, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mg_worker, args=(r, world, port, q, mode, scale)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    a = gen.with_unit_values(gen.rmat_graph(scale))
    rp, cols, vals = [np.zeros(1, np.int64)], [], []
    for rank, lo, hi, off, tot, prp, pcol, pval, st, st2, mults, bounds in res:
        assert off == int(sum(x[9]["nnz"] for x in res[:rank]))
        assert tot == sum(x[8]["nnz"] for x in res)
        assert st["nnz"] == st2["nnz"] == len(pcol) and st2["blocks"] > 1
        assert st["value_sum"] == st2["value_sum"] == float(mults)
        rp.append(prp[1:] + rp[-1][-1])
        cols.append(pcol)
        vals.append(pval)
    got = CsrMatrix(a.num_rows, a.num_cols, np.concatenate(rp), np.concatenate(cols), np.concatenate(vals))
    assert_same_product(got, O.multiply(a, a, workers=os.cpu_count() or 1), exact=False, rtol=1e-12)
