"""Multi-GPU row partition of A.

Rows of C are independent (kernel.py:11-14), so N GPUs -- one process each --
compute contiguous blocks of C's rows.  The blocks are balanced by the K0
per-row multiplications (``flops_partition``: prefix + binary search, the
idea of chunking.py:80-128 applied to flops instead of bytes), which keeps
power-law rows (R-MAT hubs) from piling up on one GPU.  B reaches the GPUs in
one of the two ways §8e names:

* **replicated** -- every rank holds a row shard of B and one all-gather
  (row lengths, columns, values) rebuilds the full B on every rank
  (``allgather_csr`` / ``replicate_b``);
* **sharded** -- every rank keeps one element range of B's column and value
  arrays in its own HBM as a CUDA VMM allocation; the ranks swap the
  allocations' file descriptors once (``exchange_fds``, a Unix socket per
  rank) and every rank maps all shards back to back into one virtual range
  (``shard_b``), so the unchanged kernels read remote parts of B straight
  from peer HBM over NVLink.  No collective runs in the multiply.

Per step each rank multiplies its block (``tsg_mg_multiply``, optionally in
streamed-C mode for products whose C exceeds HBM) and the ranks exchange
their block sizes (``exchange_offsets``: all-gather of nnz, exclusive prefix
= the block's offset in the global row pointer).  Those two all-gathers are
the only collectives.  With NCCL they run on GPU tensors; with gloo (the CPU
tests, or two processes sharing one GPU) on host tensors.
"""

import os
import secrets
import socket
import threading
import time

import numpy as np


# ---------------------------------------------------------------- host logic

def flops_partition(row_flops, world: int) -> np.ndarray:
    """Boundaries b[0..world] (b[0]=0, b[world]=rows) of contiguous row blocks
    with near-equal flops; every block boundary is the first row whose flops
    prefix reaches k/world of the total."""
    f = np.asarray(row_flops, dtype=np.int64)
    n = int(f.shape[0])
    pre = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(f, out=pre[1:])
    total = int(pre[-1])
    b = np.zeros(world + 1, dtype=np.int64)
    for k in range(1, world):
        b[k] = int(np.searchsorted(pre, (total * k + world - 1) // world, side="left"))
    b[world] = n
    return np.maximum.accumulate(np.minimum(b, n))


def shard_bounds(row_nnz, world: int) -> np.ndarray:
    """Contiguous row shards of B with near-equal entry counts."""
    return flops_partition(row_nnz, world)


def element_shards(nnz: int, world: int, granularity: int) -> int:
    """Entries per shard of B's arrays: the smallest E >= nnz / world such
    that E int32 columns (and so E fp64 values) fill whole VMM granules."""
    per = max(1, granularity // 4)
    e = -(-max(int(nnz), 1) // world)
    return -(-e // per) * per


def _coll_device(dist):
    try:
        return "cuda" if dist.get_backend() == "nccl" else "cpu"
    except Exception:
        return "cpu"


# ---------------------------------------------------------------- collectives

def exchange_offsets(local_nnz: int, dist, device=None) -> "tuple[int, int]":
    """(offset of this rank's C block in the global C, global nnz)."""
    import torch
    device = device or _coll_device(dist)
    world = dist.get_world_size()
    t = torch.tensor([int(local_nnz)], dtype=torch.int64, device=device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    o = torch.cat(outs).cpu().numpy()
    r = dist.get_rank()
    return int(o[:r].sum()), int(o.sum())


def _allgather_var(x, dist, device):
    """All-gather of 1-D tensors of different lengths (padded to the max)."""
    import torch
    world = dist.get_world_size()
    n = torch.tensor([x.numel()], dtype=torch.int64, device=device)
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    lens = [int(v.item()) for v in ns]
    cap = max(lens) if lens else 0
    pad = torch.zeros(cap, dtype=x.dtype, device=device)
    pad[:x.numel()] = x.to(device)
    outs = [torch.empty(cap, dtype=x.dtype, device=device) for _ in range(world)]
    dist.all_gather(outs, pad)
    return torch.cat([o[:l] for o, l in zip(outs, lens)])


def allgather_csr(row_counts, cols, vals, dist, device):
    """Rebuild the full (row_ptr, cols, vals) of a matrix whose contiguous row
    shards live on the ranks (rank order = row order)."""
    import torch
    counts = _allgather_var(row_counts, dist, device)
    rp = torch.zeros(counts.numel() + 1, dtype=torch.int64, device=device)
    rp[1:] = torch.cumsum(counts, 0)
    return rp, _allgather_var(cols, dist, device), _allgather_var(vals, dist, device)


def exchange_fds(my_fds, dist):
    """Give every rank every other rank's file descriptors (CUDA VMM shard
    handles): each rank serves its descriptors on an abstract Unix socket
    (SCM_RIGHTS) and connects to every peer's.  Returns, in rank order, the
    list of descriptors valid in this process (this rank's own as given)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    token = [secrets.token_hex(8) if rank == 0 else None]
    dist.broadcast_object_list(token, src=0)
    name = lambda r: "\0tsg-%s-%d" % (token[0], r)
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(name(rank))
    srv.listen(world)

    def serve():
        for _ in range(world - 1):
            conn, _ = srv.accept()
            with conn:
                socket.send_fds(conn, [b"f"], list(my_fds))

    th = threading.Thread(target=serve, daemon=True)
    th.start()
    dist.barrier()
    out = []
    for r in range(world):
        if r == rank:
            out.append(list(my_fds))
            continue
        cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        for _ in range(200):
            try:
                cli.connect(name(r))
                break
            except (FileNotFoundError, ConnectionRefusedError):
                time.sleep(0.01)
        with cli:
            _, fds, _, _ = socket.recv_fds(cli, 16, len(my_fds))
        out.append(list(fds))
    th.join()
    srv.close()
    dist.barrier()
    return out


# ---------------------------------------------------------------- B on the ranks

def replicate_b(ctx, db_rows, b_rows: int, b_cols: int, dist):
    """B replicated: this rank holds B's rows as ``db_rows`` (a DeviceCsr of
    its row shard, global columns); one all-gather of (row lengths, int32
    columns, fp64 values) rebuilds the full B in this GPU's HBM."""
    import torch
    from . import _lib
    dev = _coll_device(dist)
    rp_p, col_p, val_p = db_rows.device_ptrs()
    n, nnz = db_rows.num_rows, db_rows.nnz
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    val = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
    _lib.memcpy(ctx, rp.data_ptr(), rp_p, 8 * (n + 1))
    _lib.memcpy(ctx, col.data_ptr(), col_p, 4 * nnz)
    _lib.memcpy(ctx, val.data_ptr(), val_p, 8 * nnz)
    rpf, colf, valf = allgather_csr(torch.diff(rp).to(dev), col[:nnz].to(dev), val[:nnz].to(dev), dist, dev)
    rpf, colf, valf = rpf.cuda(), colf.cuda(), valf.cuda()
    if rpf.numel() - 1 != b_rows:
        raise ValueError("gathered %d rows, expected %d" % (rpf.numel() - 1, b_rows))
    torch.cuda.synchronize()
    return _lib.DeviceCsr.from_device(ctx, b_rows, b_cols, int(colf.numel()), rpf.data_ptr(),
                                      colf.data_ptr(), valf.data_ptr())


def shard_b(ctx, db_full, dist, sorted_rows=True, max_row=-1):
    """B sharded in peer HBM.  Every rank exports one element range of B's
    columns and values as VMM physical allocations, the descriptors are
    exchanged once, and every rank maps all ranges back to back into one
    virtual range: a DeviceCsr view whose remote pages are read over NVLink.
    ``db_full`` (this rank's copy of B, from a deterministic builder) is only
    read for this rank's range and for the replicated row pointers; drop it
    afterwards.  Returns (view, info)."""
    import torch
    from . import _lib
    world, rank = dist.get_world_size(), dist.get_rank()
    gran = _lib.shard_granularity(ctx)
    nnz = db_full.nnz
    e = element_shards(nnz, world, gran)
    rp_p, col_p, val_p = db_full.device_ptrs()
    lo, hi = min(rank * e, nnz), min((rank + 1) * e, nnz)
    sc = _lib.Shard(ctx, 4 * e)
    sv = _lib.Shard(ctx, 8 * e)
    _lib.memcpy(ctx, sc.ptr, col_p + 4 * lo, 4 * (hi - lo))
    _lib.memcpy(ctx, sv.ptr, val_p + 8 * lo, 8 * (hi - lo))
    rp = torch.empty(db_full.num_rows + 1, dtype=torch.int64, device="cuda")
    _lib.memcpy(ctx, rp.data_ptr(), rp_p, 8 * (db_full.num_rows + 1))
    fds = exchange_fds([sc.fd, sv.fd], dist)
    vc = _lib.VMap(ctx, [f[0] for f in fds], [sc.size] * world)
    vv = _lib.VMap(ctx, [f[1] for f in fds], [sv.size] * world)
    for r, f in enumerate(fds):   # imported handles keep the memory; close our copies
        if r != rank:
            for x in f:
                os.close(x)
    view = _lib.d_csr_view(ctx, db_full.num_rows, db_full.num_cols, nnz, rp.data_ptr(), vc.va, vv.va,
                           sorted_rows, max_row, owners=(rp, vc, vv, sc, sv))
    dist.barrier()
    return view, {"entries_per_shard": e, "granularity": gran, "local_bytes": sc.size + sv.size,
                  "mapped_bytes": vc.total + vv.total}


# Config 2's slabs (bench.py --b-mode sharded at N>1): every rank owns the
# fine operator's rows of its z-slab; the B rows a rank's R selects (its slab
# plus a halo plane each side) are gathered by a kernel that reads the peers'
# slabs through CUDA IPC (tsg_gather_sharded).

def local_shard_tensors(b, lo: int, hi: int, device):
    """(rp, col, val) torch tensors of B's rows [lo, hi) on `device`, row
    pointers rebased to 0, int32 columns -- the layout tsg_gather_sharded reads."""
    import torch
    rp = np.asarray(b.row_ptr[lo:hi + 1], dtype=np.int64)
    e0, e1 = int(rp[0]), int(rp[-1])
    t_rp = torch.from_numpy(rp - e0).to(device)
    t_col = torch.from_numpy(np.asarray(b.col_idx[e0:e1], dtype=np.int32)).to(device)
    t_val = None if b.values is None else torch.from_numpy(np.array(b.values[e0:e1])).to(device)
    return t_rp, t_col, t_val


def share_shards(local, lo: int, hi: int, dist):
    """Exchange every rank's shard as CUDA IPC handles (torch's tensor
    reductions; opened with lazy peer access) and return, in rank order,
    [(row_lo, row_hi, rp, col, val)] tensors -- peers' live in peer HBM."""
    from torch.multiprocessing.reductions import reduce_tensor
    mine = (lo, hi) + tuple(None if t is None else reduce_tensor(t) for t in local)
    allp = [None] * dist.get_world_size()
    dist.all_gather_object(allp, mine)
    out = []
    for r, item in enumerate(allp):
        if r == dist.get_rank():
            out.append((lo, hi) + tuple(local))
            continue
        lo_r, hi_r = item[0], item[1]
        ts = tuple(None if red is None else red[0](*red[1]) for red in item[2:])
        out.append((lo_r, hi_r) + ts)
    return out


def gather_sharded(da, shards, b_cols: int):
    """Local CSR of B (the rows A selects) from shard tensors (local or peer)."""
    from . import _lib
    ptrs = [(lo, hi, rp.data_ptr(), col.data_ptr(), 0 if val is None else val.data_ptr())
            for lo, hi, rp, col, val in shards]
    return _lib.d_gather_sharded(da, ptrs, b_cols)


# ---------------------------------------------------------------- one rank's block

def mg_multiply(da_block, db, c_budget_bytes: int = 0, keep_c: bool = False):
    """This rank's block of C = A_block * B (C ABI ``tsg_mg_multiply``)."""
    from . import _lib
    return _lib.d_mg_multiply(da_block, db, c_budget_bytes, keep_c)


def rp_host(ctx, d):
    from . import _lib
    rp = np.empty(d.num_rows + 1, dtype=np.int64)
    rp_p, _, _ = d.device_ptrs()
    _lib.memcpy(ctx, rp.ctypes.data, rp_p, rp.nbytes)
    return rp
