"""Multi-GPU row partition of A.

Rows of C are independent (kernel.py:11-14), so N GPUs each compute a
contiguous block of C's rows.  B reaches the ranks in one of two ways:

* replicated -- one all-gather rebuilds the full B on every rank
  (``allgather_csr``);
* sharded -- every rank keeps only its row shard of B; shards are shared as
  CUDA IPC handles once (``share_shards``), and each rank's kernel
  (``gather_sharded``, csrc ``tsg_gather_sharded``) loads the B rows its A
  rows select straight from peer HBM over NVLink.  No collective runs in the
  multiply.

The collectives, over torch.distributed (NCCL on B200s, gloo in the CPU
tests):

* ``allgather_csr`` -- B replicated: every rank holds a row shard of B and one
  all-gather (counts, columns, values) rebuilds the full B on every rank;
* ``exchange_offsets`` -- the row-pointer offset exchange: an all-gather of
  each rank's nnz(C slice) whose exclusive prefix places the slice in the
  global C.

``flops_partition`` balances the row blocks by the K0 per-row flops
(prefix + binary search, the same idea as chunking.py:80-128 over flops
instead of bytes), which is what keeps power-law rows (R-MAT) from piling up
on one rank.  All helpers are device-agnostic torch code.
"""

import numpy as np


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


def exchange_offsets(local_nnz: int, dist, device) -> "tuple[int, int]":
    """(offset of this rank's C slice in the global C, global nnz)."""
    import torch
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
    pad[:x.numel()] = x
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


def shard_bounds(row_nnz, world: int) -> np.ndarray:
    """Contiguous row shards of B with near-equal entry counts."""
    return flops_partition(row_nnz, world)


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
