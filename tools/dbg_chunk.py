import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import numpy as np
from conftest import gcsr, golden
from paper_1804_00695_b200 import chunking as ch
from paper_1804_00695_b200.memory import MemoryModel, MemorySpaceSpec
from oracle import oracle as O
m = MemoryModel(MemorySpaceSpec("fast", 1 << 40, 100e9, 1e-7), MemorySpaceSpec("slow", None, 10e9, 1e-6))
a, b = gcsr("chunk/a"), gcsr("chunk/b")
print(a, b, a.col_idx.max(), b.col_idx.max())
counts = O.symbolic(a, O.compress(b))
p_ac = ch.singleton_partition(a.row_byte_sizes() + ch.c_row_byte_sizes(a.num_rows, counts))
p_b = ch.singleton_partition(b.row_byte_sizes())
for name, pa, pb in (("single", p_ac, p_b),):
    try:
        c, led = ch.gpu_chunk_multiply_1(a, b, counts, pa, pb, m)
        print(name, "ok", c.nnz)
    except Exception as e:
        print(name, "ERR", e)
info = golden()[1]["chunk"]
p_ac = ch.RowPartition([ch.RowRange(x, y) for x, y in info["p_ac"]["ranges"]], info["p_ac"]["range_bytes"], a.num_rows)
p_b = ch.RowPartition([ch.RowRange(x, y) for x, y in info["p_b"]["ranges"]], info["p_b"]["range_bytes"], b.num_rows)
print(info["p_ac"]["ranges"], info["p_b"]["ranges"])
for fn in (ch.gpu_chunk_multiply_1, ch.gpu_chunk_multiply_2):
    try:
        c, led = fn(a, b, counts, p_ac, p_b, m)
        print(fn.__name__, "ok", c.nnz)
    except Exception as e:
        print(fn.__name__, "ERR", e)
