"""Debug helper: config-2 shaped R*A and RA*P at a small grid, step by step."""
import sys
import paper_1804_00695_b200 as tsg
from paper_1804_00695_b200 import generators as gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
a = gen.stencil(gen.BRICK3D, (n, n, n))
p, r = gen.aggregation((n, n, n))
print("RA", flush=True)
ra = tsg.multiply(r, a)
print("RA ok", ra.nnz, flush=True)
rap = tsg.multiply(ra, p)
print("RAP ok", rap.nnz, flush=True)
