import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from paper_1411_1994_b200 import api
from test_sharded_gpu import _run_ranks, _sharded_geometry
g = _sharded_geometry()
ctx = api.Context(0)
ref = api.reference_for(g, ctx); can = api.lattice_sum(ref, g)
t1, rep1 = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
print("single", rep1.chosen_ranks, rep1.deflated, rep1.deflate_k1, rep1.gram_rows, rep1.gram_size)
print(rep1.singular_values[0][:5], rep1.singular_values[0][75:85])
out = _run_ranks(g, 2)
for c, cn, t, rep in out:
    print("rank", rep.chosen_ranks, rep.deflated, rep.deflate_k1, rep.gram_rows, rep.gram_size)
    print(rep.singular_values[0][:5], rep.singular_values[0][75:85])
