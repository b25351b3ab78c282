import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import golden_cases as G
import paper_2603_01915_b200 as P
rec = G.load('config1')
c = P.encode_matrix(G.matrix(rec), **G.encode_kwargs(rec))
out = P.spmv(c, rec["x"], rec["y"])
ref = rec["spmv"]
bad = np.nonzero(~((out == ref) | (np.isnan(out) & np.isnan(ref))))[0]
print("bad rows", len(bad), bad[:40], "slices", np.unique(bad // 32)[:20])
m = P.decode_matrix(c)
print("decode ok", np.array_equal(m.col_idx, G.matrix(rec).col_idx))
