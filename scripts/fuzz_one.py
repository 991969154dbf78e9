"""Re-run one k-NN query of a fuzz trial against a direct-difference fp64 ranking (developer tool).

    python scripts/fuzz_one.py SEED QUERY
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import fuzz  # noqa: E402
import paper_2107_02736_b200 as g  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402

seed, qj = int(sys.argv[1]), int(sys.argv[2])
rng, kind, n, d, nq, X, Q, fam, h, scale = fuzz.gen(seed)
if float(n) * nq * d >= 3e10:  # keep the generator in step with fuzz.trial (its subset draw)
    rng.choice(nq, size=64, replace=False)
k = int(min(n, rng.choice([1, 5, 50, 100, 257])))
ds = g.Dataset.from_array(X)
gi, gd = g.knn_batch(ds, Q, k)
ri, rd = O.brute_force_knn(O.Data(X), Q[qj], k)
diff = X.astype(np.float64) - Q[qj]
dd = np.einsum("ij,ij->i", diff, diff)
order = np.lexsort((np.arange(n), dd))[:k]
print("kind", kind, "n", n, "d", d, "k", k)
print("gpu    ", gi[qj], gd[qj])
print("direct ", order, dd[order])
print("oracle ", ri, rd)
print("gpu == direct-difference ranking:", np.array_equal(gi[qj], order))
