"""Print the exact-KDE values of one fuzz trial next to the oracle's (developer tool)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import fuzz  # noqa: E402
import paper_2107_02736_b200 as g  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402

rng, kind, n, d, nq, X, Q, fam, h, scale = fuzz.gen(int(sys.argv[1]))
got = g.naive_kde(g.Dataset.from_array(X), g.KernelSpec(fam, h), Q).values
ref = O.naive_kde(O.Data(X), fam, h, Q)
rel = np.abs(got - ref) / np.maximum(ref, 1e-300)
for j in np.argsort(-rel)[:5]:
    print(f"q{j}: gpu {got[j]:.6e} oracle {ref[j]:.6e} rel {rel[j]:.2e}")
print("largest rel among oracle values >= 1e-30:", float(np.max(np.where(ref >= 1e-30, rel, 0.0))))
