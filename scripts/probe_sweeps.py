"""Time one tile sweep per (mode, encoding) on a config (pipeline ceilings)."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_02736_b200 as g
from paper_2107_02736_b200 import _lib
import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
W = workloads.make(cfg)
ds = g.Dataset.from_array(W.X)
Q = np.ascontiguousarray(W.Q)
names = {0: "kde_gauss", 1: "kde_exp", 2: "tilemin", 3: "filter(none pass)", 4: "null"}
for enc in ([0] if ds.exact_mode else []) + [1, 2]:
    for mode in (4, 2, 3, 0):
        ms = ctypes.c_double()
        _lib.check(_lib.load().dk_sweep_probe(ds.handle, Q.ctypes.data, Q.shape[0], mode, enc, ctypes.byref(ms)))
        print(json.dumps({"config": cfg, "encoding": enc, "mode": names[mode], "ms": round(ms.value, 3)}), flush=True)
