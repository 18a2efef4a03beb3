"""Replay one redundancy fuzz case against the oracle, window by window; dump at divergence."""
import random, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_redundancy import pair
seed = int(sys.argv[1])
rng = random.Random(7000 + seed)
B, G = rng.randint(1, 5), rng.randint(1, 4)
eb, em, eta = rng.randint(0, 2), rng.randint(0, 2), rng.randint(0, 3)
if eb == em == 0:
    eb = 1
I = rng.randint(1, 3)
M = rng.choice([200, 500, 1 << 20])
q = 30 if seed < 20 else 1500
strat = rng.randint(0, 7)
print("B", B, "G", G, "eb", eb, "em", em, "eta", eta, "I", I, "M", M, "strategy", strat)
o, g = pair(I, eta, G, B, eb, em, seed=seed, M=M, q=q, strategy=strat)
for w in range(40):
    lo_prev, lg_prev = o.lifecycles(0), g.lifecycles(0)
    o.step(1); g.step(1)
    mo, mg = o.metrics(0), g.metrics(0)
    if not (mo == mg).all():
        print("diverged in window", w, [(k, int(mo[k]), int(mg[k])) for k in range(32) if mo[k] != mg[k]])
        lo, lg = o.lifecycles(0), g.lifecycles(0)
        for j in np.nonzero((lo != lg).any(1))[0][:10]:
            print(" traj", j, "oracle", lo[j].tolist(), "\n       gpu   ", lg[j].tolist())
        print(" before: oracle states", np.bincount(lo_prev[:, 6], minlength=9).tolist(), "gpu", np.bincount(lg_prev[:, 6], minlength=9).tolist())
        print(" batches o", o.batches(0).tolist(), "g", g.batches(0).tolist())
        co, cg = o.commands(0), g.commands(0)
        print(" last cmds o", co[-6:].tolist(), "\n           g", cg[-6:].tolist())
        break
else:
    print("no divergence in 40 windows")
