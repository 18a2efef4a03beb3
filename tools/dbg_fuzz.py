"""Replay one GPU fuzz case window by window against the oracle; print state at the first divergence."""
import random, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import OracleSim
from tests.test_gpu_parity import _fuzz_config, gpu_from_config
seed = int(sys.argv[1])
rng = random.Random(seed)
I, eta, G, cfg, prompt, target, steps = _fuzz_config(rng)
print("I", I, "eta", eta, "G", G, "B", cfg.batch_size, "strategy", cfg.strategy)
o = OracleSim(I, eta, G, cfg)
g = gpu_from_config(I, eta, G, cfg)
o.submit(0, prompt, target); g.submit(0, prompt, target)
for w in range(120):
    io, ig = o.instances(0), g.instances(0)
    lo, lg = o.lifecycles(0), g.lifecycles(0)
    o.step(1); g.step(1)
    co, cg = o.commands(0), g.commands(0)
    if len(co) != len(cg) or not (co == cg).all():
        print("diverged in window", w)
        print("instances before (oracle):\n", io, "\n(gpu):\n", ig)
        n = min(len(co), len(cg))
        k = next((x for x in range(n) if not (co[x] == cg[x]).all()), n)
        print("oracle cmds", co[max(0, k - 6):k + 4].tolist())
        print("gpu cmds   ", cg[max(0, k - 6):k + 4].tolist())
        for j in range(8, 12):
            print("traj", j, "oracle", lo[j].tolist(), "\n        gpu   ", lg[j].tolist())
        ts = [r for r in lo if r[6] == 1]
        print("TS before (oracle): id g p T gen v", [(r[0], r[1], r[2], r[3], r[4], r[5]) for r in ts])
        print("metrics o", o.metrics(0)[:16].tolist(), "\nmetrics g", g.metrics(0)[:16].tolist())
        break
