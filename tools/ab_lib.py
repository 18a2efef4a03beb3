"""Same-box A/B of two library builds (SF_LIB paths given as argv): per-kernel serialized ms and
PDL window ms on the C5 bench windows, interleaved rounds to cancel drift."""
import os, subprocess, sys, json
libs = sys.argv[1:]
code = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2601_12784_b200 import workload as W
from paper_2601_12784_b200.staleflow import StaleFlow
p = W.preset("C5"); n = len(p.scenarios)
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = {}
for prof in (False, True):
    g = StaleFlow.from_preset(p); g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs))
    g.step(5); torch.cuda.synchronize()
    if prof: g.profile(True)
    tot = 0.0
    for _ in range(60):
        flush.zero_(); s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.step(1); e.record(); torch.cuda.synchronize(); tot += s.elapsed_time(e)
    if prof:
        ms, cnt = g.profile_read(); out["kern"] = (ms[:3] / np.maximum(cnt[:3], 1)).round(4).tolist()
    else:
        out["window"] = round(tot / 60, 4)
    g.close()
print(json.dumps(out))
'''
res = {l: [] for l in libs}
for r in range(int(os.environ.get("ROUNDS", "2"))):
    for l in libs:
        o = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SF_LIB=l), capture_output=True, text=True)
        res[l].append(json.loads(o.stdout.strip().splitlines()[-1]) if o.returncode == 0 else o.stderr[-300:])
for l in libs:
    print(os.path.basename(l), res[l])
