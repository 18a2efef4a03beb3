"""SF_CHECK build: ledger ring of scenario 0 after each window of a redundancy fuzz case, for two
launch modes compared side by side (argv: seed, windows)."""
import ctypes as C, os, random, subprocess, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import ctypes as C, random, sys, json, numpy as np
sys.path.insert(0, ".")
from tests.test_gpu_redundancy import pair
seed, W = int(sys.argv[1]), int(sys.argv[2])
rng = random.Random(7000 + seed)
B, G = rng.randint(1, 5), rng.randint(1, 4)
eb, em, eta = rng.randint(0, 2), rng.randint(0, 2), rng.randint(0, 3)
if eb == em == 0: eb = 1
I = rng.randint(1, 3); M = rng.choice([200, 500, 1 << 20]); q = 30 if seed < 20 else 1500; strat = rng.randint(0, 7)
o, g = pair(I, eta, G, B, eb, em, seed=seed, M=M, q=q, strategy=strat)
f = g.L.sf_debug_ledger; f.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int64)]
buf = np.zeros(4096, np.int64)
rows = []
for w in range(W):
    g.step(1)
    f(g.h, 0, buf.ctypes.data_as(C.POINTER(C.c_int64)))
    rows.append(buf[: 3 * (eta + 1) * (B + eb) + 2 * (eta + 1) + 1].tolist() + [int(x) for x in g.metrics(0)[[4, 15, 28, 29, 31]]])
print(json.dumps({"B": B + eb, "eta": eta, "rows": rows}))
'''
seed, W = sys.argv[1], sys.argv[2]
res = {}
for mode in ("", "SF_PDL=0"):
    env = dict(os.environ)
    if mode: env["SF_PDL"] = "0"
    out = subprocess.run([sys.executable, "-c", code, seed, W], env=env, capture_output=True, text=True)
    res[mode] = json.loads(out.stdout.strip().splitlines()[-1])
a, b = res[""], res["SF_PDL=0"]
Bt, eta = a["B"], a["eta"]
for w, (ra, rb) in enumerate(zip(a["rows"], b["rows"])):
    mark = "" if ra == rb else "  <-- differs"
    def fmt(r):
        slots = [(r[3 * i], r[3 * i + 1], r[3 * i + 2]) for i in range(Bt * (eta + 1))]
        return " ".join(f"{'.RO'[st]}{gg}v{vv}" if st else "." for st, gg, vv in slots) + f" | cnt {r[3*Bt*(eta+1):-6]} cu {r[-6]} | comp,occ,reloc,err,ab {r[-5:]}"
    print(f"w{w} PDL  {fmt(ra)}{mark}")
    if ra != rb: print(f"w{w} SER  {fmt(rb)}")
