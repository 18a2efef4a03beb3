"""SF_TRACE build: globaltimer timeline of overlapped (PDL) windows -- when each scenario's
coordinator / instance advances / ledger start and end, relative to the window's first start."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12784_b200 import workload as W
from paper_2601_12784_b200.staleflow import StaleFlow
p = W.preset("C5")
n = len(p.scenarios)
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
g = StaleFlow.from_preset(p)
g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs))
f = g.L.sf_debug_trace
f.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
NI = 4 * n
buf = np.zeros(4 * n + 2 * NI, np.int64)
g.step(5)
for w in range(5, 5 + int(os.environ.get("NW", "12"))):
    flush.zero_(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.step(1); e.record(); torch.cuda.synchronize()
    f(g.h, buf.ctypes.data_as(C.POINTER(C.c_int64)))
    sc = buf[:4 * n].reshape(n, 4).astype(np.float64)
    ins = buf[4 * n:].reshape(NI, 2).astype(np.float64)
    t0 = sc[:, 0].min()
    sc = (sc - t0) / 1e3; ins = (ins - t0) / 1e3          # us
    cd = sc[:, 1] - sc[:, 0]
    adv = ins[:, 1] - ins[:, 0]
    last = int(np.argmax(sc[:, 3]))
    li = ins[4 * last:4 * last + 4]
    print(f"w{w} {s.elapsed_time(e)*1e3:6.0f}us | coord end p50 {np.median(sc[:,1]):5.0f} p99 {np.percentile(sc[:,1],99):5.0f} max {sc[:,1].max():5.0f} | "
          f"adv start p50 {np.median(ins[:,0]):5.0f} max {ins[:,0].max():5.0f} end max {ins[:,1].max():5.0f} dur p50 {np.median(adv):4.0f} max {adv.max():4.0f} | "
          f"ledger end max {sc[:,3].max():5.0f} | last scen {last}: coord {sc[last,0]:.0f}-{sc[last,1]:.0f} adv {li[:,0].min():.0f}-{li[:,1].max():.0f} led {sc[last,2]:.0f}-{sc[last,3]:.0f}")
