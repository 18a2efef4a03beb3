"""A second, independent transcription of SF-SIM-1 in plain Python with exact rationals.

TEST INFRASTRUCTURE ONLY (SURVEY §4 item 2, §8(c) "whole simulation" pin).  Written from
DESIGN.md §3 / SURVEY §8(c) (W0-W9, B1-B8, ledger §3.3), NOT from oracle/sf_oracle.cpp: it shares
no code with the oracle or the CUDA library and is used to diff the oracle on tiny configs.

Every cost-model comparison (Eq 2-4 waterfall P:640-670, Alg 2, Alg 4)
is evaluated with `fractions.Fraction`.  The oracle and the library evaluate the same comparisons
in fp64 (reading A3), so they can only disagree with this file where two compared quantities are
within rounding of each other: every such near-tie is recorded in `self.ambiguous` and a caller
discards that configuration.  Redundancy / filtering (f2) are not transcribed.
"""
from __future__ import annotations

from fractions import Fraction

POOL, TS, TRANSIT, WAIT, RUN, DONE, CONSUMED = range(7)
IDLE, TICK, PULL = range(3)
REL = Fraction(1, 10**9)             # near-tie band for the exact comparisons


class FracSim:
    def __init__(self, I, eta, G, B, k1, k2, k3, k4, k5, kp, M, mu, phi_tp, phi_wait, delta, r, q, R,
                 strategy, atw):
        self.I, self.eta, self.G, self.B = I, eta, G, B
        self.k = (k1, k2, k3, k4, k5, kp)
        self.M, self.mu, self.phi_tp, self.phi_wait = M, Fraction(mu), Fraction(phi_tp), phi_wait
        self.delta, self.r, self.q, self.R = delta, r, q, R
        self.sf_route, self.sf_sync, self.sf_mig = bool(strategy & 1), bool(strategy & 2), bool(strategy & 4)
        self.atw = atw
        self.prompt, self.target = [], []            # per group / per trajectory
        self.loc, self.gen, self.inst_of, self.nroutes, self.npre, self.nint = [], [], [], [], [], []
        self.tdone, self.ready, self.rewarded = [], [], []
        self.vg, self.nrew, self.cvbuf = [], [], []
        self.ingested = self.live = 0
        self.ps, self.t, self.window, self.busy, self.pub_at = 0, 0, 0, False, 0
        self.buf = {}                                 # ledger: V_buf -> list of [state, g, v]
        self.cu = 0
        self.rewards = []                             # (t_reward, traj)
        self.cmds, self.batches = [], []
        self.m = dict.fromkeys(["windows", "ticks", "iters", "tokens", "done", "routes", "ints", "pulls",
                                "preempt", "batches", "valid", "invalid", "viol", "pubs", "ingested",
                                "occupied", "reserves", "reloc"], 0)
        self.hist = [0] * 9
        self.ambiguous = []
        self.cov = dict.fromkeys(["forfeit", "tail", "drain", "held", "prefill"], 0)   # feature coverage
        self.inst = [dict(v=0, kv=0, run=[], wait=[], c=0, st=IDLE, nb=0, pu=0, pull=None, ints=[],
                          arr=[], pre=0, pv=0, acc=0, now=False) for _ in range(I)]

    # ------------------------------------------------------------------ inputs
    def submit(self, prompts, targets):
        for a, p in enumerate(prompts):
            self.prompt.append(int(p)); self.vg.append(-1); self.nrew.append(0); self.cvbuf.append(-1)
            for m in range(self.G):
                self.target.append(int(targets[a * self.G + m]))
                for lst, x in ((self.loc, POOL), (self.gen, 0), (self.inst_of, -1), (self.nroutes, 0),
                               (self.npre, 0), (self.nint, 0), (self.tdone, -1), (self.ready, 0),
                               (self.rewarded, False)):
                    lst.append(x)

    def ctx(self, j):
        return self.prompt[j // self.G] + self.gen[j]

    # ------------------------------------------------------------------ exact comparisons
    def cmp(self, a, b, what, same=False):
        """sign(a - b); records a near-tie unless both sides are the same expression on the same
        inputs (then fp64 rounds them identically too) or both are exactly 0 (the literal 0 of
        gamma = 0 or n = 0, or a difference of two equal rationals: fp64 gives 0.0 for those)."""
        if not same and (a or b) and abs(a - b) <= REL * max(abs(a), abs(b)):
            self.ambiguous.append((self.window, what))
        return (a > b) - (a < b)

    def T(self, n, kv):                                          # Eq 2
        k1, k2, k3, k4, _, _ = self.k
        return Fraction(0) if n == 0 else Fraction(n, k1 * kv + max(k2, k3 * n) + k4)

    def gamma(self, s, l):                                       # Eq 3 admission
        return s[1] + self.k[4] * l <= self.M and s[3] == 0

    def dT(self, s, l):                                          # Eq 3 marginal gain
        if not self.gamma(s, l):
            return Fraction(0)
        return self.T(s[2] + 1, s[1] + self.k[4] * l) - self.T(s[2], s[1])

    # ------------------------------------------------------------------ ledger (§4.2)
    def slots(self, b):
        return self.buf.setdefault(b, [[0, -1, -1] for _ in range(self.B)])

    def verify(self, v, led):
        return any(any(e[0] == 0 for e in led.get(b, [[0]])) for b in range(max(v, self.cu), v + self.eta + 1))

    def reserve(self, g, v, led):                                # latest buffer, highest slot
        for b in range(v + self.eta, max(v, self.cu) - 1, -1):
            row = led.setdefault(b, [[0, -1, -1] for _ in range(self.B)])
            for s in reversed(range(self.B)):
                if row[s][0] == 0:
                    row[s] = [1, g, v]
                    return True
        return False

    def complete_group(self, g):
        hb, hs = next((b, s) for b in sorted(self.buf) if b >= self.cu
                      for s in range(self.B) if self.buf[b][s][1] == g and self.buf[b][s][0])
        assert self.buf[hb][hs][0] == 1, "completed group not Reserved"
        self.buf[hb][hs] = [0, -1, -1]
        while True:                                              # cascade (A13)
            mv = next(((b, s) for b in range(self.cu, hb) for s in range(self.B)
                       if self.slots(b)[s][0] == 1 and self.slots(b)[s][2] + self.eta >= hb), None)
            if mv is None:
                break
            self.buf[hb][hs], self.buf[mv[0]][mv[1]] = self.buf[mv[0]][mv[1]], [0, -1, -1]
            hb, hs = mv
            self.m["reloc"] += 1
        b = self.cu
        while all(e[0] for e in self.slots(b)):
            b += 1
        s = next(s for s in range(self.B) if self.slots(b)[s][0] == 0)
        self.buf[b][s] = [2, g, self.vg[g]]
        assert self.vg[g] <= b <= self.vg[g] + self.eta
        self.m["occupied"] += 1

    # ------------------------------------------------------------------ routing (Alg 2) and sync (Alg 3)
    def route_pass(self, S, items, led, commit):
        """items: (traj, group version or -1, l) in MLQ order.  Returns [(traj, inst)]."""
        out, pass_v = [], {}
        for (j, v, l) in items:
            g = j // self.G
            v = pass_v.get(g, v)
            cand = [i for i in range(self.I) if (S[i][0] >= v if v >= 0 else self.verify(S[i][0], led))]
            if not cand:
                break
            if self.sf_route:
                k1, k2, k3, k4, k5, _ = self.k
                thr = self.mu * Fraction(1, k1 * k5 * l + max(k2, k3) + k4)        # Eq 4
                sel = None
                for ver in sorted({S[i][0] for i in cand}):
                    best, bi = None, None
                    for i in (i for i in cand if S[i][0] == ver):
                        d = self.dT(S[i], l)
                        if best is None or self.cmp(d, best, "dT", same=S[i][1:] == S[bi][1:]) > 0:
                            best, bi = d, i
                    if self.cmp(best, thr, "thr") >= 0:
                        sel = bi
                        break
                if sel is None:
                    break
            else:
                sel = min(cand, key=lambda i: (S[i][2] + S[i][3], i))
            if v < 0:
                v = pass_v[g] = S[sel][0]
                assert self.reserve(g, v, led)
                if commit:
                    self.vg[g] = v
                    self.m["reserves"] += 1
            if self.gamma(S[sel], l):
                S[sel] = (S[sel][0], S[sel][1] + self.k[4] * l, S[sel][2] + 1, S[sel][3])
            else:
                S[sel] = (S[sel][0], S[sel][1], S[sel][2], S[sel][3] + 1)
            out.append((j, sel))
        return out

    def mlq(self):
        res = [j for j in range(len(self.loc)) if self.loc[j] == TS]
        res.sort(key=lambda j: (self.vg[j // self.G] < 0, self.vg[j // self.G], j))
        return [(j, self.vg[j // self.G], self.ctx(j)) for j in res]

    def interrupt(self, i, victims, S):
        n = self.inst[i]
        for j in victims:
            self.cmds.append((self.window, 2, i, j))
            n["ints"].append((j, self.ctx(j)))
            self.loc[j] = TS
            self.ready[j] = n["nb"] if n["st"] == TICK else self.t
            self.nint[j] += 1
        self.m["ints"] += len(victims)
        n["acc"] -= len(victims)

    def coordinate(self):
        for j in range(len(self.loc)):
            if self.loc[j] == TS:
                self.ready[j] = self.t
        items = self.mlq()
        S = [(n["v"], n["kv"], len(n["run"]), len(n["wait"])) for n in self.inst]
        if self.sf_sync:                                         # Alg 3 (A16)
            chosen = []
            for i in range(self.I):
                if self.ps > S[i][0] and not any(
                        (S[i][0] >= v if v >= 0 else self.verify(S[i][0], self.buf)) for (_, v, _) in items):
                    tmp = list(S)
                    tmp[i] = (self.ps,) + S[i][1:]
                    scratch = {b: [list(e) for e in row] for b, row in self.buf.items()}
                    if any(x == i for (_, x) in self.route_pass(tmp, items, scratch, False)):
                        chosen.append(i)
        else:
            chosen = [i for i in range(self.I) if S[i][0] < self.ps]
        for i in chosen:
            n = self.inst[i]
            if n["run"] or n["wait"]:
                self.interrupt(i, n["run"] + n["wait"], S)
            self.cmds.append((self.window, 3, i, -1))
            n["pull"] = self.ps
            self.m["pulls"] += 1
            n["pv"], n["acc"] = self.ps, 0
            S[i] = (self.ps, 0, 0, 0)
        if self.sf_mig:                                          # Alg 4
            excess = [max(0, S[i][3] - self.phi_wait) for i in range(self.I)]
            Tm = [self.T(S[i][2], S[i][1]) for i in range(self.I)]
            hi = lo = 0
            for i in range(1, self.I):
                # T = n / L is one correctly rounded division: equal rationals give equal doubles
                if self.cmp(Tm[i], Tm[hi], "Tmax", same=Tm[i] == Tm[hi]) > 0:
                    hi = i
                if self.cmp(Tm[i], Tm[lo], "Tmin", same=Tm[i] == Tm[lo]) < 0:
                    lo = i
            drain = Tm[lo] > 0 and self.cmp(Tm[hi] / Tm[lo], self.phi_tp, "gap") > 0 \
                and S[hi][2] + S[hi][3] - excess[hi] > 0
            tails = {}
            for i in range(self.I):
                if excess[i]:
                    tails[i] = self.inst[i]["wait"][-excess[i]:]
                    self.cov["tail"] += 1
                    self.interrupt(i, tails[i], S)
                    S[i] = S[i][:3] + (S[i][3] - excess[i],)
            if drain:
                self.cov["drain"] += 1
                n = self.inst[hi]
                self.interrupt(hi, [j for j in n["run"] + n["wait"] if j not in tails.get(hi, [])], S)
                S[hi] = (S[hi][0], 0, 0, 0)
        for (j, i) in self.route_pass(S, self.mlq(), self.buf, True):
            self.cmds.append((self.window, 1, i, j))
            self.loc[j], self.inst_of[j] = TRANSIT, i
            self.nroutes[j] += 1
            self.inst[i]["arr"].append((self.ready[j] + self.r, j))
            self.inst[i]["acc"] += 1
            self.m["routes"] += 1

    # ------------------------------------------------------------------ boundary B1-B8
    def boundary(self, i, b):
        n = self.inst[i]
        k1, k2, k3, k4, k5, kp = self.k
        n["now"] = False
        ended, pulled = n["st"] == TICK and b == n["nb"], n["st"] == PULL and b == n["pu"]
        if n["st"] != PULL:
            for (j, c) in n["ints"]:                                             # B1
                if j in n["run"]:
                    n["run"].remove(j)
                    n["kv"] -= k5 * c
                    self.cov["forfeit"] += ended
                else:
                    n["wait"].remove(j)
            n["ints"] = []
        if ended:
            for j in n["run"]:                                                   # B2
                self.gen[j] += 1
                n["kv"] += k5
                self.m["tokens"] += 1
            for j in [j for j in n["run"] if self.gen[j] == self.target[j]]:    # B3
                n["run"].remove(j)
                n["kv"] -= k5 * self.ctx(j)
                n["c"] += 1
                self.loc[j], self.tdone[j] = DONE, b
                self.rewards.append((b + self.R, j))
                self.m["done"] += 1
            n["st"] = IDLE
        if pulled:
            n["v"], n["c"], n["st"] = n["pullv"], 0, IDLE
        while n["kv"] > self.M:                                                  # B4
            j = n["run"].pop()
            n["kv"] -= k5 * self.ctx(j)
            n["wait"].insert(0, j)
            self.loc[j] = WAIT
            self.npre[j] += 1
            self.m["preempt"] += 1
        if n["pull"] is not None:                                                # B5
            n["pullv"], n["pull"], n["st"], n["pu"] = n["pull"], None, PULL, b + self.q
            return
        due = sorted(a for a in n["arr"] if a[0] <= b)                           # B6
        n["arr"] = [a for a in n["arr"] if a[0] > b]
        self.cov["held"] += len(due) * pulled
        for (_, j) in due:
            n["wait"].append(j)
            self.loc[j] = WAIT
        while n["wait"] and n["kv"] + k5 * self.ctx(n["wait"][0]) <= self.M:     # B7
            j = n["wait"].pop(0)
            n["run"].append(j)
            n["kv"] += k5 * self.ctx(j)
            n["pre"] += self.ctx(j)
            self.loc[j] = RUN
        if n["run"]:                                                             # B8
            n["nb"] = b + k1 * n["kv"] + max(k2, k3 * len(n["run"])) + k4 + kp * n["pre"]
            self.cov["prefill"] += kp * n["pre"] > 0
            n["pre"], n["st"] = 0, TICK
            self.m["iters"] += len(n["run"])
            self.m["ticks"] += 1
        else:
            n["st"] = IDLE

    def next_b(self, n):
        if n["st"] == TICK:
            return n["nb"]
        if n["st"] == PULL:
            return n["pu"]
        return min([self.t] * n["now"] + [a[0] for a in n["arr"]], default=None)

    # ------------------------------------------------------------------ one window W0-W9
    def consume(self):
        row = self.slots(self.cu)
        self.batches.append(self.cu)
        for (_, g, v) in row:
            st = self.cu - v
            if not 0 <= st <= self.eta:
                self.m["viol"] += 1
            self.hist[min(max(st, 0), 8)] += 1
            self.cvbuf[g] = self.cu
            for j in range(g * self.G, (g + 1) * self.G):
                if self.rewarded[j]:
                    self.loc[j] = CONSUMED
            self.batches += [g, v]
        self.cu += 1
        self.live -= self.B
        self.m["batches"] += 1

    def window_step(self):
        t, t_end = self.t, self.t + self.delta
        if self.atw > 0:                                                         # W0 (A24)
            if self.busy and self.pub_at <= t:
                self.ps, self.busy = self.ps + 1, False
                self.m["pubs"] += 1
            if not self.busy and all(e[0] == 2 for e in self.slots(self.cu)):
                self.consume()
                self.busy, self.pub_at = True, t + self.atw * self.delta
        while self.live < (self.eta + 1) * self.B and self.ingested < len(self.prompt):   # W1
            for j in range(self.ingested * self.G, (self.ingested + 1) * self.G):
                self.loc[j] = TS
            self.ingested += 1
            self.live += 1
            self.m["ingested"] += 1
        ok = True                                                                # W2 (R-EQ1)
        for n in self.inst:
            quiet = not n["ints"] and n["pull"] is None and not n["arr"] and n["st"] != PULL
            eq1 = n["pv"] == n["v"] and n["acc"] == len(n["run"]) + len(n["wait"]) + n["c"]
            if quiet and not eq1:
                self.m["viol"] += 1
            ok = ok and quiet and eq1
        if ok:
            self.m["valid"] += 1
            self.coordinate()
        else:
            self.m["invalid"] += 1
        for n in self.inst:                                                      # W6
            if n["st"] == IDLE and (n["pull"] is not None or n["ints"]):
                n["now"] = True
        for i, n in enumerate(self.inst):                                        # W7
            while (b := self.next_b(n)) is not None and b <= t_end:
                self.boundary(i, b)
        self.rewards.sort()                                                      # W8
        for (tr, j) in [e for e in self.rewards if e[0] <= t_end]:
            g = j // self.G
            self.rewarded[j] = True
            self.nrew[g] += 1
            if self.nrew[g] == self.G:
                self.complete_group(g)
        self.rewards = [e for e in self.rewards if e[0] > t_end]
        self.t, self.window = t_end, self.window + 1                             # W9
        self.m["windows"] += 1

    # ------------------------------------------------------------------ observables (oracle layouts)
    def lifecycles(self):
        return [[j, j // self.G, self.prompt[j // self.G], self.target[j], self.gen[j], self.vg[j // self.G],
                 self.loc[j], self.inst_of[j], self.nroutes[j], self.npre[j], self.nint[j],
                 self.cvbuf[j // self.G], self.tdone[j]] for j in range(len(self.loc))]

    def instances(self):
        return [[n["v"], n["kv"], len(n["run"]), len(n["wait"]), n["c"], n["st"],
                 n["nb"] if n["st"] == TICK else (n["pu"] if n["st"] == PULL else -1)] for n in self.inst]

    def metrics(self):
        m = self.m
        return ([m["windows"], m["ticks"], m["iters"], m["tokens"], m["done"], m["routes"], m["ints"], m["pulls"],
                 m["preempt"], m["batches"], m["valid"], m["invalid"], m["viol"], m["pubs"], m["ingested"],
                 m["occupied"]] + self.hist + [None, self.t, m["reserves"], m["reloc"], 0, self.t, 0])
