"""Mutation check of the oracle's pins ("done when each of these mutations fails at
least one CPU test").

Each mutant is a one-site textual change to a copy of oracle/sf_oracle.cpp that a plausible mistake
in reading the paper would make.  The copy is compiled to a temporary library and the pin tests
(hand timelines T1/T3, Eq 1 gatekeeping, cascade pins, the exact-rational transcription diff, the
SPEC worked examples) are run against it in a subprocess (`SFO_ORACLE_LIB`, oracle/oracle.py).
Every mutant must make at least one of them fail; the unmodified oracle passes them (the normal run).
"""
import concurrent.futures as cf
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "sf_oracle.cpp")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_fraction.py", "tests/test_oracle_sim.py::test_T1_hand_timeline",
        "tests/test_oracle_cost_strategies.py", "tests/test_oracle_ledger.py"]

# name -> (exact text in sf_oracle.cpp, replacement, the reading it violates)
MUTANTS = {
    "preempt_fifo": ("int j = n.run.back();\n    n.run.pop_back();",
                     "int j = n.run.front();\n    n.run.erase(n.run.begin());", "B4 / A21 LIFO preemption"),
    "preempt_to_wait_back": ("n.wait.push_front(j);", "n.wait.push_back(j);", "B4 / A21 wait front"),
    "token_on_interrupt": ("if (it != n.run.end()) { n.kv -= (int64_t)P.k5 * jc.second; n.run.erase(it); continue; }",
                           "if (it != n.run.end()) { if (tick_end) s.traj[j].gen += 1; n.kv -= (int64_t)P.k5 * jc.second; "
                           "n.run.erase(it); continue; }", "B1 / A18 forfeited token"),
    "prefill_dropped": ("P.kp * prefill;", "0 * prefill;", "A20 prefill stall"),
    "cascade_latest_buffer": ("for (int bb = cu; bb < hb && !found; ++bb) {",
                              "for (int bb = hb - 1; bb >= cu && !found; --bb) {", "A13 earliest buffer"),
    "cascade_highest_slot": ("for (int ss = 0; ss < B; ++ss) {\n          const Entry &e = buf[bb][ss];\n"
                             "          if (e.st == E_RESERVED",
                             "for (int ss = B - 1; ss >= 0; --ss) {\n          const Entry &e = buf[bb][ss];\n"
                             "          if (e.st == E_RESERVED", "A13 lowest slot"),
    "reserve_lowest_slot": ("for (int s = B - 1; s >= 0; --s) {", "for (int s = 0; s < B; ++s) {", "P:364 / S:127 latest slot"),
    "eq1_not_enforced": ("if (!(quiescent && eq1)) valid = false;", "(void)eq1;", "Eq 1 / R-EQ1 gatekeeping"),
    "case1_wait_head": ("std::vector<int> victims(w.end() - case1_k[i], w.end());",
                        "std::vector<int> victims(w.begin(), w.begin() + case1_k[i]);", "A7 wait tail"),
    "case2_drain_imin": ("if (remaining > 0) case2 = imax;", "if (remaining > 0) case2 = imin;", "A8 drain imax"),
    "interrupt_ready_now": ("s.traj[j].ready = apply_time(i);", "s.traj[j].ready = t;", "A18 t_ready = apply time"),
}


def _build(name, text, repl, tmp):
    src = open(SRC).read()
    assert src.count(text) == 1, f"mutant {name}: anchor text not found exactly once in sf_oracle.cpp"
    path = os.path.join(tmp, f"{name}.cpp")
    with open(path, "w") as f:
        f.write(src.replace(text, repl))
    lib = os.path.join(tmp, f"lib_{name}.so")
    subprocess.run(["g++", "-std=c++17", "-O1", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                    "-I", os.path.join(ROOT, "oracle"), path, "-o", lib, "-lpthread"], check=True)
    return lib


def _run_pins(lib):
    env = dict(os.environ, SFO_ORACLE_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *PINS],
                       cwd=ROOT, env=env, capture_output=True, text=True)
    return r.returncode, r.stdout[-600:]


def test_every_mutant_fails_a_pin():
    with tempfile.TemporaryDirectory() as tmp:
        with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            libs = {n: ex.submit(_build, n, t, r, tmp) for n, (t, r, _) in MUTANTS.items()}
            results = {n: ex.submit(_run_pins, f.result()) for n, f in libs.items()}
            survivors = {n: f.result()[1] for n, f in results.items() if f.result()[0] == 0}
    assert not survivors, f"mutants not caught by any pin: {list(survivors)}"
