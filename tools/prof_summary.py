"""Summarise gpurun_out/prof (tools/profile_round.sh) into profiles/<round>/: the launch list
summary, ncu_kernels.json (per window kernel: DRAM bytes per launch, instructions, issue-slot and
occupancy figures -- read by bench.py for roofline.traffic and the issue-slot roofline), the
details pages and the hottest source lines."""
import collections, csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "gpurun_out", "prof")
dst = os.path.join(ROOT, "profiles", sys.argv[1] if len(sys.argv) > 1 else "r02")
os.makedirs(dst, exist_ok=True)

# launch list -> per-kernel totals over the timed steps of the command
lines = [l for l in open(os.path.join(src, "launches.csv")) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    t = tot.setdefault(name, [0, 0.0])
    t[0] += 1
    t[1] += float(r[vi]) / 1e3
win = {k: v for k, v in tot.items() if any(x in k for x in ("k_begin_coord", "k_advance", "k_ledger"))}
s = sum(v[1] for v in win.values()) or 1.0
with open(os.path.join(dst, "launch_summary.csv"), "w") as f:
    f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none, cold-cache serialised)\n")
    f.write("# command: python bench.py --profile-run --steps 1 --warmup 0 --windows 300 --no-extra (C5, 4096 scenarios; incl. the replay context)\n")
    f.write("kernel,launches,total_us,avg_us,share_of_window_kernels\n")
    for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{k},{n},{us:.1f},{us / n:.1f},{(us / s if k in win else 0):.3f}\n")

# full capture -> key metrics per kernel
raw = list(csv.reader(open(os.path.join(src, "full_raw.csv"))))
hdr, units = raw[0], raw[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__average_warp_latency_per_inst_issued.ratio",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__occupancy_limit_registers",
        "smsp__warps_eligible.avg.per_cycle_active", "sm__cycles_elapsed.avg"]
out = {}
kn = hdr.index("Kernel Name")


def val(r, name):
    i = hdr.index(name)
    x = float(r[i].replace(",", ""))
    u = units[i]
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)


for r in raw[2:]:
    name = r[kn].split("(")[0].split()[-1].split("<")[0].split("::")[-1]
    d = {w: f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip() for w in want if w in hdr}
    d["dram_bytes_per_launch"] = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    if "smsp__issue_active.avg.pct_of_peak_sustained_active" in hdr:
        d["issue_active_frac"] = val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100.0
    if "sm__warps_active.avg.pct_of_peak_sustained_active" in hdr:
        d["achieved_occupancy"] = val(r, "sm__warps_active.avg.pct_of_peak_sustained_active") / 100.0
    if "smsp__warps_eligible.avg.per_cycle_active" in hdr:
        d["eligible_warps_per_sched"] = val(r, "smsp__warps_eligible.avg.per_cycle_active")
    # stall breakdown: warp cycles per issued instruction spent in each stall reason (the CPI stack)
    st = {}
    for i, hname in enumerate(hdr):
        if hname.startswith("smsp__average_warps_issue_stalled_") and hname.endswith("_per_issue_active.ratio"):
            try:
                st[hname[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
            except ValueError:
                pass
    d["stall_cycles_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:10])
    out[name] = d
json.dump({"source": "ncu --set full, window 181 of the C5 workload (tools/profile_round.sh)", "kernels": out},
          open(os.path.join(dst, "ncu_kernels.json"), "w"), indent=1)
traffic = {k: v["dram_bytes_per_launch"] for k, v in out.items()}

# details page per kernel + hot source lines
det = list(csv.reader(open(os.path.join(src, "full_details.csv"))))
dh = det[0]
for name in out:
    with open(os.path.join(dst, f"{name}_details.txt"), "w") as f:
        for r in det[1:]:
            if r[dh.index("Kernel Name")].split("(")[0].split()[-1].split("<")[0].split("::")[-1] == name:
                f.write(f"{r[dh.index('Section Name')]:<40} {r[dh.index('Metric Name')]:<50} {r[dh.index('Metric Unit')]:<12} {r[dh.index('Metric Value')]}\n")
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), os.path.join(src, "full_src.csv"), "40"],
               stdout=open(os.path.join(dst, "window_kernels_lines.txt"), "w"))
print(open(os.path.join(dst, "launch_summary.csv")).read())
print(json.dumps(traffic, indent=1))
