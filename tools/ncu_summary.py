"""Summarise the ncu outputs of tools/profile_round.sh into profiles/ (run
here, no GPU needed):  python tools/ncu_summary.py <tag>"""
import csv, json, os, subprocess, sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)
gdir = os.path.join(ROOT, "gpurun_out")

# 1. launch list -> per-kernel shares
rows = list(csv.reader(open(os.path.join(gdir, "launches.csv"))))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = defaultdict(lambda: [0, 0.0])
for d in data:
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
    name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
lines = ["# ncu launch list (%s): `ncu --metrics gpu__time_duration.sum --clock-control none` of "
         "`python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e` (cold-cache, serialised: compare "
         "shares)" % tag, "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append("| %s | %d | %.1f | %.1f%% |" % (n[:70], c, v, 100 * v / tot))
open(os.path.join(out_dir, "%s_launches.md" % tag), "w").write("\n".join(lines) + "\n")
import shutil
shutil.copy(os.path.join(gdir, "launches.csv"), os.path.join(out_dir, "%s_launches.csv" % tag))

# 1b. F1 launch list (k_batch only)
f1csv = os.path.join(gdir, "launches_f1.csv")
if os.path.exists(f1csv):
    shutil.copy(f1csv, os.path.join(out_dir, "%s_launches_f1.csv" % tag))

# 2. full-set metrics of the captured kernels
kern_rows = []
hdr = units = None
for repname in ("prof_full.ncu-rep", "prof_sparse.ncu-rep", "prof_f1.ncu-rep"):
    rep = os.path.join(gdir, repname)
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    for r in rows[2:]:
        kern_rows.append((h, rows[1], r))
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum", "sm__cycles_active.avg",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second"]
traffic = {}
md = ["# ncu --set full (%s)" % tag, ""]
for hdr, units, d in kern_rows:
    name = d[hdr.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")
    md += ["## %s" % name, "", "| metric | value | unit |", "|---|---|---|"]
    vals = {}
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            md.append("| %s | %s | %s |" % (k, d[i], units[i]))
            vals[k] = (d[i], units[i])
    st = [(hdr[i], d[i]) for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled")
          and not hdr[i].endswith("not_issued")]
    st = sorted([(a.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(b.replace(",", "")))
                 for a, b in st if b not in ("", "n/a")], key=lambda x: -x[1])
    md += ["", "stall samples: " + ", ".join("%s=%d" % (a, b) for a, b in st[:8]), ""]
    def tobytes(v):
        x, u = float(v[0].replace(",", "")), v[1]
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    if "dram__bytes_read.sum" in vals:
        traffic[name] = {"dram_bytes_per_launch": tobytes(vals["dram__bytes_read.sum"]) +
                         tobytes(vals["dram__bytes_write.sum"]),
                         "source": "profiles/%s_full.md (ncu --set full, one launch)" % tag}
        if "smsp__inst_executed.sum" in vals:
            traffic[name]["inst_per_launch"] = float(vals["smsp__inst_executed.sum"][0].replace(",", ""))
open(os.path.join(out_dir, "%s_full.md" % tag), "w").write("\n".join(md) + "\n")
if "k_fitness" in traffic:
    traffic["k_sweep"] = traffic["k_fitness"]      # bench.py key (sweep + fused fold kernel)
json.dump(traffic, open(os.path.join(out_dir, "traffic.json"), "w"), indent=1)
print(open(os.path.join(out_dir, "%s_launches.md" % tag)).read())
print(json.dumps(traffic, indent=1))
