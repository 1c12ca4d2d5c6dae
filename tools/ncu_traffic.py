"""Record per-launch ncu numbers of a capture in profiles/traffic.json, keyed
by kernel and bench configuration, so bench.py's roofline `traffic` and
issue-rate figures come from a capture of the SAME launch window it times.

    python tools/ncu_traffic.py REP.ncu-rep CONFIG_KEY "source description" [summary.md]

CONFIG_KEY e.g. C4_w1 (config, ranks).  Every kernel in the report gets
{inst_per_launch, dram_bytes_per_launch, time_us, issue_active_pct,
warps_active, smem_wavefronts, smem_excess_wavefronts}; several launches of
one kernel are averaged.  With a 4th argument a markdown summary is written.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
METRICS = {
    "gpu__time_duration.sum": "time_us",
    "smsp__inst_executed.sum": "inst_per_launch",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_excess_wavefronts",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
UNIT = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
        "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0, "GHz": 1e9, "MHz": 1e6}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"]
        # kernel name without namespace, "void " and template arguments
        # (bench.py looks kernels up by their plain names)
        name = name.split("(")[0].replace("<unnamed>::", "").replace("void ", "").strip()
        name = name.split("<")[0]
        rec = {}
        for m, k in METRICS.items():
            if m not in d or d[m] in ("", "n/a"):
                continue
            v = float(d[m].replace(",", ""))
            v *= UNIT.get(u.get(m, ""), 1.0)
            rec[k] = v
        res.setdefault(name, []).append(rec)
    agg = {}
    for name, recs in res.items():
        a = {k: sum(r.get(k, 0.0) for r in recs) / len(recs) for k in recs[0]}
        a["dram_bytes_per_launch"] = a.pop("dram_read", 0.0) + a.pop("dram_write", 0.0)
        a["launches_captured"] = len(recs)
        agg[name] = a
    return agg


def main():
    rep, key, src = sys.argv[1], sys.argv[2], sys.argv[3]
    md = sys.argv[4] if len(sys.argv) > 4 else None
    agg = read(rep)
    path = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(path)) if os.path.exists(path) else {}
    for name, a in agg.items():
        ent = tj.setdefault(name, {})
        ent[key] = dict(a, source=src)
    json.dump(tj, open(path, "w"), indent=1)
    if md:
        with open(md, "w") as f:
            f.write("# ncu capture: %s\n\n%s\n\n" % (os.path.basename(rep), src))
            f.write("| kernel | time us | warp-inst | DRAM MB | issue active % | warps active | smem wavefronts "
                    "| excess | regs |\n|---|---|---|---|---|---|---|---|---|\n")
            for name, a in agg.items():
                f.write("| %s | %.1f | %.4g | %.2f | %.1f | %.1f | %.4g | %.4g | %d |\n" % (
                    name, a.get("time_us", 0), a.get("inst_per_launch", 0), a["dram_bytes_per_launch"] / 1e6,
                    a.get("issue_active_pct", 0), a.get("warps_active", 0), a.get("smem_wavefronts", 0),
                    a.get("smem_excess_wavefronts", 0), a.get("registers", 0)))
    print(json.dumps(agg, indent=1))


if __name__ == "__main__":
    main()
