"""SASS evidence for the kernels' instruction choices (run here, no GPU):
cuobjdump -sass of libpga.so, per kernel counts of the mnemonics that prove
the design -- UTMALDG (TMA tensor loads), HSETP2 / SEL / DADD (the pair
sweep's inner step), DMMA (fp64 tensor-core Gram), ATOMS (shared atomics),
SYNCS (mbarrier), and the totals.  Writes profiles/r02_sass_counts.json.

    python tools/sass_counts.py
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
LIB = os.path.join(ROOT, "paper_1403_4099_b200", "libpga.so")
OPS = ["UTMALDG", "UBLKCP", "HSETP2", "SEL", "DADD", "DFMA", "DMMA", "ATOMS", "ATOMG", "RED", "SYNCS",
       "SHFL", "MATCH", "LDS", "STS", "LDG", "STG", "LDSM", "MUFU", "BAR", "UCGABAR", "REDUX", "VOTE"]
KERNELS = ["k_fitness", "k_fitness_sparse", "k_breed2", "k_breed", "k_gram", "k_select_cluster",
           "k_select_small", "k_sus2", "k_qsum", "k_merge_level", "k_sort_runs", "k_stats", "k_batch",
           "k_pairtab", "k_clean", "k_ewma"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    res = {}
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            res[cur] = {"total": 0}
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(1)
            res[cur]["total"] += 1
            if op in OPS:
                res[cur][op] = res[cur].get(op, 0) + 1
    pretty = {}
    for mangled, cnt in res.items():
        dem = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
        name = dem.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        base = re.sub(r"<.*", "", name).split("::")[-1]
        if base in KERNELS:
            pretty[name] = cnt
    path = os.path.join(ROOT, "profiles", "r02_sass_counts.json")
    json.dump({"source": "cuobjdump -sass paper_1403_4099_b200/libpga.so (static instruction counts per "
                         "kernel, sm_100a)", "kernels": pretty}, open(path, "w"), indent=1, sort_keys=True)
    for k in sorted(pretty):
        c = pretty[k]
        print("%-45s %s" % (k[:45], " ".join("%s=%d" % (o, c[o]) for o in ["total"] + OPS if o in c)))


if __name__ == "__main__":
    sys.exit(main())
