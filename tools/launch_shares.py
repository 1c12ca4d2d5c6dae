"""Per-generation kernel shares from an ncu launch list (run here, no GPU):

    python tools/launch_shares.py LAUNCHES.csv OUT.md "title"

The GA window runs from the first k_mates launch to the launch before the
dense roofline pass bench.py runs after its timed region (the first
k_resync_gm, or a k_fitness launch longer than 200 us); generations = the
k_breed2 / k_breed launches in it.  ncu serialises launches and runs them
cold-cache: compare shares, not absolute times."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
            name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "").strip()
            out.append((name, v))
    return out


def main():
    src, dst, title = sys.argv[1], sys.argv[2], sys.argv[3]
    ks = load(src)
    i0 = next(i for i, (n, _) in enumerate(ks) if n.startswith("k_mates"))
    i1 = len(ks)
    for i in range(i0, len(ks)):
        n, v = ks[i]
        if n.startswith("k_resync_gm") or (n == "k_fitness" and v > 200.0):
            i1 = i
            break
    win = ks[i0:i1]
    gens = sum(1 for n, _ in win if n.startswith("k_breed"))
    agg = defaultdict(float)
    for n, v in win:
        agg[n] += v
    tot = sum(agg.values())
    with open(dst, "w") as f:
        f.write("# %s\n\nRaw: `%s`.  GA window: %d generations (launches from the first k_mates to the "
                "dense roofline pass); ncu serialises launches and runs them cold-cache, so compare shares, "
                "not absolute times; the side-stream kernels (k_mates, k_mutmask, k_stats) overlap the main "
                "stream in a normal run.\n\n| kernel | per generation us | share of the serialised sum |\n"
                "|---|---|---|\n" % (title, src.split("/")[-1], gens))
        for n, v in sorted(agg.items(), key=lambda x: -x[1]):
            f.write("| %s | %.1f | %.1f%% |\n" % (n, v / gens, 100 * v / tot))
        f.write("| **sum** | %.1f | 100%% |\n" % (tot / gens))
    print(open(dst).read())


if __name__ == "__main__":
    main()
