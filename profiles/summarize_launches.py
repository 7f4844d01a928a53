"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and shares, as committed under profiles/:

    python profiles/summarize_launches.py gpurun_out/launches.csv "<command line>" > profiles/rNN/...
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hd = rows[h]
    ki, vi, mi, ui = (hd.index(k) for k in ("Kernel Name", "Metric Value", "Metric Name",
                                             "Metric Unit"))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[h + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
                  "msecond": 1.0}.get(r[ui], 1e-6)
            name = r[ki][:70]
            tot[name] += v
            cnt[name] += 1
    if len(sys.argv) > 2:
        print(f"# {sys.argv[2]}")
    print("# cold-cache, serialised per-launch times: compare shares, not absolutes")
    s = sum(tot.values()) or 1.0
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:72s} launches={cnt[k]:4d} total={v:10.3f} ms share={100 * v / s:5.1f}%")


if __name__ == "__main__":
    main()
