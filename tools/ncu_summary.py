"""Summarise an `ncu --csv` metrics dump: mean of every metric per kernel name."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = collections.defaultdict(lambda: collections.defaultdict(list))
    units = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        data[name][d["Metric Name"]].append(v)
        units[d["Metric Name"]] = d.get("Metric Unit", "")
    for name, mets in data.items():
        print(name)
        for m, vs in sorted(mets.items()):
            print(f"   {m:60s} {sum(vs) / len(vs):14.4g} {units[m]}  (n={len(vs)})")


if __name__ == "__main__":
    main(sys.argv[1])
