"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel name."""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
        name = name.split("<")[0] + ("<" + d["Kernel Name"].split("<")[1].split(">")[0] + ">"
                                     if "<" in d["Kernel Name"] else "")
        ns = float(d["Metric Value"].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'ms total':>9s} {'share':>7s}")
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:8d} {ns / 1e6:9.3f} {ns / tot * 100:6.1f}%")
    print(f"{'total':60s} {sum(v[0] for v in agg.values()):8d} {tot / 1e6:9.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
