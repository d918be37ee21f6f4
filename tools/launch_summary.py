#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel name, the
count and summed duration over the LAST `--evals` evaluations (split at the K1 generator)."""
import csv
import re
import sys
from collections import OrderedDict


def rows(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    for r in csv.DictReader(txt[i:].splitlines()):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            yield r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r.get("Metric Unit", "")


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"void |exageo::|\(anonymous namespace\)::", "", name)
    return name[:60]


def main():
    path = sys.argv[1]
    evals = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rs = list(rows(path))
    starts = [i for i, (n, _, _) in enumerate(rs) if "gen_panels" in n]
    sel = rs[starts[-evals]:] if starts else rs
    agg = OrderedDict()
    tot = 0.0
    for n, v, u in sel:
        us = v / 1000.0 if u == "nsecond" or u == "ns" else (v if u in ("usecond", "us") else v * 1000.0)
        a = agg.setdefault(short(n), [0, 0.0])
        a[0] += 1
        a[1] += us
        tot += us
    print(f"{path}: {len(sel)} launches, {tot:.1f} us summed (serialised)")
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:60s} {c:5d}  {us:10.1f} us  {100 * us / tot:5.1f}%")


if __name__ == "__main__":
    main()
