"""Markdown summary of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launches_md.py LAUNCHES.csv "title" "command" > profiles/NAME.md"""
import csv
import re
import sys
from collections import OrderedDict

path, title, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
L = []
for r in rows:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^void ", "", r[ix["Kernel Name"]])
    name = re.sub(r"\(.*\)$", "", name)
    us = float(r[ix["Metric Value"]].replace(",", "")) / (1e3 if r[ix["Metric Unit"]] == "ns" else 1)
    L.append((name, r[ix["Grid Size"]], r[ix["Block Size"]], us))
per = OrderedDict()
for n, g, b, us in L:
    c, t = per.get(n, (0, 0.0))
    per[n] = (c + 1, t + us)
tot = sum(us for *_, us in L)
print(f"# {title}\n\nCommand: `{cmd}`; raw CSV alongside.  Times are ncu's serialised, cold-cache "
      "per-launch durations (never bench values).\n")
print(f"{len(L)} launches, {tot:,.1f} us in total.  Per kernel:\n")
print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
for n, (c, t) in per.items():
    print(f"| `{n}` | {c} | {t:,.1f} | {t / c:,.1f} | {100 * t / tot:.1f} % |")
print("\nFirst 16 launches (the main line: L2 flush fill, then ONE kernel launch per C4 fixpoint):\n")
print("| # | kernel | grid | block | us |\n|---|---|---|---|---|")
for i, (n, g, b, us) in enumerate(L[:16]):
    print(f"| {i} | `{n}` | {g} | {b} | {us:,.1f} |")
