"""Summarise an ncu --page source --csv dump: stall reasons and top instructions."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = collections.Counter()
per = []
for r in rows[2:]:
    if len(r) <= max(cols):
        continue
    d = {h[i]: int(r[i]) if r[i].isdigit() else 0 for i in cols}
    tot.update(d)
    per.append((sum(d.values()), r[0][-5:], r[1].strip()[:70], max(d, key=d.get) if any(d.values()) else ""))
s = sum(tot.values())
print("total", s)
for k, v in tot.most_common(12):
    print(f"  {k:28s} {v:7d} {100 * v / s:5.1f}%")
for x in sorted(per, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{x[0]:6d} {x[1]} {x[3]:24s} {x[2]}")
