"""Per-launch sequence from an ncu --csv launch list (gpu__time_duration.sum and
launch__grid_size): prints the launches whose name matches REGEX, in order, with
their grid size -- to tell apart the passes of one kernel.

    python tools/ncu_sequence.py <launches.csv> [regex] [first] [count]
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
rx = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
first = int(sys.argv[3]) if len(sys.argv) > 3 else 0
count = int(sys.argv[4]) if len(sys.argv) > 4 else 60
launch = {}
order = []
for r in rows[hi + 1:]:
    d = dict(zip(hdr, r))
    key = d.get("ID")
    if key not in launch:
        launch[key] = {"name": re.sub(r"^.*::", "", d["Kernel Name"].split("(")[0]), "grid": d.get("Grid Size", "")}
        order.append(key)
    launch[key][d["Metric Name"]] = d["Metric Value"]
sel = [launch[k] for k in order if rx is None or rx.search(launch[k]["name"])]
for L in sel[first:first + count]:
    print(f"{L['name']:36s} grid={L.get('launch__grid_size', L['grid']):>8s} t={L.get('gpu__time_duration.sum', '?'):>12s}")
