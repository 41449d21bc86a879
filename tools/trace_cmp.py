#!/usr/bin/env python
"""Print the median phase stamps of tools/trace.py JSON lines side by side."""
import json
import sys

KEYS = ["after_pdl_wait", "prod_rowoff", "prod_struct_off", "p0_after_empty", "p0_after_tma", "p0_before_arrive",
        "p1_before_arrive", "cons_first_full", "cons_unit0_done", "prod_done", "cons_done", "exit"]
KEYS += [f"u{j}_{w}" for j in range(3) for w in ("empty_ok", "slice_issued", "tma_issued", "copies_issued")]
rows = []
for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            d = json.loads(line)
            last = d
    rows.append((path.split("/")[-1], last))
print("%-18s" % "slot (median us)" + "".join("%12s" % r[0][:11] for r in rows))
for k in KEYS:
    if all(k in r[1] for r in rows):
        print("%-18s" % k + "".join("%12.2f" % r[1][k][1] for r in rows))
print("%-18s" % "span" + "".join("%12.2f" % r[1]["span_us"] for r in rows))
