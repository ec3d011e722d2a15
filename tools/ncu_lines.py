"""Per-source-line stall summary from `ncu --page source --print-source cuda,sass --csv`.

usage: zcat src.csv.gz | python tools/ncu_lines.py [top]
"""
import csv
import sys

top = int(sys.argv[1]) if len(sys.argv) > 1 else 45
r = csv.reader(sys.stdin)
f = None
hdr = None
rows = []
for row in r:
    if not row:
        continue
    if row[0] == "File Path":
        f = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if row[0]:
        def num(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        rows.append((f, int(row[0]), row[1], num(row[4]), num(row[7]), row))
tot = sum(x[3] for x in rows)
print("total samples", tot)
si = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
for fn, ln, src, s, e, row in sorted(rows, key=lambda x: -x[3])[:top]:
    st = sorted(((num(row[i]), hdr[i][6:]) for i in si), reverse=True)[:2]
    print(f"{s / tot * 100:5.1f}% {fn[:8]}:{ln:<5d} inst={e:9.3g} "
          f"{st[0][1]}={st[0][0] / max(s, 1) * 100:.0f}% {st[1][1]}={st[1][0] / max(s, 1) * 100:.0f}%"
          f" | {src.strip()[:70]}")
