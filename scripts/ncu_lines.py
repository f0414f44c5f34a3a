"""Aggregate warp-stall samples per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass`."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
func = None; hdr = None; data = defaultdict(lambda: defaultdict(float)); src = {}
cur_line = None
for r in rows:
    if not r: continue
    if r[0] == 'Function Name': func = r[1][:60]; continue
    if r[0] == 'Line No': hdr = r; ci = {h: i for i, h in enumerate(r)}; continue
    if hdr is None or len(r) < 5: continue
    if r[0]:
        cur_line = int(r[0]); src[(func, cur_line)] = r[1]
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    data[func][cur_line] += s
for f, d in data.items():
    tot = sum(d.values()) or 1
    print('==', f, 'samples', tot)
    for ln, s in sorted(d.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
        print(f"{s/tot:6.1%} L{ln:4d} {src.get((f, ln), '')[:100].strip()}")
