"""Top stall lines from `ncu -i rep --page source --csv -k regex:<k>` output."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
# there may be several kernels; split on the 'Kernel Name' marker
blocks, cur = [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = {'name': r[1], 'rows': []}; blocks.append(cur); continue
    if cur is not None: cur['rows'].append(r)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for b in blocks:
    hdr = b['rows'][0]; ci = {h: i for i, h in enumerate(hdr)}
    k = ci['Warp Stall Sampling (All Samples)']
    data = []
    for r in b['rows'][1:]:
        if len(r) > k and r[k]:
            data.append((float(r[k]), r[ci['Address']] if 'Address' in ci else '', r[ci['Source']][:110]))
    tot = sum(d[0] for d in data) or 1
    data.sort(reverse=True)
    print('==', b['name'][:80], 'total samples', tot)
    for d in data[:n]: print(f"{d[0]/tot:6.1%} {d[1]:>8} {d[2]}")
