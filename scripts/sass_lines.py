"""Instruction count per source line for one kernel (nvdisasm -g output)."""
import re, sys, collections
fn = sys.argv[2]
cnt = collections.Counter(); cur = None; infn = False
for line in open(sys.argv[1]):
    if '.section' in line and '.text.' in line:
        infn = fn in line
        continue
    if not infn: continue
    m = re.search(r'line (\d+)', line); mf = re.search(r'File "([^"]+)"', line)
    if m and '//##' in line:
        cur = ((mf.group(1).split('/')[-1] if mf else '?'), int(m.group(1))); continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/', line) and cur:
        cnt[cur] += 1
print('total', sum(cnt.values()))
for (f, l), c in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25): print(c, f, l)
