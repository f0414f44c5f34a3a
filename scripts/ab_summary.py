"""Dev tool: one line per A/B run from lines `LABEL {sched_ab.py json}`:
LABEL  case:b2b_us/flushed_mean_us ...   (stdin or file arguments)."""
import fileinput
import json

for ln in fileinput.input():
    ln = ln.strip()
    if "{" not in ln or ln.startswith("[gpurun]"):
        continue
    k, js = ln.split(" ", 1)
    d = json.loads(js)
    print(k, " ".join(f"{c}:{v['b2b_us']}/{v.get('flushed_mean_us', v['flushed_us'])}"
                      for c, v in d.items() if c != "env"))
