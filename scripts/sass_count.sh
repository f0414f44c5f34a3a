#!/bin/sh
# SASS instruction count per kernel of the built library (code-size check)
cuobjdump -sass "${1:-paper_2604_16883_b200/_lib/libsinkr_cuda.so}" 2>/dev/null |
  awk '/Function : /{f=$3} /^ +\/\*[0-9a-f][0-9a-f][0-9a-f][0-9a-f]+\*\//{c[f]++} END{for(k in c) print c[k], k}' | sort -rn
