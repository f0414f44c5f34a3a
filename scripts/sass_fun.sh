#!/bin/sh
# SASS of one kernel (mangled-name substring) from the built library
cuobjdump -sass "${2:-paper_2604_16883_b200/_lib/libsinkr_cuda.so}" 2>/dev/null |
  awk -v pat="$1" '/Function : /{p = index($0, pat) > 0} p'
