#!/bin/bash
# A/B of library variants on the C4 sweep, cold first-run schedule, interleaved on one box:
# tools/ab_c4.sh VARIANT... (tools/variants/libssb_VARIANT.so; "main" = the in-tree build)
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in "$@"; do
    if [ "$v" = main ]; then unset SSB_LIB; else export SSB_LIB=tools/variants/libssb_$v.so; fi
    echo "== $v"; COLD=1 python tools/probe_heavy.py 0
  done
done
