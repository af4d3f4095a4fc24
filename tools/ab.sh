#!/bin/bash
# A/B the current libssb.so against tools/variants/libssb_$1.so with probe_ab.py (alternating, 2 rounds)
v=${1:-head}; mode=${2:-full}
for i in 1 2; do
  echo "== current"; python tools/probe_ab.py $mode
  echo "== $v"; SSB_LIB=tools/variants/libssb_$v.so python tools/probe_ab.py $mode
done
