#!/bin/bash
# per-phase clock64 breakdown of single instances (debug build tools/libssb_timing.so)
cp paper_2410_17840_b200/libssb.so /tmp/libssb_real.so
trap 'cp /tmp/libssb_real.so paper_2410_17840_b200/libssb.so' EXIT
cp tools/libssb_timing.so paper_2410_17840_b200/libssb.so
for w in ${@:-trailworst larryworst c1}; do echo "== $w"; python tools/run_one.py $w 1 2>&1 | grep PHASES | head -4; done
