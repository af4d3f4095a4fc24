#!/bin/bash
# The GPU suite against the assert build (SSB_DEBUG: bounds of every table / ring / bucket index,
# request ids, block counts, and the KV pool conserved after every engine step), in place of
# compute-sanitizer (closed on this pool): tools/debug_suite.sh [pytest args]
cd "$(dirname "$0")/.."
bash tools/build_variant.sh debug -DSSB_DEBUG
SSB_LIB=tools/variants/libssb_debug.so python -m pytest tests -m gpu -x -q "$@"
SSB_LIB=tools/variants/libssb_debug.so python tools/sanitize.py
