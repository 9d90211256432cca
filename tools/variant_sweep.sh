#!/bin/bash
# time tools/step_timing.py against every built library variant
for so in paper_2601_17091_b200/_build/librocket_b200.so paper_2601_17091_b200/_build/variants/*.so; do
  echo "== $so"
  RK_LIB_PATH=$so python tools/step_timing.py ${1:-20000} 2>&1 | grep -v RK_PROFILE
done
