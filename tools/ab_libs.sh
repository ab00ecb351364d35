#!/bin/bash
# A/B two builds of libzoomr on the same box: tools/ab_libs.sh libA.so libB.so [rounds]
for r in $(seq 1 ${3:-2}); do
  for L in "$1" "$2"; do
    echo -n "$L: "; ZOOMR_LIB_OVERRIDE=$PWD/$L VARS=${VARS:-nophys} python tools/ab_step.py 2>&1 | grep us/step
  done
done
