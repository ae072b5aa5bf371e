#!/bin/bash
# A/B of library builds on one box: tools/ab_step.py per build, alternated, twice.
#   bash tools/ab_libs.sh CONFIG ROUNDS lib1.so lib2.so ...
cfg=$1; rounds=$2; shift 2
for pass in 1 2; do
  for lib in "$@"; do
    echo -n "pass $pass $(basename $lib): "
    ENC_LIB_PATH=$lib python tools/ab_step.py --config $cfg --rounds $rounds base: 2>&1 | tail -1 | cut -c1-60
  done
done
