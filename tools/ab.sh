#!/bin/bash
# Same-box A/B of library builds: tools/ab.sh "SWEEP ARGS" lib1.so lib2.so ... (alternates twice)
args="$1"; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    GIRIH_LIB=$(realpath "$lib") python tools/sweep.py $args
  done
done
