#!/bin/bash
# Same-box A/B of two library builds (GIRIH_LIB): device-resident MLUP/s, fresh process per run,
# three interleaved rounds.   bash tools/lib_ab.sh KIND N STEPS CHAIN LIB_A LIB_B   (under gpurun)
set -u
cd "$(dirname "$0")/.."
kind=$1; n=$2; steps=$3; chain=$4; a=$5; b=$6
for rep in 1 2 3; do
  for lib in $a $b; do
    echo "$(basename $lib) rep=$rep $(GIRIH_LIB=$lib timeout 300 python tools/one_step.py $kind $n $steps $chain)"
  done
done
