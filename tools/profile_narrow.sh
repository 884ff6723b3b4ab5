#!/bin/bash
# ncu captures of the output-columns-only (NARROW) default kernels (run under gpurun, one GPU):
# each plain command exits 0 first, then the same command runs under `ncu --set full`.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out
cap() {  # name, skip-launches, command...
  local name=$1 skip=$2; shift 2
  "$@" > $out/${name}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:zwave -s $skip -c 1 \
      -o $out/$name -f "$@" > $out/${name}_ncu.log 2>&1
  echo "$name rc=$?"
}
cap r2n_const7pt_256_chain 1 python tools/one_step.py 0 256 100 1
cap r2n_const25pt_512 3 env GIRIH_NO_GRAPHS=1 python tools/one_step.py 2 512 4 -1
cap r2n_const7pt_512 3 env GIRIH_NO_GRAPHS=1 python tools/one_step.py 0 512 4 -1
