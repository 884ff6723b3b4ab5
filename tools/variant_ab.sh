#!/bin/bash
# Same-box variant A/B: device-resident MLUP/s of each compiled variant in fresh processes (two
# rounds, interleaved), then the DRAM bytes of one mid-run launch per variant under ncu.
#   bash tools/variant_ab.sh KIND N STEPS "VARIANTS" [ZCHUNKS]   (under gpurun; out: gpurun_out/)
set -u
cd "$(dirname "$0")/.."
kind=$1; n=$2; steps=$3; vars=$4; zc=${5:-0}
out=gpurun_out/variant_ab_${kind}_${n}.txt
: > $out
for rep in 1 2; do
  for v in $vars; do
    echo "rep=$rep $(python tools/one_step.py $kind $n $steps -1 $zc 0 $v)" >> $out
  done
done
for v in $vars; do
  GIRIH_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:zwave -s 2 -c 1 --csv python tools/one_step.py $kind $n 4 -1 $zc 0 $v 2>/dev/null \
    | grep -E "dram__|gpu__time" | awk -F'","' -v v=$v '{print "variant=" v, $(NF-2), $NF}' >> $out
done
cat $out
