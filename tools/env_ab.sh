#!/bin/bash
# Same-box A/B of environment switches: device-resident MLUP/s
# of each setting in fresh processes (two interleaved rounds), then the DRAM bytes of one mid-run
# launch per setting under ncu.
#   bash tools/env_ab.sh KIND N STEPS VARIANT "A=1 B=2;A=0;..." [TAG]   (under gpurun)
set -u
cd "$(dirname "$0")/.."
kind=$1; n=$2; steps=$3; var=$4; sets=$5; tag=${6:-env}
out=gpurun_out/${tag}_${kind}_${n}.txt
: > $out
IFS=';' read -ra S <<< "$sets"
for rep in 1 2; do
  for e in "${S[@]}"; do
    echo "[$e] rep=$rep $(env $e python tools/one_step.py $kind $n $steps -1 0 0 $var)" >> $out
  done
done
for e in "${S[@]}"; do
  env $e GIRIH_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:zwave -s 2 -c 1 --csv python tools/one_step.py $kind $n 4 -1 0 0 $var 2>/dev/null \
    | grep -E "dram__|gpu__time" | awk -F'","' -v e="$e" '{print "[" e "]", $(NF-2), $NF}' >> $out
done
cat $out
