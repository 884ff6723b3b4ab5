#!/bin/bash
# chained vs plain steps over z-chunk counts (device-resident, default variant per kind)
for kn in "0 256" "0 512" "1 256" "1 512" "2 256" "2 512" "3 256" "3 512" "1 128" "3 128"; do
  set -- $kn
  python tools/one_step.py $1 $2 100 -1 0
  for z in 4 8 16; do python tools/one_step.py $1 $2 100 1 $z; done
done
