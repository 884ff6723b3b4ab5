#!/bin/bash
# auto configuration (chained where the policy says so) on the small BASELINE C5 / C1-C3 grids
for kn in "1 64" "3 64" "0 64" "2 64" "1 128" "3 128" "0 128" "2 128" "0 256" "2 256" "3 256" "1 256"; do
  set -- $kn
  python tools/one_step.py $1 $2 100 0 0
done
