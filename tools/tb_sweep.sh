#!/bin/bash
# fused depth per pass on chained launches (auto z chunks, default variant per depth)
for n in 64 128 256; do for tb in 1 2 3 4; do python tools/one_step.py 0 $n 100 1 0 $tb; done; done
for n in 64 128; do for tb in 1 2; do python tools/one_step.py 2 $n 100 1 0 $tb; done; done
for n in 64 128; do for tb in 1 2 3 4; do python tools/one_step.py 1 $n 100 1 0 $tb; done; done
